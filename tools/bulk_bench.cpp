// Probe (not product code): the per-bulk cost of the paper's fill loop through the C ABI alone
// (no Python): bh_fill_host per bulk vs the persistent consumer (bh_bulk_fill per bulk, and
// bh_bulk_submit with bulks in flight), TH1D 1000 fixed bins, bulks of 32768 pinned events.
// Build: g++ -O2 -I include tools/bulk_bench.cpp -L paper_2401_13310_b200 -lbhist -L/usr/local/cuda/lib64 -lcudart
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "bhist.h"
#define CK(x) do { int r_ = (x); if (r_) { printf("%s -> %d %s\n", #x, r_, bh_last_error()); exit(1); } } while (0)
int main(int argc, char **argv) {
    const long total = 1L << 23, bulk = argc > 1 ? atol(argv[1]) : 32768;
    double *host;
    cudaHostAlloc((void **)&host, sizeof(double) * total, cudaHostAllocDefault);
    for (long i = 0; i < total; ++i) host[i] = (double)((i * 2654435761u) % 1000003) / 1000003.0;
    bh_axis ax = {1000, 0.0, 1.0, nullptr};
    bh_hist *h;
    CK(bh_create(1, &ax, 0, &h));
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    for (int rep = 0; rep < 2; ++rep) {
        CK(bh_reset(h, nullptr));
        CK(bh_set_chunk(h, bulk));
        cudaDeviceSynchronize();
        auto t0 = now();
        for (long i = 0; i < total; i += bulk) { const double *c[1] = {host + i}; CK(bh_fill_host(h, bulk, c, nullptr, nullptr)); }
        int64_t e; CK(bh_read(h, nullptr, nullptr, nullptr, &e, nullptr));
        auto t1 = now();
        CK(bh_reset(h, nullptr));
        cudaDeviceSynchronize();
        auto t2 = now();
        CK(bh_bulk_begin(h, 0, 0, nullptr));
        auto t2b = now();
        for (long i = 0; i < total; i += bulk) { const double *c[1] = {host + i}; CK(bh_bulk_fill(h, bulk, c, nullptr)); }
        auto t2c = now();
        CK(bh_bulk_end(h));
        CK(bh_read(h, nullptr, nullptr, nullptr, &e, nullptr));
        auto t3 = now();
        CK(bh_reset(h, nullptr));
        cudaDeviceSynchronize();
        auto t4 = now();
        CK(bh_bulk_begin(h, 0, 0, nullptr));
        int64_t t = 0;
        for (long i = 0; i < total; i += bulk) { const double *c[1] = {host + i}; CK(bh_bulk_submit(h, bulk, c, nullptr, &t)); }
        CK(bh_bulk_wait(h, t));
        CK(bh_bulk_end(h));
        CK(bh_read(h, nullptr, nullptr, nullptr, &e, nullptr));
        auto t5 = now();
        const double nb = (double)total / bulk;
        printf("bulk %ld: fill_host %.2f us/bulk | consumer sync %.2f us/bulk (begin %.1f us, loop %.2f us/bulk, end+read %.1f us) | pipelined %.2f us/bulk | entries %lld\n",
               bulk, us(t0, t1) / nb, us(t2, t3) / nb, us(t2, t2b), us(t2b, t2c) / nb, us(t2c, t3), us(t4, t5) / nb, (long long)e);
    }
    return 0;
}
