// Design probe 6 (not product code): float64 (w, w^2) adds into 1M random L2-resident cells
// (C3w's bin space, 16 MB) -- does pairing the two halves of a cell into ONE warp RED
// instruction (two lanes, one 16-byte cell, one 32-byte sector) raise the L2 atomic rate?
//   0 u64     : RED.E.ADD.64 of 1 per event (one array)                 -- integer baseline
//   1 split   : RED.E.ADD.F64 to sumw[b] and sumw2[b] (two arrays, two instructions)
//   2 inter   : RED.E.ADD.F64 to cell[b].x, then cell[b].y (interleaved, two instructions)
//   3 paired  : lanes (2i, 2i+1) add (w, w^2) of one event into cell[b] in ONE instruction;
//               two instructions cover the warp's 32 events (16 events each)
//   4 paired_u64: like 3 with u64 adds (integer reference for the pairing effect)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb6 mb6.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(512) k(double *a, double *b, unsigned long long *u, int ncell, int iters) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
        const uint32_t h = hsh(tid * 0x9E3779B9u + it * 0x85EBCA6Bu);
        const uint32_t c = __umulhi(h, ncell);
        const double w = 0.5 + (h & 1023) * (1.0 / 1024);
        if (MODE == 0) {
            atomicAdd(u + c, 1ull);
        } else if (MODE == 1) {
            atomicAdd(a + c, w);
            atomicAdd(b + c, w * w);
        } else if (MODE == 2) {
            atomicAdd(a + 2 * (size_t)c, w);
            atomicAdd(a + 2 * (size_t)c + 1, w * w);
        } else if (MODE == 3) {
            const int src0 = lane >> 1, src1 = 16 + (lane >> 1);
            const uint32_t c0 = __shfl_sync(0xffffffffu, c, src0), c1 = __shfl_sync(0xffffffffu, c, src1);
            const double w0 = __shfl_sync(0xffffffffu, w, src0), w1 = __shfl_sync(0xffffffffu, w, src1);
            const int k = lane & 1;
            atomicAdd(a + 2 * (size_t)c0 + k, k ? w0 * w0 : w0);
            atomicAdd(a + 2 * (size_t)c1 + k, k ? w1 * w1 : w1);
        } else {
            const int src0 = lane >> 1, src1 = 16 + (lane >> 1);
            const uint32_t c0 = __shfl_sync(0xffffffffu, c, src0), c1 = __shfl_sync(0xffffffffu, c, src1);
            const int k = lane & 1;
            atomicAdd(u + 2 * (size_t)c0 + k, 1ull);
            atomicAdd(u + 2 * (size_t)c1 + k, 1ull);
        }
    }
}

template <int MODE>
void run(const char *name, double *a, double *b, unsigned long long *u, int ncell, int blocks, int thr, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<blocks, thr>>>(a, b, u, ncell, iters);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k<MODE><<<blocks, thr>>>(a, b, u, ncell, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ev = (double)blocks * thr * iters;
    printf("%-12s cells %8d blocks %5d thr %4d  %8.3f ms  %7.1f G events/s  %s\n", name, ncell, blocks, thr, best,
           ev / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int ncell = 1 << 20;
    double *a, *b; unsigned long long *u;
    cudaMalloc(&a, 2 * sizeof(double) * ncell);
    cudaMalloc(&b, sizeof(double) * ncell);
    cudaMalloc(&u, 2 * sizeof(unsigned long long) * ncell);
    cudaMemset(a, 0, 2 * sizeof(double) * ncell);
    cudaMemset(b, 0, sizeof(double) * ncell);
    cudaMemset(u, 0, 2 * sizeof(unsigned long long) * ncell);
    for (int nc : {1 << 20, 1 << 16}) {
        for (int blocks : {148 * 4, 148 * 8}) {
            const int thr = 512, iters = (1 << 28) / (blocks * thr);
            run<0>("u64", a, b, u, nc, blocks, thr, iters);
            run<1>("f64 split", a, b, u, nc, blocks, thr, iters);
            run<2>("f64 inter", a, b, u, nc, blocks, thr, iters);
            run<3>("f64 paired", a, b, u, nc, blocks, thr, iters);
            run<4>("u64 paired", a, b, u, nc, blocks, thr, iters);
        }
    }
    return 0;
}
