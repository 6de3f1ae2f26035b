// Design probe 5 (not product code): reading PINNED HOST memory from a kernel, 148 CTAs:
// 1-D TMA bulk copies (cp.async.bulk global->shared) of CH bytes with D copies in flight per
// CTA, vs per-thread ld.global.cv loads, vs cudaMemcpyAsync (copy engine).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb5 mb5.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_tma(const char *src, size_t bytes, int ch, int depth, unsigned long long *sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)depth * ch);
    if (threadIdx.x == 0) {
        for (int d = 0; d < depth; ++d) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + d)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t per = bytes / gridDim.x / ch * ch;
    const char *s = src + (size_t)blockIdx.x * per;
    const int nch = (int)(per / ch);
    unsigned long long acc = 0;
    if (threadIdx.x == 0) {
        uint32_t ph[64] = {};
        for (int c = 0; c < nch + depth; ++c) {
            if (c >= depth) {                         // wait the copy issued depth steps ago
                const int d = (c - depth) % depth;
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done) : "r"(su(bar + d)), "r"(ph[d]) : "memory");
                ph[d] ^= 1u;
                acc += sm[(size_t)d * ch];
            }
            if (c < nch) {
                const int d = c % depth;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + d)), "r"(ch) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su(sm + (size_t)d * ch)), "l"(s + (size_t)c * ch), "r"(ch), "r"(su(bar + d)) : "memory");
            }
        }
        atomicAdd(sink, acc);
    }
}
__global__ void k_ldcv(const double *src, size_t n, unsigned long long *sink) {
    double a = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) a += __ldcv(src + i);
    if (a == 12345.678) atomicAdd(sink, 1ull);
}
int main() {
    const size_t bytes = 256ull << 20;
    char *h;
    cudaHostAlloc((void **)&h, bytes, cudaHostAllocMapped);
    for (size_t i = 0; i < bytes; i += 4096) h[i] = 1;
    char *d;
    cudaMalloc(&d, bytes);
    unsigned long long *sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    auto T = [&](const char *nm, auto L) {
        L();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        L();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("%-40s %8.3f ms  %6.1f GB/s  %s\n", nm, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    T("cudaMemcpyAsync H2D", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); });
    T("ld.global.cv, 148x1024 threads", [&] { k_ldcv<<<148, 1024>>>((const double *)h, bytes / 8, sink); });
    T("ld.global.cv, 1184x1024 threads", [&] { k_ldcv<<<1184, 1024>>>((const double *)h, bytes / 8, sink); });
    for (int ch : {2048, 8192, 32768})
        for (int depth : {1, 2, 4, 8}) {
            if ((size_t)ch * depth > 190 * 1024) continue;
            char nm[64];
            snprintf(nm, 64, "TMA %6d B x %d in flight per CTA", ch, depth);
            T(nm, [&] { k_tma<<<148, 32, (size_t)ch * depth + 8 * depth>>>(h, bytes, ch, depth, sink); });
        }
    return 0;
}
