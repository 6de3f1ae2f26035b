// bhist_bulk.cuh — persistent bulk consumer (bh_bulk_begin / bh_bulk_submit / bh_bulk_end).
//
// The paper's GPU fill runs per bulk of events (32768 by default): "transfers
// bulk of events to the GPU and launches kernels ... per bulk", and at such
// sizes "large kernel launch and memory transfer overheads" dominate.  Here
// one kernel stays resident for a whole sequence of bulks: the host posts each bulk as a
// descriptor (event count + pointers to its PINNED host columns) in a ring in mapped host
// memory; every CTA polls the ring, reads its share of the bulk's events straight from host
// memory over PCIe (zero-copy: no cudaMemcpy, no staging buffer, no launch per bulk), runs
// the three steps of PAPER.md:126 into its block-private bins and register statistics, and
// the last CTA to finish a bulk tells the host that the bulk's host bytes are consumed (the
// buffer may then be refilled: the race of PAPER.md:223 cannot happen).  Private bins are
// flushed and the statistics reduced once, when the host posts the end of the sequence.
#pragma once
#include "bhist_kernels.cuh"

namespace bh {

constexpr int kBulkRing = 4;              // descriptors in flight

struct BulkDesc {                         // written by the host (plain stores, then seq last)
    long long seq;                        // 1, 2, ...: the bulk's sequence number (0: never posted)
    long long n;                          // events; -1: end of the sequence
    const double *x[kMaxDim];             // device-accessible (UVA) pointers to pinned host columns
    const double *w;                      // weights or nullptr
    long long pad[2];
};

struct BulkCtl {                          // pinned, mapped host memory (cudaHostAllocMapped)
    BulkDesc ring[kBulkRing];             // bulk seq uses ring[(seq - 1) % kBulkRing]
    long long done;                       // written by the device: last bulk whose bytes are consumed
    long long status;                     // written by the device: 0 ok, 1 timed out waiting for a bulk
    long long pad[6];
};

__device__ __forceinline__ long long ld_acquire_sys(const long long *p) {
    long long v;
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(long long *p, long long v) {
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Host columns are read with ld.global.cv (no stale cached copy: the host rewrites the same
// buffers bulk after bulk).
__device__ __forceinline__ double ld_host(const double *p) { return __ldcv(p); }

template <int DIM, bool W, int SINK, int VM>
__global__ void __launch_bounds__((ThreadsOf<SINK>::v), SINK == SINK_GLOBAL ? 2 : 1)
    k_bulk(FillP p, BulkCtl *ctl, unsigned long long *arrive, long long timeout_ns) {
    extern __shared__ __align__(16) unsigned char smem[];
    using Sink_t = typename SinkOf<SINK, W>::T;
    Sink_t sink;
    if constexpr (SINK == SINK_GLOBAL) sink.pp = &p;
    if constexpr (SINK == SINK_CACHE) sink.pp = &p;
    if constexpr (SINK == SINK_CACHE) sink.init(smem, p.cache_slots);
    else if constexpr (SINK == SINK_PRIV || SINK == SINK_PRIVA) sink.init(smem, p.G, p.replicas, p.wc_off);
    else sink.init(smem, p.G);
    if constexpr (VM == 1 || VM == 3) stage_axes<DIM>(p.ax, smem);
    __syncthreads();

    __shared__ long long s_n;
    __shared__ const double *s_x[kMaxDim];
    __shared__ const double *s_w;
    Acc<DIM, W> acc;
    acc.zero();
    const unsigned long long G = gridDim.x;
    long long seq = 1;
    for (;; ++seq) {
        if (threadIdx.x == 0) {
            const BulkDesc *d = &ctl->ring[(seq - 1) % kBulkRing];
            const unsigned long long t0 = globaltimer();
            long long n = -2;
            while (true) {
                if (ld_acquire_sys(&d->seq) == seq) {        // the descriptor's fields are visible now
                    n = *reinterpret_cast<const volatile long long *>(&d->n);
                    break;
                }
                if (globaltimer() - t0 > (unsigned long long)timeout_ns) break;
                __nanosleep(64);
            }
            s_n = n;
            if (n > 0) {
#pragma unroll
                for (int a = 0; a < DIM; ++a) s_x[a] = reinterpret_cast<const double *const volatile *>(d->x)[a];
                s_w = *reinterpret_cast<const double *const volatile *>(&d->w);
            }
            if (n == -2 && blockIdx.x == 0) st_release_sys(&ctl->status, 1);
        }
        __syncthreads();
        const long long n = s_n;
        if (n < 0) {
            if (n == -2) return;          // the host went away: leave the state unflushed
            break;                        // end of the sequence
        }
        // this CTA's contiguous share of the bulk, coalesced over its threads
        const long long lo = (long long)(((unsigned long long)n * blockIdx.x) / G);
        const long long hi = (long long)(((unsigned long long)n * (blockIdx.x + 1)) / G);
        // warp-uniform trips: SINK_PRIVA's warp hot-bin caches are used by converged full warps
        for (long long i0 = lo; i0 < hi; i0 += blockDim.x) {
            const long long i = i0 + threadIdx.x;
            if (SINK == SINK_PRIVA) __syncwarp();
            if (i < hi) {
                double x[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) x[a] = ld_host(s_x[a] + i);
                do_event<DIM, W, VM>(p, x, W ? ld_host(s_w + i) : 1.0, sink, acc, smem);
            }
        }
        __syncthreads();                  // every load of this CTA's share has returned
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned long long old = atomicAdd(arrive, 1ull);
            if (old == (unsigned long long)seq * G - 1) {      // the last CTA of bulk `seq`
                atomicAdd(p.entries, (unsigned long long)n);
                __threadfence_system();
                st_release_sys(&ctl->done, seq);
            }
        }
    }
    if constexpr (SINK != SINK_GLOBAL) {
        sink.drain();
        __syncthreads();
        sink.flush(p, smem);
    }
    acc.finalize_unit();
    block_stats_finish<Acc<DIM, W>::K>(p, acc.s);     // entries_add = 0: added per bulk above
    // the end of the sequence is "consumed" once every CTA has flushed (bh_bulk_end waits for it)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(arrive, 1ull) == (unsigned long long)seq * G - 1) {
            __threadfence_system();
            st_release_sys(&ctl->done, seq);
        }
    }
}

}  // namespace bh
