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
    long long done[kBulkRing];            // written by the device: done[slot] = seq once bulk seq (of
                                          // that slot) is consumed (bulks may finish out of order)
    long long status;                     // written by the device: 0 ok, 1 timed out waiting for a bulk
    long long pad[7];
};

// Polling the ring and signalling "done" cross PCIe.  BH_BULK_ORDER=1: acquire/release at
// system scope; 0: relaxed system-scope accesses (every host-memory read of the kernel is
// uncached, and a value is used only after the load that returned it, so a descriptor is read
// after its sequence number, and a bulk's loads have all returned before its "done" is sent).
#ifndef BH_BULK_ORDER
#define BH_BULK_ORDER 0
#endif
__device__ __forceinline__ long long ld_acquire_sys(const long long *p) {
    long long v;
#if BH_BULK_ORDER
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
#else
    asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
#endif
    return v;
}
__device__ __forceinline__ void st_release_sys(long long *p, long long v) {
#if BH_BULK_ORDER
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#else
    asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#endif
}
// Device-memory side of the ring: CTA 0 alone polls the host ring across PCIe and forwards
// each descriptor here; the other CTAs poll this copy in L2 (148 pollers on host memory
// slowed every bulk to ~0.5 ms).
struct BulkDev {
    unsigned long long arrive[kBulkRing]; // CTA arrivals of the bulk in each slot (reset by its last CTA)
    long long pad[4];
    BulkDesc ring[kBulkRing];             // forwarded descriptors (n = -2: abort)
};

__device__ __forceinline__ long long ld_acquire_gpu(const long long *p) {
    long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(long long *p, long long v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Host columns are read with ld.global.cv (no stale cached copy: the host rewrites the same
// buffers bulk after bulk) when no shared memory is left for staging; otherwise each CTA
// pulls its share of a bulk into shared memory with 1-D TMA bulk copies (cp.async.bulk), two
// tiles in flight: large PCIe read requests instead of one 32-byte sector per warp load.
__device__ __forceinline__ double ld_host(const double *p) { return __ldcv(p); }

__device__ __forceinline__ uint32_t bulk_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bulk_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bulk_smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_mbar_tx(uint64_t *bar, uint32_t bytes) {      // expect, no arrive
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(bulk_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bulk_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(bulk_smem_u32(bar)), "r"(parity)
                     : "memory");
}
__device__ __forceinline__ void bulk_tma_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     bulk_smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(bulk_smem_u32(bar))
                 : "memory");
}

template <int DIM, bool W, int SINK, int VM>
__global__ void __launch_bounds__((ThreadsOf<SINK>::v), SINK == SINK_GLOBAL ? 2 : 1)
    k_bulk(FillP p, BulkCtl *ctl, BulkDev *dev, long long timeout_ns, int32_t stage_off, int32_t te) {
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
    uint32_t phase[2] = {0u, 0u};                 // TMA staging: mbarrier parity per stage
    if (te > 0 && threadIdx.x == 0) {
        constexpr int NCOL = DIM + (W ? 1 : 0);
        uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + stage_off + 2 * NCOL * (te + 4) * 8);
        bulk_mbar_init(mbar, 1);
        bulk_mbar_init(mbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long long seq = 1;
    for (;; ++seq) {
        if (threadIdx.x == 0) {
            const int slot = (int)((seq - 1) % kBulkRing);
            BulkDesc *dd = &dev->ring[slot];
            const unsigned long long t0 = globaltimer();
            long long n = -2;
            if (blockIdx.x == 0) {
                const BulkDesc *d = &ctl->ring[slot];
                while (true) {
                    if (ld_acquire_sys(&d->seq) == seq) {        // then the descriptor's fields
                        n = *reinterpret_cast<const volatile long long *>(&d->n);
                        break;
                    }
                    if (globaltimer() - t0 > (unsigned long long)timeout_ns) break;
                }
                if (n > 0) {
#pragma unroll
                    for (int a = 0; a < DIM; ++a) s_x[a] = reinterpret_cast<const double *const volatile *>(d->x)[a];
                    s_w = *reinterpret_cast<const double *const volatile *>(&d->w);
                    for (int a = 0; a < DIM; ++a) dd->x[a] = s_x[a];
                    dd->w = s_w;
                }
                dd->n = n;                                       // -2: abort (forwarded as well)
                st_release_gpu(&dd->seq, seq);
                if (n == -2) st_release_sys(&ctl->status, 1);
            } else {
                while (true) {
                    if (ld_acquire_gpu(&dd->seq) == seq) {
                        n = *reinterpret_cast<const volatile long long *>(&dd->n);
                        break;
                    }
                    if (globaltimer() - t0 > 2ull * (unsigned long long)timeout_ns) break;   // safety net
                    __nanosleep(32);
                }
                if (n > 0) {
#pragma unroll
                    for (int a = 0; a < DIM; ++a) s_x[a] = reinterpret_cast<const double *const volatile *>(dd->x)[a];
                    s_w = *reinterpret_cast<const double *const volatile *>(&dd->w);
                }
            }
            s_n = n;
        }
        __syncthreads();
        const long long n = s_n;
        if (n < 0) {
            if (n == -2) return;          // the host went away: leave the state unflushed
            break;                        // end of the sequence
        }
        // this CTA's contiguous share of the bulk, its inner boundaries on the 16-byte grid of
        // the first column (no off-grid ends for the TMA staging when the columns share a phase)
        const long long ph = (long long)((reinterpret_cast<uintptr_t>(s_x[0]) >> 3) & 1);
        auto bound = [&](unsigned long long k) -> long long {
            if (k == 0) return 0;
            if (k == G) return n;
            const long long b = ((((long long)(((unsigned long long)n * k) / G)) + ph) & ~1LL) - ph;
            return b < 0 ? 0 : (b > n ? n : b);
        };
        const long long lo = bound(blockIdx.x), hi = bound(blockIdx.x + 1);
        if (te > 0) {
            // TMA-staged: tiles of te events, stage k % 2.  Per column the 16-byte-aligned middle
            // of the tile comes by TMA; a leading / trailing event off the 16-byte grid is loaded
            // by thread 0 (no byte outside the bulk is read).  Event i of the tile sits at index
            // i - a0 + 2 - lead of the staged column, so the TMA destination is 16-byte aligned.
            constexpr int NCOL = DIM + (W ? 1 : 0);
            const int cstride = te + 4;                                  // doubles per staged column
            double *stg = reinterpret_cast<double *>(smem + stage_off);
            uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + stage_off + 2 * NCOL * cstride * 8);
            int *lead = reinterpret_cast<int *>(mbar + 2);
            const long long ntile = (hi - lo + te - 1) / te;
            auto issue = [&](long long k) {                              // thread 0
                const int st = (int)(k & 1);
                const long long a0 = lo + k * te, a1 = a0 + te < hi ? a0 + te : hi;
                uint32_t total = 0;
                long long b0[NCOL], b1[NCOL];
#pragma unroll
                for (int c = 0; c < NCOL; ++c) {
                    const double *col = c < DIM ? s_x[c] : s_w;
                    const int ld = (int)((reinterpret_cast<uintptr_t>(col + a0) >> 3) & 1);
                    b0[c] = a0 + ld;
                    b1[c] = a1 - (long long)((reinterpret_cast<uintptr_t>(col + a1) >> 3) & 1);
                    if (b1[c] < b0[c]) b1[c] = b0[c];
                    lead[st * NCOL + c] = ld;
                    total += (uint32_t)((b1[c] - b0[c]) * 8);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk_mbar_tx(mbar + st, total);
#pragma unroll
                for (int c = 0; c < NCOL; ++c)
                    if (b1[c] > b0[c])
                        bulk_tma_g2s(stg + (st * NCOL + c) * cstride + 2, (c < DIM ? s_x[c] : s_w) + b0[c],
                                     (uint32_t)((b1[c] - b0[c]) * 8), mbar + st);
                // the off-grid ends (<= 2 events per column), all loads in flight together
                double hv[NCOL], tv[NCOL];
#pragma unroll
                for (int c = 0; c < NCOL; ++c) {
                    const double *col = c < DIM ? s_x[c] : s_w;
                    const long long t = b1[c] > b0[c] ? b1[c] : b0[c];       // first event after the TMA part
                    if (b0[c] > a0) hv[c] = ld_host(col + a0);
                    if (t < a1) tv[c] = ld_host(col + t);
                }
#pragma unroll
                for (int c = 0; c < NCOL; ++c) {
                    double *dst = stg + (st * NCOL + c) * cstride + 2 - lead[st * NCOL + c];
                    const long long t = b1[c] > b0[c] ? b1[c] : b0[c];
                    if (b0[c] > a0) dst[0] = hv[c];
                    if (t < a1) dst[t - a0] = tv[c];
                }
                bulk_mbar_arrive(mbar + st);                             // the phase completes when
            };                                                           // the TMA bytes land too
            if (threadIdx.x == 0 && ntile > 0) issue(0);
            for (long long k = 0; k < ntile; ++k) {
                const int st = (int)(k & 1);
                if (threadIdx.x == 0 && k + 1 < ntile) issue(k + 1);    // stage st^1 was released below
                bulk_mbar_wait(mbar + st, phase[st]);
                phase[st] ^= 1u;
                const long long a0 = lo + k * te, a1 = a0 + te < hi ? a0 + te : hi;
                for (long long i0 = a0; i0 < a1; i0 += blockDim.x) {
                    const long long i = i0 + threadIdx.x;
                    if (SINK == SINK_PRIVA) __syncwarp();
                    if (i < a1) {
                        double x[DIM];
#pragma unroll
                        for (int a = 0; a < DIM; ++a) x[a] = stg[(st * NCOL + a) * cstride + (i - a0) + 2 - lead[st * NCOL + a]];
                        const double wv = W ? stg[(st * NCOL + NCOL - 1) * cstride + (i - a0) + 2 - lead[st * NCOL + NCOL - 1]] : 1.0;
                        do_event<DIM, W, VM>(p, x, wv, sink, acc, smem);
                    }
                }
                __syncthreads();                                         // stage st free again
            }
        } else {
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
        }
        __syncthreads();                  // every load of this CTA's share has returned
        if (threadIdx.x == 0) {
            // per-slot arrivals: with several bulks in flight a fast CTA may finish bulk seq+1
            // before a slow one finishes seq
            const int slot = (int)((seq - 1) % kBulkRing);
            __threadfence();
            if (atomicAdd(&dev->arrive[slot], 1ull) == G - 1) {   // the last CTA of bulk `seq`
                dev->arrive[slot] = 0ull;                          // the slot's next bulk is seq+4,
                atomicAdd(p.entries, (unsigned long long)n);       // posted after done[slot] = seq
                __threadfence();
                if (BH_BULK_ORDER) __threadfence_system();
                st_release_sys(&ctl->done[slot], seq);
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
        const int slot = (int)((seq - 1) % kBulkRing);
        __threadfence();
        if (atomicAdd(&dev->arrive[slot], 1ull) == G - 1) {
            __threadfence_system();                   // the flushed bins / stats before "done"
            st_release_sys(&ctl->done[slot], seq);
        }
    }
}

}  // namespace bh
