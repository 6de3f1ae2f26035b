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

constexpr int kBulkStages = 4;               // TMA-staged tiles in flight per CTA

struct BulkTile {                             // per stage, written by the scheduler before its arrive
    long long a0, a1;                         // event range of the tile within its bulk
    long long seq, n;                         // the bulk
    int kind;                                 // 0 tile, 1 end of the sequence, 2 abort
    int last;                                 // the last tile of this CTA's share of the bulk
    int lead[kMaxDim + 1];                    // per column: 1 if the tile starts off the 16-byte grid
};

__device__ __forceinline__ bool bulk_mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(bulk_smem_u32(bar)), "r"(parity)
                 : "memory");
    return done != 0;
}

// The bulk `seq`'s descriptor, if posted (CTA 0: the host ring, forwarded to the device
// mailbox; other CTAs: the mailbox).  Returns false if not there yet.
// line/lbar (CTA 0 of the TMA path): each poll fetches the host descriptor's whole 64-byte
// line with one TMA bulk copy -- one PCIe round trip and a consistent snapshot of the line
// (the host writes the fields before the sequence number), instead of one round trip per field.
template <int NCOL, int DIM>
__device__ __forceinline__ bool bulk_desc(BulkCtl *ctl, BulkDev *dev, long long seq, long long &n,
                                          const double *(&col)[NCOL], BulkDesc *line = nullptr,
                                          uint64_t *lbar = nullptr, uint32_t *lph = nullptr) {
    const int slot = (int)((seq - 1) % kBulkRing);
    BulkDesc *dd = &dev->ring[slot];
    const BulkDesc *d = blockIdx.x == 0 ? &ctl->ring[slot] : dd;
    if (blockIdx.x == 0 && line) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bulk_mbar_expect_tx(lbar, (uint32_t)sizeof(BulkDesc));
        bulk_tma_g2s(line, d, (uint32_t)sizeof(BulkDesc), lbar);
        bulk_mbar_wait(lbar, *lph);
        *lph ^= 1u;
        d = line;
        if (d->seq != seq) return false;
    } else if ((blockIdx.x == 0 ? ld_acquire_sys(&d->seq) : ld_acquire_gpu(&d->seq)) != seq) {
        return false;
    }
    n = *reinterpret_cast<const volatile long long *>(&d->n);
    if (n > 0) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) col[a] = reinterpret_cast<const double *const volatile *>(d->x)[a];
        if (NCOL > DIM) col[NCOL - 1] = *reinterpret_cast<const double *const volatile *>(&d->w);
    }
    if (blockIdx.x == 0) {                    // forward to the other CTAs
        if (n > 0) {
            for (int a = 0; a < DIM; ++a) dd->x[a] = col[a];
            dd->w = NCOL > DIM ? col[NCOL - 1] : nullptr;
        }
        dd->n = n;
        st_release_gpu(&dd->seq, seq);
    }
    return true;
}

// bulk `seq` is done by this CTA: count it; the last CTA adds the entries and tells the host
__device__ __forceinline__ void bulk_arrive(BulkCtl *ctl, BulkDev *dev, const FillP &p, long long seq, long long n) {
    const int slot = (int)((seq - 1) % kBulkRing);
    __threadfence();
    if (atomicAdd(&dev->arrive[slot], 1ull) == (unsigned long long)gridDim.x - 1) {
        dev->arrive[slot] = 0ull;             // the slot's next bulk is seq+4, posted after done[slot] = seq
        if (n > 0) atomicAdd(p.entries, (unsigned long long)n);
        __threadfence();
        if (BH_BULK_ORDER) __threadfence_system();
        st_release_sys(&ctl->done[slot], seq);
    }
}

// This CTA's contiguous share [lo, hi) of a bulk of n events, the inner boundaries on the
// 16-byte grid of the first column (no off-grid tile ends when the columns share a phase).
__device__ __forceinline__ void bulk_share(long long n, const double *col0, long long &lo, long long &hi) {
    const unsigned long long G = gridDim.x;
    const long long ph = (long long)((reinterpret_cast<uintptr_t>(col0) >> 3) & 1);
    auto bound = [&](unsigned long long k) -> long long {
        if (k == 0) return 0;
        if (k == G) return n;
        const long long b = ((((long long)((unsigned long long)n * k / G)) + ph) & ~1LL) - ph;
        return b < 0 ? 0 : (b > n ? n : b);
    };
    lo = bound(blockIdx.x);
    hi = bound(blockIdx.x + 1);
}

template <int DIM, bool W, int SINK, int VM>
__global__ void __launch_bounds__((ThreadsOf<SINK>::v), SINK == SINK_GLOBAL ? 2 : 1)
    k_bulk(FillP p, BulkCtl *ctl, BulkDev *dev, long long timeout_ns, int32_t stage_off, int32_t te) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NCOL = DIM + (W ? 1 : 0);
    using Sink_t = typename SinkOf<SINK, W>::T;
    Sink_t sink;
    if constexpr (SINK == SINK_GLOBAL || SINK == SINK_CACHE) sink.bind(p);
    if constexpr (SINK == SINK_CACHE) sink.init(smem, p.cache_slots);
    else if constexpr (SINK == SINK_PRIV || SINK == SINK_PRIVA) sink.init(smem, p.G, p.replicas, p.wc_off);
    else sink.init(smem, p.G);
    if constexpr (VM == 1 || VM == 3) stage_axes<DIM>(p.ax, smem);

    __shared__ long long s_end;               // sequence number of the end descriptor; < 0: aborted
    Acc<DIM, W> acc;
    acc.zero();

    if (te > 0) {
        // ---- warp-specialized: the last warp's lane 0 schedules (descriptors, TMA bulk copies of
        // the host columns into kBulkStages shared-memory stages, per-bulk completion); the other
        // warps consume tiles.  Tiles of the NEXT bulk are fetched while the current one is
        // processed, so the PCIe round trips of consecutive bulks overlap.  Per column the 16-byte-
        // aligned middle of a tile comes by TMA, a leading / trailing event off the grid by a load
        // (no byte outside the bulk is read); event i of a tile sits at index i - a0 + 2 - lead.
        const int cstride = te + 4;
        double *stg = reinterpret_cast<double *>(smem + stage_off);
        uint64_t *full = reinterpret_cast<uint64_t *>(smem + stage_off + (size_t)kBulkStages * NCOL * cstride * 8);
        uint64_t *empty = full + kBulkStages;
        BulkTile *meta = reinterpret_cast<BulkTile *>(empty + kBulkStages);
        BulkDesc *line = reinterpret_cast<BulkDesc *>(meta + kBulkStages);   // 16-byte aligned
        uint64_t *lbar = reinterpret_cast<uint64_t *>(line + 1);
        const int nw = (int)(blockDim.x >> 5), warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
        if (threadIdx.x == 0) {
            for (int s = 0; s < kBulkStages; ++s) {
                bulk_mbar_init(full + s, 1);
                bulk_mbar_init(empty + s, (uint32_t)((nw - 1) * 32));   // every consumer thread
            }
            bulk_mbar_init(lbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (warp == nw - 1) {
            if (lane == 0) {
                // ---- scheduler
                long long seq = 0, n = 0, lo = 0, hi = 0, k = 0, ntile = 0;
                const double *col[NCOL] = {};
                bool have = false, ended = false;
                long long issued = 0, retired = 0;
                uint32_t eph[kBulkStages] = {};
                uint32_t lph = 0;
                unsigned long long t0 = globaltimer();
                auto retire = [&](bool block) {       // the oldest tile in flight, once consumed
                    const int st = (int)(retired % kBulkStages);
                    if (!block && !bulk_mbar_test(empty + st, eph[st])) return false;
                    bulk_mbar_wait(empty + st, eph[st]);
                    eph[st] ^= 1u;
                    if (meta[st].last) bulk_arrive(ctl, dev, p, meta[st].seq, meta[st].n);
                    ++retired;
                    return true;
                };
                while (true) {
                    // retire consumed tiles (bulk completions go out as early as possible)
                    while (retired < issued - (ended ? 1 : 0) && retire(false)) {}
                    if (ended) {
                        if (retired >= issued - 1) break;
                        continue;
                    }
                    if (issued - retired >= kBulkStages) { retire(true); continue; }
                    if (!have) {                      // the next bulk's descriptor
                        long long m;
                        if (!bulk_desc<NCOL, DIM>(ctl, dev, seq + 1, m, col, line, lbar, &lph)) {
                            if (issued == retired && globaltimer() - t0 > (unsigned long long)timeout_ns) m = -2;
                            else continue;            // poll again (and retire meanwhile)
                            if (blockIdx.x == 0) {    // abort: forward it, tell the host
                                BulkDesc *dd = &dev->ring[seq % kBulkRing];
                                dd->n = -2;
                                st_release_gpu(&dd->seq, seq + 1);
                                st_release_sys(&ctl->status, 1);
                            }
                        }
                        ++seq;
                        t0 = globaltimer();
                        if (m < 0) {                  // end (-1) or abort (-2): a marker tile
                            const int st = (int)(issued % kBulkStages);
                            meta[st].kind = m == -1 ? 1 : 2;
                            meta[st].last = 0;
                            s_end = m == -1 ? seq : -1;
                            bulk_mbar_arrive(full + st);
                            ++issued;
                            ended = true;
                            continue;
                        }
                        n = m;
                        if (n > 0) bulk_share(n, col[0], lo, hi);
                        else lo = hi = 0;
                        ntile = hi > lo ? (hi - lo + te - 1) / te : 1;   // an empty share: one empty tile
                        k = 0;
                        have = true;
                    }
                    // issue tile k of bulk seq into the next stage
                    const int st = (int)(issued % kBulkStages);
                    const long long a0 = lo + k * te, a1 = a0 + te < hi ? a0 + te : hi;
                    BulkTile &mt = meta[st];
                    mt.a0 = a0;
                    mt.a1 = a1;
                    mt.seq = seq;
                    mt.n = n;
                    mt.kind = 0;
                    mt.last = k + 1 == ntile;
                    uint32_t total = 0;
                    long long b0[NCOL], b1[NCOL];
#pragma unroll
                    for (int c = 0; c < NCOL; ++c) {
                        const int ld = a1 > a0 ? (int)((reinterpret_cast<uintptr_t>(col[c] + a0) >> 3) & 1) : 0;
                        b0[c] = a0 + ld;
                        b1[c] = a1 > a0 ? a1 - (long long)((reinterpret_cast<uintptr_t>(col[c] + a1) >> 3) & 1) : a0;
                        if (b1[c] < b0[c]) b1[c] = b0[c];
                        mt.lead[c] = ld;
                        total += (uint32_t)((b1[c] - b0[c]) * 8);
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    bulk_mbar_tx(full + st, total);
#pragma unroll
                    for (int c = 0; c < NCOL; ++c)
                        if (b1[c] > b0[c])
                            bulk_tma_g2s(stg + (size_t)(st * NCOL + c) * cstride + 2, col[c] + b0[c],
                                         (uint32_t)((b1[c] - b0[c]) * 8), full + st);
                    double hv[NCOL], tv[NCOL];                  // off-grid ends, in flight together
#pragma unroll
                    for (int c = 0; c < NCOL; ++c) {
                        const long long t = b1[c] > b0[c] ? b1[c] : b0[c];
                        if (b0[c] > a0) hv[c] = ld_host(col[c] + a0);
                        if (t < a1) tv[c] = ld_host(col[c] + t);
                    }
#pragma unroll
                    for (int c = 0; c < NCOL; ++c) {
                        double *dst = stg + (size_t)(st * NCOL + c) * cstride + 2 - mt.lead[c];
                        const long long t = b1[c] > b0[c] ? b1[c] : b0[c];
                        if (b0[c] > a0) dst[0] = hv[c];
                        if (t < a1) dst[t - a0] = tv[c];
                    }
                    bulk_mbar_arrive(full + st);                // completes with the TMA bytes
                    ++issued;
                    if (++k == ntile) have = false;
                }
            }
            __syncwarp();
        } else {
            // ---- consumers: tiles in issue order
            const int ct = (int)threadIdx.x, nct = (nw - 1) * 32;
            uint32_t fph[kBulkStages] = {};
            for (long long t = 0;; ++t) {
                const int st = (int)(t % kBulkStages);
                bulk_mbar_wait(full + st, fph[st]);
                fph[st] ^= 1u;
                const BulkTile &mt = meta[st];
                if (mt.kind != 0) break;
                const long long a0 = mt.a0, a1 = mt.a1;
                int lead[NCOL];
#pragma unroll
                for (int c = 0; c < NCOL; ++c) lead[c] = mt.lead[c];
                for (long long i0 = a0; i0 < a1; i0 += nct) {    // warp-uniform trips (PRIVA)
                    const long long i = i0 + ct;
                    if (SINK == SINK_PRIVA) __syncwarp();
                    if (i < a1) {
                        double x[DIM];
#pragma unroll
                        for (int a = 0; a < DIM; ++a) x[a] = stg[(size_t)(st * NCOL + a) * cstride + (i - a0) + 2 - lead[a]];
                        const double wv = W ? stg[(size_t)(st * NCOL + NCOL - 1) * cstride + (i - a0) + 2 - lead[NCOL - 1]] : 1.0;
                        do_event<DIM, W, VM>(p, x, wv, sink, acc, smem);
                    }
                }
                bulk_mbar_arrive(empty + st);                   // this thread is done with the stage
            }
        }
        __syncthreads();
        if (s_end < 0) return;                // the host went away: leave the state unflushed
    } else {
        // ---- no shared memory left for staging: every CTA polls the descriptors itself (CTA 0
        // the host ring, forwarding) and its threads read their share with ld.global.cv
        __shared__ long long s_n;
        __shared__ const double *s_col[NCOL];
        __syncthreads();
        for (long long seq = 1;; ++seq) {
            if (threadIdx.x == 0) {
                const unsigned long long t0 = globaltimer();
                long long n = -2;
                const double *col[NCOL] = {};
                while (!bulk_desc<NCOL, DIM>(ctl, dev, seq, n, col)) {
                    if (globaltimer() - t0 > (unsigned long long)timeout_ns) {
                        n = -2;
                        if (blockIdx.x == 0) {
                            BulkDesc *dd = &dev->ring[(seq - 1) % kBulkRing];
                            dd->n = -2;
                            st_release_gpu(&dd->seq, seq);
                            st_release_sys(&ctl->status, 1);
                        }
                        break;
                    }
                }
                s_n = n;
                for (int c = 0; c < NCOL; ++c) s_col[c] = col[c];
                if (n == -1) s_end = seq;
                if (n == -2) s_end = -1;
            }
            __syncthreads();
            const long long n = s_n;
            if (n < 0) break;
            long long lo = 0, hi = 0;
            if (n > 0) bulk_share(n, s_col[0], lo, hi);
            for (long long i0 = lo; i0 < hi; i0 += blockDim.x) {  // warp-uniform trips (PRIVA)
                const long long i = i0 + threadIdx.x;
                if (SINK == SINK_PRIVA) __syncwarp();
                if (i < hi) {
                    double x[DIM];
#pragma unroll
                    for (int a = 0; a < DIM; ++a) x[a] = ld_host(s_col[a] + i);
                    do_event<DIM, W, VM>(p, x, W ? ld_host(s_col[NCOL - 1] + i) : 1.0, sink, acc, smem);
                }
            }
            __syncthreads();                  // every load of this CTA's share has returned
            if (threadIdx.x == 0) bulk_arrive(ctl, dev, p, seq, n);
        }
        if (s_end < 0) return;
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
    if (threadIdx.x == 0) bulk_arrive(ctl, dev, p, s_end, 0);
}

}  // namespace bh
