// bhist_sort.cuh — SORT strategy: two-pass partitioned fill for large bin spaces.
//
// The north star's "sort-then-segmented-reduce path for large 2D/3D bin spaces":
// a one-digit radix partition of the global bin index followed by a per-partition
// shared-memory reduction.  A 1M-bin TH2D/TH3D does not fit one SM's shared memory
// (the paper's per-block copy, assumes it does), and adding
// straight into the L2-resident histogram costs one L2 atomic per event (GLOBAL /
// CACHE, ~1e11 events/s).  Here:
//
//   pass 1 (k_part_scatter): the tile's columns arrive in shared memory by TMA bulk
//     copies (two tiles in flight); the three steps of PAPER.md:126 up to the bin index
//     -- FindBin per axis, global bin g, the GetStats sums in registers -- then the
//     event's record (local bin l = g mod 2^pb, and w) is ranked within its partition
//     p = g >> pb by a returning shared-memory atomic, the tile's records are sorted by
//     partition in shared memory (segments padded to RC-record chunks) and written out
//     with coalesced 16-byte stores, plus one row of segment offsets per tile.
//   plan   (k_part_plan): per-partition record totals -> prefix -> pass-2 balance.
//   pass 2 (k_part_reduce): each CTA owns a contiguous stretch of the (partition,
//     tile) order of about equal record count; per batch of tiles every thread walks an
//     equal share of the segments' chunks; the partition's 2^pb bins live in shared
//     memory (u32 counts by `red.shared.add.u32`; double2 (sumw, sumw2) by 128-bit CAS
//     behind a per-thread register cache of a repeating bin), and are added to the
//     global bins once per partition the CTA touched (the merge stage of PAPER.md:162-165).
//   probe  (k_part_probe): AUTO's hotness test on a sample (see bhist.cu auto_sort).
//
// Records cost 2 B (unit) or 10 B (weighted) per event written + read back, instead of
// one L2 atomic per event; no shared-memory state is bigger than 128 KB.
#pragma once
#include <type_traits>

#include "bhist_kernels.cuh"

namespace bh {

constexpr int kPartThreads = 1024;                   // pass 1: 1 CTA per SM (2 x 512 measured no faster)
// events per thread per tile; a staged tile (NCOL columns) is <= 64 KB
__host__ __device__ constexpr int part_ev(int dim, bool w) { return dim + (w ? 1 : 0) >= 3 ? 2 : 4; }
constexpr int kPartMaxP = 2048;                      // partitions (bins / 2^pb) supported
#ifndef BH_REDUCE_CTAS
#define BH_REDUCE_CTAS 1
#endif
constexpr int kReduceCtas = BH_REDUCE_CTAS;          // pass 2 CTAs per SM
constexpr int kReduceThreads = 1024 / kReduceCtas;   // (1 CTA per SM owns 128 KB of bins)

struct PartP {
    const int32_t *gate;        // AUTO: run only if *gate == 1 (SORT chosen on the device); nullptr: always
    uint16_t *rec_l;            // [ntiles * kPartTile] local bin, tile-major, partition-sorted within a tile
    double *rec_w;              // weighted: the weights, same order
    uint32_t *offs;             // [ntiles * (P + 1)] segment starts of each tile
    unsigned long long *cnt;    // [P] records per partition (pass 1 adds; plan reads and zeroes)
    unsigned long long *cp;     // [P + 1] exclusive prefix of cnt (plan writes)
    int32_t P, pb, ntiles;
    int32_t tile;               // events per tile (kPartThreads * part_ev)
    int32_t ts;                 // scratch slots per tile (>= tile + P*(RC-1), multiple of 8)
};

// ------------------------------------------------------------------ pass 1
// Segments are padded to RC records with the sentinel 0xffff (never a local bin: pb <= 15)
// so that pass 2 reads them in aligned RC-record chunks; a tile's records occupy
// q.ts >= tile + P*(RC-1) slots of the scratch.
constexpr uint16_t kPartPad = 0xffffu;
#ifndef BH_PART_STAGES
#define BH_PART_STAGES 2
#endif
constexpr int kPartStages = BH_PART_STAGES;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar` (UBLKCP.S.G)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Pass 1.  One CTA of kPartThreads per SM; each tile's columns (and weights) are
// staged in shared memory by TMA bulk copies, kPartStages tiles in flight, so HBM
// streams while the CTA bins, ranks and scatters the previous tile.  Tiles that are
// partial or whose columns are not 16-byte aligned are loaded by the threads instead.
template <int DIM, bool W, int VM, int RC>
__global__ void __launch_bounds__(kPartThreads, 1) k_part_scatter(FillP p, PartP q) {
    if (gated_off(q.gate, gate_bit(1))) return;
    constexpr int NCOL = DIM + (W ? 1 : 0);
    constexpr int kEv = part_ev(DIM, W);
    constexpr int kTile = kPartThreads * kEv;
    constexpr uint32_t kStageBytes = (uint32_t)NCOL * kTile * 8u;
    extern __shared__ __align__(16) unsigned char smem[];
    // layout: [stage 0..S-1: NCOL x f64[tile]] [mbar S x u64] [stage_w f64[ts] (W)] [stage_l u16[ts]]
    //         [cnt u32[P]] [start u32[P+1]] [axis tables (VM 1, at tab_off)]
    const int ts = q.ts;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + kPartStages * kStageBytes);
    unsigned char *rec = smem + kPartStages * kStageBytes + 8 * kPartStages;
    double *stw = reinterpret_cast<double *>(rec);
    uint16_t *stl = reinterpret_cast<uint16_t *>(rec + (W ? 8 * (size_t)ts : 0));
    uint32_t *cnt = reinterpret_cast<uint32_t *>(rec + (W ? 8 * (size_t)ts : 0) + 2 * (size_t)ts);
    uint32_t *start = cnt + q.P;
    const int P = q.P, pb = q.pb;
    const uint32_t lmask = (1u << pb) - 1u;
    const int n = (int)p.n;                          // one launch covers < 2^31 events
    const double *col[NCOL];
#pragma unroll
    for (int a = 0; a < DIM; ++a) col[a] = p.x[a];
    if (W) col[NCOL - 1] = p.w;
    bool aligned = true;
#pragma unroll
    for (int a = 0; a < NCOL; ++a) aligned &= (reinterpret_cast<uintptr_t>(col[a]) & 15) == 0;
    auto tma_ok = [&](int t) { return aligned && t < q.ntiles && (t + 1) * kTile <= n; };
    auto issue = [&](int t, int st) {                // thread 0 only
        double *dst = reinterpret_cast<double *>(smem + st * kStageBytes);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(mbar + st, kStageBytes);
#pragma unroll
        for (int a = 0; a < NCOL; ++a) bulk_g2s(dst + a * kTile, col[a] + (size_t)t * kTile, kTile * 8u, mbar + st);
    };

    if constexpr (VM == 1) stage_axes<DIM>(p.ax, smem);
    for (int i = threadIdx.x; i < P; i += kPartThreads) cnt[i] = 0u;
    if (threadIdx.x == 0) {
        for (int st = 0; st < kPartStages; ++st) mbar_init(mbar + st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < kPartStages; ++st) {
            const int t = blockIdx.x + st * gridDim.x;
            if (tma_ok(t)) issue(t, st);
        }
    }
    __syncthreads();

    Acc<DIM, W> acc;
    acc.zero();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t phase = 0;                              // bit st: parity of stage st's next completion
    int k = 0;
    for (int t = blockIdx.x; t < q.ntiles; t += gridDim.x, ++k) {
        const int st = k % kPartStages;
        const double *sx = reinterpret_cast<const double *>(smem + st * kStageBytes);
        const int e0 = t * kTile;
        const int m = min(kTile, n - e0);
        if (tma_ok(t)) {
            mbar_wait(mbar + st, (phase >> st) & 1u);
            phase ^= 1u << st;
        } else {                                     // partial / unaligned tile: the threads load it
            double *dx = reinterpret_cast<double *>(smem + st * kStageBytes);
            for (int i = threadIdx.x; i < m; i += kPartThreads)
#pragma unroll
                for (int a = 0; a < NCOL; ++a) dx[a * kTile + i] = ld_stream(col[a] + e0 + i);
            __syncthreads();
        }
        // step (1), per axis -> global bin; step (3) stats; rank in partition
        int pp[kEv];
        uint32_t key[kEv];                           // rank << 16 | local bin
        double wk[kEv];                              // the weights again, for the scatter
        auto bin_rank = [&](auto full) {             // full tiles: no per-event bounds checks
#pragma unroll
            for (int u = 0; u < kEv; ++u) {
                const int i = u * kPartThreads + threadIdx.x;
                const bool ok = decltype(full)::value || i < m;
                double x[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) x[a] = sx[a * kTile + i];
                const double w = W ? sx[(NCOL - 1) * kTile + i] : 1.0;
                wk[u] = w;
                int g = 0, mul = 1;
                bool inr = true;
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    const int b = find_bin<VM>(p.ax[a], x[a], smem);
                    inr &= (b >= 1) & (b <= p.ax[a].n);
                    g += b * mul;
                    if (a + 1 < DIM) mul = (a == 0) ? p.st1 : p.st2;
                }
                if (ok && inr) acc.add(x, w);        // in range only (R6)
                pp[u] = ok ? (int)((uint32_t)g >> pb) : -1;
                // the returned old count is the rank (equal addresses of a warp are resolved
                // by the shared-memory atomic unit)
                key[u] = ((uint32_t)g & lmask) | (ok ? atomicAdd(cnt + pp[u], 1u) << 16 : 0u);
            }
        };
        if (m == kTile) bin_rank(std::true_type{});
        else bin_rank(std::false_type{});
        __syncthreads();                             // (A) stage consumed, counts complete
        if (threadIdx.x == 0) {
            const int tn = t + kPartStages * gridDim.x;
            if (tma_ok(tn)) issue(tn, st);           // refill this stage with a later tile
        }
        if (warp == 0) {                             // padded exclusive scan; pads; counts
            uint32_t run = 0;
            uint32_t *orow = q.offs + (size_t)t * (P + 1);
            for (int c0 = 0; c0 < P; c0 += 32) {
                const int i = c0 + lane;
                const uint32_t v = i < P ? cnt[i] : 0u;
                const uint32_t vp = (v + RC - 1) / RC * RC;
                uint32_t inc = vp;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t uu = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += uu;
                }
                if (i < P) {
                    const uint32_t s0 = run + inc - vp;
                    start[i] = s0;
                    orow[i] = s0;
                    cnt[i] = 0u;
                    for (uint32_t j = s0 + v; j < s0 + vp; ++j) {
                        stl[j] = kPartPad;
                        if (W) stw[j] = 0.0;
                    }
                    if (v) atomicAdd(q.cnt + i, (unsigned long long)v);
                }
                run += __shfl_sync(0xffffffffu, inc, 31);
            }
            if (lane == 0) { start[P] = run; orow[P] = run; }
        }
        __syncthreads();                             // (B)
#pragma unroll
        for (int u = 0; u < kEv; ++u) {              // records -> partition-sorted staging
            if (pp[u] >= 0) {
                const uint32_t pos = start[pp[u]] + (key[u] >> 16);
                stl[pos] = (uint16_t)(key[u] & 0xffffu);
                if (W) stw[pos] = wk[u];
            }
        }
        __syncthreads();                             // (C)
        const int tot = (int)start[P];               // padded record count of the tile
        uint4 *ol = reinterpret_cast<uint4 *>(q.rec_l + (size_t)t * ts);
        for (int i = threadIdx.x; i < (tot + 7) / 8; i += kPartThreads) ol[i] = reinterpret_cast<const uint4 *>(stl)[i];
        if (W) {
            uint4 *ow = reinterpret_cast<uint4 *>(q.rec_w + (size_t)t * ts);
            for (int i = threadIdx.x; i < (tot + 1) / 2; i += kPartThreads) ow[i] = reinterpret_cast<const uint4 *>(stw)[i];
        }
        // the next tile rewrites the staging only after its barrier (A), when every
        // thread has finished this copy
    }
    acc.finalize_unit();
    block_stats_finish<Acc<DIM, W>::K>(p, acc.s);
}

#ifndef BH_FILL_TU
// ------------------------------------------------------------------ hotness probe (AUTO)
// One CTA bins a sample of a fill's events (probe_load; global-memory FindBin) and
// writes the largest partition's count: AUTO uses SORT for later large unit-weight fills
// only when no partition is hot (a hot partition serializes pass 1's rank atomics).
constexpr int kProbeHash = 4096;
constexpr int kProbeMarg = 4096;                  // window: bins per axis (flow included) the probe histograms

// The probes' sample: kProbeRuns runs of consecutive events spread evenly over the fill
// (sample k = event (k / run) * (n / kProbeRuns) + k % run): a warp reads 32 consecutive
// events per column, not 32 scattered 32-byte sectors; a batch of kProbeBatch samples per
// thread is loaded before any is binned.  (Strided single events cost ~70 us per probe.)
constexpr int kProbeBatch = 4;
constexpr int kProbeRuns = 64;
template <int DIM>
__device__ __forceinline__ void probe_load(const FillP &p, int k0, int samples, double (&xv)[kProbeBatch][DIM]) {
    const int run = samples / kProbeRuns;
    const int64_t gap = p.n / kProbeRuns;
#pragma unroll
    for (int j = 0; j < kProbeBatch; ++j) {
        const int k = k0 + j * (int)blockDim.x;
        const int64_t e = (int64_t)(k / run) * gap + (k % run);
#pragma unroll
        for (int a = 0; a < DIM; ++a) xv[j][a] = k < samples ? __ldg(p.x[a] + e) : 0.0;
    }
}

// Block-wide: shortest run of consecutive bins holding >= T samples, from the inclusive-
// exclusive prefix sums ps[0..n] (ps[0] = 0): each thread takes starts l, finds the first end
// r with ps[r] - ps[l] >= T by binary search, and the block keeps the minimum (len, l).
// Returns (len << 16) | lo, or 0xffffffff when no run holds T.  All threads call it.
__device__ inline unsigned int shortest_cover(const unsigned int *ps, int n, unsigned int T, unsigned int *red) {
    if (threadIdx.x == 0) *red = 0xffffffffu;
    __syncthreads();
    unsigned int bestv = 0xffffffffu;
    for (int l = threadIdx.x; l < n; l += blockDim.x) {
        const unsigned int need = ps[l] + T;
        if (ps[n] < need) continue;
        int lo = l + 1, hi = n;                      // first r in [l+1, n] with ps[r] >= need
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ps[mid] >= need) hi = mid; else lo = mid + 1;
        }
        bestv = min(bestv, ((unsigned int)(lo - l) << 16) | (unsigned int)l);
    }
    bestv = __reduce_min_sync(0xffffffffu, bestv);
    if ((threadIdx.x & 31) == 0) atomicMin(red, bestv);
    __syncthreads();
    const unsigned int v = *red;
    __syncthreads();
    return v;
}

// in-place exclusive prefix sums of m[0..n) into ps[0..n] (warp 0; n <= kProbeMarg)
__device__ inline void prefix_sums(const unsigned int *m, int n, unsigned int *ps) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x, per = (n + 31) / 32, b = lane * per;
        unsigned int loc = 0;
        for (int i = b; i < min(n, b + per); ++i) loc += m[i];
        unsigned int inc = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        unsigned int run = inc - loc;
        for (int i = b; i < min(n, b + per); ++i) { ps[i] = run; run += m[i]; }
        if (lane == 31) ps[n] = inc;
    }
    __syncthreads();
}

template <int DIM>
__global__ void __launch_bounds__(1024, 1) k_part_probe(FillP p, int pb, int P, int samples, int amax, unsigned int *out) {
    // out[0]: largest partition count; out[1]: largest count of a hashed bin bucket
    // (4096 buckets: a single hot bin shows up as one large bucket); out[2]: the unit-weight
    // decision, 2 (WINDOW) when a box of <= amax bins (per-axis shortest intervals holding
    // the same share q of the sample's marginals, the largest q that fits) holds >= 50% of
    // the samples, else 1 (SORT) when no partition holds > 5% and no bucket > 1% of the
    // samples, else 0 (CACHE); out[3]: the weighted decision, 1 (GLOBAL) when no bucket holds
    // > 1/512 of the samples (a bin with a share f of n events costs f*n serialized
    // same-address REDs, ~0.55 G/s), else 0 (CACHE); out[4..7]: the box (x0, wx, y0, wy) --
    // read by the gated fills on the device, so AUTO's choice depends on the data only, never
    // on timing.  Window: DIM <= 2, axes of <= kProbeMarg bins each (flow included).
    extern __shared__ unsigned int pc[];
    unsigned int *hc = pc + P;
    unsigned int *m0 = hc + kProbeHash, *m1 = m0 + kProbeMarg;
    unsigned int *ps0 = m1 + kProbeMarg, *ps1 = ps0 + kProbeMarg + 1;    // prefix sums [n + 1]
    int *gs = reinterpret_cast<int *>(ps1 + kProbeMarg + 1);     // [samples] axis bins, packed
    __shared__ unsigned int red;
    __shared__ int box[4];
    __shared__ unsigned int inbox;
    const int n0 = p.ax[0].n + 2, n1 = DIM >= 2 ? p.ax[1].n + 2 : 1;
    const bool win = DIM <= 2 && amax > 0 && n0 <= kProbeMarg && n1 <= kProbeMarg;
    for (int i = threadIdx.x; i < P + kProbeHash + 2 * kProbeMarg; i += blockDim.x) pc[i] = 0u;
    if (threadIdx.x == 0) inbox = 0u;
    __syncthreads();
    double xv[kProbeBatch][DIM];
    for (int base = 0; base < samples; base += kProbeBatch * (int)blockDim.x) {     // warp-uniform trips
      const int k0 = base + (int)threadIdx.x;
      probe_load<DIM>(p, k0, samples, xv);       // the batch's (random) loads first
#pragma unroll
      for (int j = 0; j < kProbeBatch; ++j) {
        const int k = k0 + j * (int)blockDim.x;
        const bool ok = k < samples;
        int g = 0, mul = 1, bb[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            bb[a] = find_bin(p.ax[a], xv[j][a]);
            g += bb[a] * mul;
            if (a + 1 < DIM) mul = (a == 0) ? p.st1 : p.st2;
        }
        if (!ok) continue;
        atomicAdd(pc + ((uint32_t)g >> pb), 1u);
        atomicAdd(hc + (((uint32_t)g * 2654435761u) >> 20), 1u);
        if (win) {
            atomicAdd(m0 + bb[0], 1u);
            if (DIM >= 2) atomicAdd(m1 + bb[DIM >= 2 ? 1 : 0], 1u);
            gs[k] = bb[0] | (DIM >= 2 ? bb[DIM >= 2 ? 1 : 0] << 16 : 0);
        }
      }
    }
    __syncthreads();
    unsigned int m = 0, mh = 0;
    for (int i = threadIdx.x; i < P; i += blockDim.x) m = max(m, pc[i]);
    for (int i = threadIdx.x; i < kProbeHash; i += blockDim.x) mh = max(mh, hc[i]);
    m = __reduce_max_sync(0xffffffffu, m);
    mh = __reduce_max_sync(0xffffffffu, mh);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, m);
        atomicMax(out + 1, mh);
    }
    // the box: bisection on the sample share q (the largest q whose per-axis shortest
    // intervals fit amax bins), each interval found block-parallel on prefix sums
    if (threadIdx.x == 0) { box[0] = 0; box[1] = 0; box[2] = 0; box[3] = 0; }
    if (win) {
        prefix_sums(m0, n0, ps0);
        if (DIM >= 2) prefix_sums(m1, n1, ps1);
        unsigned int qlo = 0, qhi = (unsigned int)samples + 1;        // qlo fits, qhi does not
        unsigned int b0 = 0, b1 = 1u << 16;
        while (qhi - qlo > 1u + (unsigned int)samples / 1024) {
            const unsigned int q = (qlo + qhi) / 2;
            const unsigned int c0 = shortest_cover(ps0, n0, q, &red);
            const unsigned int c1 = DIM >= 2 ? shortest_cover(ps1, n1, q, &red) : (1u << 16);
            if (c0 != 0xffffffffu && c1 != 0xffffffffu && (int64_t)(c0 >> 16) * (c1 >> 16) <= amax) {
                qlo = q; b0 = c0; b1 = c1;
            } else {
                qhi = q;
            }
        }
        if (threadIdx.x == 0 && qlo > 0) {
            box[0] = (int)(b0 & 0xffffu); box[1] = (int)(b0 >> 16);
            box[2] = (int)(b1 & 0xffffu); box[3] = (int)(b1 >> 16);
        }
    }
    __syncthreads();
    if (win && box[1] > 0) {
        unsigned int c = 0;
        for (int k = threadIdx.x; k < samples; k += blockDim.x) {
            const int b0 = gs[k] & 0xffff, b1 = gs[k] >> 16;
            c += (unsigned)(b0 - box[0]) < (unsigned)box[1] && (unsigned)(b1 - box[2]) < (unsigned)box[3];
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if ((threadIdx.x & 31) == 0) atomicAdd(&inbox, c);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long S = (unsigned long long)samples;
        out[2] = 2ull * inbox >= S && box[1] > 0 ? 2u : (20ull * out[0] <= S && 100ull * out[1] <= S) ? 1u : 0u;
        out[3] = 512ull * out[1] <= S ? 1u : 0u;
        for (int i = 0; i < 4; ++i) out[4 + i] = (unsigned int)box[i];
    }
}

// ------------------------------------------------------------------ hot-cell probe (AUTO, weighted PRIVA)
// One CTA counts the global bins of a sample (probe_load) in a shared-memory hash table,
// picks up to kHotW cells holding >= 1/64 of the sample each (hottest first), maps them
// into the direct-mapped slot table (a colliding colder cell is dropped), and sets flag = 2
// when the mapped cells hold >= 20% of the sample (then the lane-private window pays for the
// shared memory it takes from the replicas / slots); flag = 1 passes on k_part_probe's GLOBAL
// decision (weighted CACHE fills).  Deterministic: a fixed sample, fixed tie-breaks.
constexpr int kHotHash = 4096;
template <int DIM>
__global__ void __launch_bounds__(1024, 1) k_hot_probe(FillP p, int samples, const unsigned int *gdec, HotTab *out) {
    __shared__ int32_t key[kHotHash];
    __shared__ uint32_t cnt[kHotHash];
    __shared__ int32_t pick[kHotW];
    __shared__ uint32_t pickc[kHotW];
    for (int i = threadIdx.x; i < kHotHash; i += blockDim.x) { key[i] = -1; cnt[i] = 0u; }
    __syncthreads();
    double xv[kProbeBatch][DIM];
    for (int base = 0; base < samples; base += kProbeBatch * (int)blockDim.x) {     // warp-uniform trips
      const int k0 = base + (int)threadIdx.x;
      probe_load<DIM>(p, k0, samples, xv);
#pragma unroll
      for (int j = 0; j < kProbeBatch; ++j) {
        const bool ok = k0 + j * (int)blockDim.x < samples;
        int g = 0, mul = 1;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            g += find_bin(p.ax[a], xv[j][a]) * mul;
            if (a + 1 < DIM) mul = (a == 0) ? p.st1 : p.st2;
        }
        // equal cells of the warp first (hot cells would serialize the table's atomics)
        const unsigned m = __match_any_sync(0xffffffffu, ok ? g : -1 - (int)(threadIdx.x & 31));
        if (!ok || (int)(threadIdx.x & 31) != __ffs(m) - 1) continue;
        int hs = (int)(((uint32_t)g * 2654435761u) >> 20);
        for (int t = 0; t < 8; ++t, hs = (hs + 1) & (kHotHash - 1)) {       // a sparse cell may be dropped
            const int old = atomicCAS(key + hs, -1, g);
            if (old == -1 || old == g) { atomicAdd(cnt + hs, (unsigned)__popc(m)); break; }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {                                   // warp 0: the hottest cells, in order
        const int lane = threadIdx.x;
        for (int r = 0; r < kHotW; ++r) {
            uint32_t best = 0;
            int bi = kHotHash;
            for (int i = lane; i < kHotHash; i += 32)
                if (cnt[i] > best) { best = cnt[i]; bi = i; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            const bool ok = 64ull * best >= (unsigned long long)samples && bi < kHotHash;
            if (lane == 0) {
                pick[r] = ok ? key[bi] : -1;
                pickc[r] = ok ? best : 0u;
                if (ok) cnt[bi] = 0u;
            }
            __syncwarp();
        }
        if (lane == 0) {
            for (int i = 0; i < kHotSlots; ++i) out->tab[i] = make_int2(-1, 0);
            unsigned long long covered = 0;
            int nwin = 0;
            for (int r = 0; r < kHotW; ++r) {
                out->cell[r] = -1;
                if (pick[r] < 0) continue;
                int2 &slot = out->tab[hot_slot(pick[r])];
                if (slot.x != -1) continue;                   // collides with a hotter cell
                slot = make_int2(pick[r], r);
                out->cell[r] = pick[r];
                covered += pickc[r];
                nwin = r + 1;
            }
            out->nwin = nwin;
            // the gate word of the weighted fill: 1 GLOBAL (k_part_probe's decision, when given),
            // else 2 (window kernel) or 0 (plain sink)
            out->flag = gdec && __ldcg(gdec) == 1u ? 1 : 5ull * covered >= (unsigned long long)samples ? 2 : 0;
        }
    }
}

// ------------------------------------------------------------------ plan
// One warp: cp = exclusive prefix of cnt (records per partition); cnt is zeroed for
// the next chunk.
__global__ void k_part_plan(PartP q) {
    if (gated_off(q.gate, gate_bit(1))) return;
    const int lane = threadIdx.x;
    unsigned long long run = 0;
    for (int c0 = 0; c0 < q.P; c0 += 32) {
        const int i = c0 + lane;
        const unsigned long long v = i < q.P ? q.cnt[i] : 0ull;
        unsigned long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (i < q.P) { q.cp[i] = run + inc - v; q.cnt[i] = 0ull; }
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) q.cp[q.P] = run;
}

#endif  // BH_FILL_TU

// ------------------------------------------------------------------ pass 2
// Position X in [0, R] of the virtual record order (partition-major, then tile) ->
// (partition, tile), assuming a partition's records spread evenly over the tiles.
// Monotone in X, so consecutive CTAs cover every (partition, tile) pair exactly once.
__device__ __forceinline__ void part_pos(const PartP &q, unsigned long long X, int &pp, int &tt) {
    const unsigned long long R = q.cp[q.P];
    if (X >= R) { pp = q.P; tt = 0; return; }
    int lo = 0, hi = q.P - 1;                        // last partition with cp[p] <= X
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (q.cp[mid] <= X) lo = mid; else hi = mid - 1;
    }
    const unsigned long long c = q.cp[lo + 1] - q.cp[lo];   // > 0, since cp[lo] <= X < cp[lo+1]
    pp = lo;
    tt = (int)(((X - q.cp[lo]) * (unsigned long long)q.ntiles) / c);
}

// Weighted pass 2: a per-thread sticky one-entry cache in front of the shared-memory
// bins.  A thread adds records of its cached bin in registers; once the cached bin has
// repeated, other bins go straight to the 128-bit CAS, so a hot bin stays in registers
// instead of serializing the CTA's warps on one shared-memory cell.
struct LaneCache {
    uint32_t l = kPartPad, n = 0;
    double s1 = 0.0, s2 = 0.0;
    __device__ __forceinline__ void add(unsigned char *bins, uint32_t rl, double w) {
        if (rl == l) {
            ++n;
            s1 += w;
            s2 = fma(w, w, s2);
        } else if (n >= 2) {
            add2_shared(reinterpret_cast<double2 *>(bins) + rl, w, w * w);
        } else {
            if (n) add2_shared(reinterpret_cast<double2 *>(bins) + l, s1, s2);
            l = rl;
            n = 1;
            s1 = w;
            s2 = w * w;
        }
    }
    __device__ __forceinline__ void flush(unsigned char *bins) {
        if (n) add2_shared(reinterpret_cast<double2 *>(bins) + l, s1, s2);
        l = kPartPad;
        n = 0;
    }
};

constexpr int kReduceBatch = 2048;                   // tiles whose segments are balanced at once

// Pass 2.  The CTA's stretch of (partition, tile) pairs is processed in batches of
// tiles: the segments' chunk counts are prefix-summed in shared memory and every thread
// takes an equal contiguous range of chunks (so one hot partition with long segments
// still keeps all 32 warps busy), walking the segments in order.
template <bool W, int RC>
__global__ void __launch_bounds__(kReduceThreads, kReduceCtas) k_part_reduce(FillP p, PartP q) {
    if (gated_off(q.gate, gate_bit(1))) return;
    extern __shared__ __align__(16) unsigned char smem[];
    // layout: [bins (2^pb cells)] [o0 u32[batch]] [cp u32[batch+1]] [scan scratch u32[32]]
    const size_t binbytes = (size_t)(W ? 16 : 4) << q.pb;
    uint32_t *so0 = reinterpret_cast<uint32_t *>(smem + binbytes);
    uint32_t *scp = so0 + kReduceBatch;
    uint32_t *wsum = scp + kReduceBatch + 1;
    const int C = gridDim.x;
    const unsigned long long R = q.cp[q.P];
    if (R == 0) return;
    int pa, ta, pz, tz;
    part_pos(q, R * blockIdx.x / C, pa, ta);
    part_pos(q, R * (blockIdx.x + 1) / C, pz, tz);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int P = q.P, nb_full = 1 << q.pb;
    LaneCache lc;                                    // weighted: hot bins accumulate in registers
    for (int part = pa; part <= pz && part < P; ++part) {
        const int t0 = part == pa ? ta : 0;
        const int t1 = part == pz ? tz : q.ntiles;
        if (t0 >= t1 || q.cp[part + 1] == q.cp[part]) continue;     // uniform
        const int gb0 = part << q.pb;
        const int nb = min(nb_full, p.G - gb0);
        if (W) {
            double2 *d = reinterpret_cast<double2 *>(smem);
            for (int i = threadIdx.x; i < nb; i += kReduceThreads) d[i] = make_double2(0.0, 0.0);
        } else {
            uint32_t *c = reinterpret_cast<uint32_t *>(smem);
            for (int i = threadIdx.x; i < nb; i += kReduceThreads) c[i] = 0u;
        }
        for (int tb0 = t0; tb0 < t1; tb0 += kReduceBatch) {
            const int nt = min(kReduceBatch, t1 - tb0);
            __syncthreads();                         // every thread is done with the previous batch
            // chunk counts of the batch's segments -> block-wide exclusive scan
            constexpr int PER = kReduceBatch / kReduceThreads;
            uint32_t v[PER], tsum = 0;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int i = threadIdx.x * PER + j;
                v[j] = 0;
                if (i < nt) {
                    const uint32_t *row = q.offs + (size_t)(tb0 + i) * (P + 1) + part;
                    const uint32_t o0 = __ldg(row);
                    so0[i] = o0;
                    v[j] = (__ldg(row + 1) - o0) / RC;
                }
                tsum += v[j];
            }
            uint32_t inc = tsum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += u;
            }
            if (lane == 31) wsum[warp] = inc;
            __syncthreads();
            if (warp == 0) {
                uint32_t x = wsum[lane], xi = x;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xffffffffu, xi, o);
                    if (lane >= o) xi += u;
                }
                wsum[lane] = xi - x;                 // exclusive warp offsets
            }
            __syncthreads();
            uint32_t run = wsum[warp] + inc - tsum;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int i = threadIdx.x * PER + j;
                if (i <= nt) scp[i] = run;           // scp[nt] = total
                run += v[j];
            }
            if (threadIdx.x == kReduceThreads - 1 && nt == kReduceBatch) scp[nt] = run;
            __syncthreads();
            const uint32_t CT = scp[nt];
            uint32_t c = (uint32_t)((unsigned long long)CT * threadIdx.x / kReduceThreads);
            const uint32_t cend = (uint32_t)((unsigned long long)CT * (threadIdx.x + 1) / kReduceThreads);
            // tile of chunk c: last j with scp[j] <= c
            int lo = 0, hi = nt - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (scp[mid] <= c) lo = mid; else hi = mid - 1;
            }
            int j = lo;
            constexpr int U = W ? 2 : 4;
            while (c < cend) {
                uint16_t l[U][RC];
                double w[U][RC];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool ok = c + u < cend;
                    size_t at = 0;
                    if (ok) {
                        while (c + u >= scp[j + 1]) ++j;
                        at = (size_t)(tb0 + j) * q.ts + so0[j] + (size_t)(c + u - scp[j]) * RC;
                    }
                    if (RC == 8) {
                        uint4 vv = make_uint4(~0u, ~0u, ~0u, ~0u);
                        if (ok) vv = __ldg(reinterpret_cast<const uint4 *>(q.rec_l + at));
                        const uint32_t uu[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                        for (int k = 0; k < RC && k < 8; ++k) l[u][k] = (uint16_t)(uu[k >> 1] >> (16 * (k & 1)));
                    } else if (RC == 4) {
                        uint2 vv = make_uint2(~0u, ~0u);
                        if (ok) vv = __ldg(reinterpret_cast<const uint2 *>(q.rec_l + at));
                        const uint32_t uu[2] = {vv.x, vv.y};
#pragma unroll
                        for (int k = 0; k < RC && k < 4; ++k) l[u][k] = (uint16_t)(uu[k >> 1] >> (16 * (k & 1)));
                    } else {
#pragma unroll
                        for (int k = 0; k < RC; ++k) l[u][k] = ok ? __ldg(q.rec_l + at + k) : kPartPad;
                    }
                    if (W) {
                        if (RC % 2 == 0) {
#pragma unroll
                            for (int k = 0; k < RC; k += 2) {
                                double2 vv = make_double2(0.0, 0.0);
                                if (ok) vv = __ldg(reinterpret_cast<const double2 *>(q.rec_w + at + k));
                                w[u][k] = vv.x;
                                w[u][k + 1 < RC ? k + 1 : k] = vv.y;
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < RC; ++k) w[u][k] = ok ? __ldg(q.rec_w + at + k) : 0.0;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int k = 0; k < RC; ++k)
                        if (l[u][k] != kPartPad) {
                            if (W) lc.add(smem, l[u][k], w[u][k]);
                            else asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(smem_u32(smem) + 4u * l[u][k]) : "memory");
                        }
                c += U;
            }
        }
        if (W) lc.flush(smem);
        __syncthreads();
        // merge stage: this CTA's partial bins of the partition -> global
        if (W) {
            const double *d = reinterpret_cast<const double *>(smem);
            double *o = p.sw + 2 * (size_t)gb0;
            for (int i = threadIdx.x; i < 2 * nb; i += kReduceThreads)
                if (d[i] != 0.0) red_f64(o + i, d[i]);
        } else {
            const uint32_t *cc = reinterpret_cast<const uint32_t *>(smem);
            for (int i = threadIdx.x; i < nb; i += kReduceThreads)
                if (cc[i]) red_u64(p.count + gb0 + i, (unsigned long long)cc[i]);
        }
        __syncthreads();
    }
}

}  // namespace bh
