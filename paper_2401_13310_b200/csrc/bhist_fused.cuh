// bhist_fused.cuh — one-pass fill of several histograms from shared columns (bh_fill_multi).
//
// The paper's future work "compute multiple histograms using data in different (parts of
// the) columns" in one pass; RDataFrame runs every action of a dataframe in
// one event loop.  Each histogram runs the same three steps as k_fill
// (PAPER.md:126): FindBin per axis, bin += w with sum w^2, the GetStats sums.
//
// The kernel is a template over the histogram set, instantiated at run time with NVRTC
// (bhist_jit.cu) for the exact set a bh_fill_multi call names, so every histogram's shape
// (dimension, weights, axis kinds, sink, columns) is a compile-time constant and its
// statistics live in registers.  Histograms whose private state does not fit one SM's
// shared memory together are split over the CTAs of a thread-block CLUSTER ("roles"):
// the R CTAs of a cluster walk the same event tiles, each role reading the columns its
// histograms need; a column several roles read is fetched from DRAM once and served to
// the other roles from L2, kept there by a cluster barrier every few tiles (the roles stay
// within sync_tiles tiles of each other, so the re-read lines are still resident).
#pragma once
#include "bhist_kernels.cuh"

#ifndef BH_FUSED_THREADS
#define BH_FUSED_THREADS 512
#endif
#ifndef BH_FUSED_EPT
#define BH_FUSED_EPT 2       // events per thread per tile (loads in flight before processing)
#endif

namespace bh {

constexpr int kFusedMaxHist = 8;
constexpr int kFusedMaxCols = 8;

struct FusedH {
    AxisP ax[kMaxDim];            // tab_off: byte offset of the staged tables (VM 1 / 3 axes)
    int32_t st1, st2, G, K;
    int32_t smem_off;             // PRIV sinks: byte offset of the private bins
    unsigned long long *count;    // unit-weight counts [G]
    double *sw;                   // weighted (sum w, sum w^2) pairs [2G]
    double *stats, *partials;     // running stats [K]; per-cluster partials [nclusters * K]
    unsigned long long *entries;
    unsigned int *counter;        // last-CTA ticket of this histogram
};

struct FusedP {
    int64_t n;
    const double *cols[kFusedMaxCols];
    const double *w;
    int32_t nclusters;            // clusters in the grid (= CTAs per role)
    int32_t sync_tiles;           // cluster barrier every sync_tiles tiles
    FusedH h[kFusedMaxHist];
};

// Sinks: block-private bins in shared memory (plain: one ATOMS / 128-bit CAS per event;
// AGG: lanes of a warp on the same bin first combine, one update per distinct bin -- the
// hot bins of small histograms; ADAPT (weighted): plain CAS while a warp's adds do not
// collide, aggregated adds after a collision-heavy add, as PrivSink's SINK_PRIVA), or
// warp-aggregated atomics straight into the L2-resident global bins (bin spaces too large
// for shared memory).
enum FusedSink { FS_PRIV = 0, FS_PRIV_AGG = 1, FS_GLOBAL_AGG = 2, FS_PRIV_ADAPT = 3 };

// An axis' scalars as compile-time constants (C++20 floating-point template arguments):
// the kernel is compiled for these exact axes, so FindBin runs on literals instead of
// parameter loads; the device pointers (edges, tables) stay run-time parameters.
struct AxNone {};
template <int A, class T0, class T1, class T2> struct PickAx { using type = T0; };
template <class T0, class T1, class T2> struct PickAx<1, T0, T1, T2> { using type = T1; };
template <class T0, class T1, class T2> struct PickAx<2, T0, T1, T2> { using type = T2; };
template <int N, double XMIN, double XMAX, double D, double INV, int GCELLS, double GSCALE, int G16, int TABOFF>
struct AxC {};
__device__ __forceinline__ AxisP ax_const(const AxisP &rt, AxNone *) { return rt; }
template <int N, double XMIN, double XMAX, double D, double INV, int GCELLS, double GSCALE, int G16, int TABOFF>
__device__ __forceinline__ AxisP ax_const(const AxisP &rt, AxC<N, XMIN, XMAX, D, INV, GCELLS, GSCALE, G16, TABOFF> *) {
    AxisP a;
    a.n = N;
    a.var = rt.var;
    a.xmin = XMIN;
    a.xmax = XMAX;
    a.D = D;
    a.inv = INV;
    a.e = rt.e;
    a.guide = rt.guide;
    a.gcells = GCELLS;
    a.gscale = GSCALE;
    a.e32 = rt.e32;
    a.tab_off = TABOFF;
    a.g16 = G16;
    a.tab_img = rt.tab_img;
    a.tab_bytes = rt.tab_bytes;
    a.lg = rt.lg;
    a.kb = rt.kb;
    return a;
}

// One histogram.  VMa per axis: 0 fixed, 1 variable with tables staged in shared memory
// (guide mode at run time), 2 variable searched in global memory, 3 variable compact.
// AXa: the axis' constants (AxC) or AxNone (read from the parameters).
template <int ID_, int DIM_, bool W_, int SINK_, int C0, int C1, int C2, int VM0, int VM1, int VM2,
          class AX0 = AxNone, class AX1 = AxNone, class AX2 = AxNone>
struct HS {
    template <int A> using Ax = typename PickAx<A, AX0, AX1, AX2>::type;
    static_assert(ID_ >= 0 && ID_ < 8 && DIM_ >= 1 && DIM_ <= 3 && SINK_ >= 0 && SINK_ <= 3, "bad histogram spec");
    static_assert(C0 >= 0 && C0 < 8 && C1 >= 0 && C1 < 8 && C2 >= 0 && C2 < 8, "column index out of range");
    static_assert(VM0 >= 0 && VM0 <= 3 && VM1 >= 0 && VM1 <= 3 && VM2 >= 0 && VM2 <= 3, "bad axis mode");
    static_assert(SINK_ != 3 || W_, "the adaptive sink is for weighted histograms");
    static constexpr int ID = ID_, DIM = DIM_, SINK = SINK_;
    static constexpr bool W = W_;
    static constexpr int K = NStats<DIM_>::K;
    static constexpr unsigned colmask = (1u << C0) | (DIM_ > 1 ? 1u << C1 : 0u) | (DIM_ > 2 ? 1u << C2 : 0u);
    static constexpr int col[3] = {C0, C1, C2};
    static constexpr int vm[3] = {VM0, VM1, VM2};
};

// A warp group: histograms that the same warps fill (their stats live in those threads'
// registers).  A role (one CTA of the cluster) splits its warps evenly over 1-2 groups,
// which walk the same event tiles; the role's shared memory holds every group's bins.
template <class... Hs>
struct Grp {};
// SHARED: columns other roles or groups read too (default L2 policy; the others stream
// with evict-first).
template <unsigned SHARED, class... Gs>
struct Role {};

template <int VM>
__device__ __forceinline__ int fused_find_bin(const AxisP &a, double x, const unsigned char *smem) {
    if (VM == 0) return find_bin_fixed(a, x);
    if (VM == 3) return find_bin_var_compact(a, x, smem + a.tab_off);
    if (VM == 1) return find_bin_var_smem_any(a, x, smem + a.tab_off);
    return find_bin_var_global(a, x);
}

// registers: one Acc (+ the adaptive sink's warp flag) per histogram of the group
template <class... Hs> struct AccT;
template <> struct AccT<> {
    __device__ __forceinline__ void zero() {}
};
template <class H, class... Rest> struct AccT<H, Rest...> {
    Acc<H::DIM, H::W> a;
    bool agg;
    AccT<Rest...> rest;
    __device__ __forceinline__ void zero() { a.zero(); agg = false; rest.zero(); }
};

// warp-aggregated add: lanes of `act` holding the same bin g combine (count by popc, sums
// of w and w*w by a shuffle walk over the peer mask); the group leader gets the totals
template <bool W>
__device__ __forceinline__ bool agg_group(unsigned act, unsigned peers, double w, double &s1, double &s2,
                                          unsigned &cnt) {
    const int lane = (int)(threadIdx.x & 31);
    cnt = (unsigned)__popc(peers);
    if (W) {
        const int rounds = __reduce_max_sync(act, cnt);
        s1 = 0.0;
        s2 = 0.0;
        unsigned m = peers;
        for (int k = 0; k < rounds; ++k) {
            const int src = m ? __ffs(m) - 1 : lane;
            const double v = __shfl_sync(act, w, src);
            if (m) { s1 += v; s2 = fma(v, v, s2); m &= m - 1; }
        }
    }
    return lane == __ffs(peers) - 1;
}

template <class H, class A>
__device__ __forceinline__ void fused_sink(const FusedH &F, int g, double w, bool valid, unsigned char *smem, A &acc) {
    if constexpr (H::SINK == FS_PRIV) {
        if (!valid) return;
        if constexpr (H::W) add2_shared(reinterpret_cast<double2 *>(smem + F.smem_off) + g, w, w * w);
        else asm volatile("red.shared.add.u32 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(smem + F.smem_off) + 4u * (uint32_t)g)
                          : "memory");
    } else if constexpr (H::SINK == FS_PRIV_ADAPT) {
        // plain CAS while adds do not collide; after an add where >= 8 lanes lost their CAS,
        // aggregate (one CAS per distinct cell) while some cell holds >= 4 lanes
        double2 *cell = reinterpret_cast<double2 *>(smem + F.smem_off) + g;
        __syncwarp();
        const unsigned act = __ballot_sync(0xffffffffu, valid);
        const bool agg = __any_sync(0xffffffffu, acc.agg);
        if (agg) {
            const unsigned peers = __match_any_sync(0xffffffffu, valid ? g : -1);
            acc.agg = __any_sync(0xffffffffu, valid && __popc(peers) >= BH_AGG_STAY);
            if (!valid) return;
            double s1, s2;
            unsigned cnt;
            if (agg_group<true>(act, peers, w, s1, s2, cnt)) add2_shared(cell, s1, s2);
        } else {
            const int lost = valid ? add2_shared_count(cell, w, w * w) : 0;
            acc.agg = __popc(__ballot_sync(0xffffffffu, lost > 0)) >= BH_AGG_ENTER;
        }
    } else {
        __syncwarp();
        const unsigned act = __ballot_sync(0xffffffffu, valid);
        if (!valid) return;
        const unsigned peers = __match_any_sync(act, g);
        double s1, s2;
        unsigned cnt;
        const bool lead = agg_group<H::W>(act, peers, w, s1, s2, cnt);
        if constexpr (H::SINK == FS_GLOBAL_AGG && H::W) {    // group sums: paired-lane REDs
            red_sw_pairs(act, __ballot_sync(act, lead), F.sw, g, s1, s2);
            return;
        }
        if (!lead) return;
        if constexpr (H::SINK == FS_PRIV_AGG) {
            if constexpr (H::W) add2_shared(reinterpret_cast<double2 *>(smem + F.smem_off) + g, s1, s2);
            else atomicAdd(reinterpret_cast<uint32_t *>(smem + F.smem_off) + g, cnt);
        } else if constexpr (!H::W) {
            red_u64(F.count + g, (unsigned long long)cnt);
        }
    }
}

template <class... Hs> struct Proc;
template <> struct Proc<> {
    static constexpr int NSTATS = 0;
    template <class X>
    static __device__ __forceinline__ void event(const FusedP &, const X &, double, bool, unsigned char *, AccT<> &) {}
    static __device__ __forceinline__ void init(const FusedP &, unsigned char *) {}
    static __device__ __forceinline__ void flush(const FusedP &, unsigned char *, int, int) {}
    static __device__ __forceinline__ void warp_stats(double *, int, int, AccT<> &) {}
    static __device__ __forceinline__ void partials(const FusedP &, const double *, int, int, int, int, int) {}
    static __device__ __forceinline__ void tickets(const FusedP &, bool *, int, int) {}
    static __device__ __forceinline__ void last_sum(const FusedP &, const bool *, int, int, int, int) {}
};

template <class H, class... Rest> struct Proc<H, Rest...> {
    static constexpr int NSTATS = H::K + Proc<Rest...>::NSTATS;      // this group's stats from H on
    // FindBin on axis A (step (1), per axis) and its term of the global bin
    template <int A, class X>
    static __device__ __forceinline__ void axis_step(const FusedH &F, const X &x, double (&xa)[H::DIM], int &g,
                                                     bool &inr, const unsigned char *smem) {
        xa[A] = x[H::col[A]];
        const AxisP ax = ax_const(F.ax[A], static_cast<typename H::template Ax<A> *>(nullptr));
        const int b = fused_find_bin<H::vm[A]>(ax, xa[A], smem);
        inr &= (b >= 1) & (b <= ax.n);
        g += A == 0 ? b : b * (A == 1 ? F.st1 : F.st2);
    }
    // steps (1)-(3) of PAPER.md:126 for histogram H on one event (x: the group's columns)
    template <class X>
    static __device__ __forceinline__ void event(const FusedP &p, const X &x, double w, bool valid, unsigned char *smem,
                                                 AccT<H, Rest...> &acc) {
        const FusedH &F = p.h[H::ID];
        double xa[H::DIM];
        int g = 0;
        bool inr = true;
        axis_step<0>(F, x, xa, g, inr, smem);
        if constexpr (H::DIM > 1) axis_step<1>(F, x, xa, g, inr, smem);
        if constexpr (H::DIM > 2) axis_step<2>(F, x, xa, g, inr, smem);
        const double wv = H::W ? w : 1.0;
        fused_sink<H>(F, g, wv, valid, smem, acc);
        if (valid && inr) acc.a.add(xa, wv);
        Proc<Rest...>::event(p, x, w, valid, smem, acc.rest);
    }
    // zero the private bins, stage the variable-axis tables (every thread of the CTA)
    static __device__ __forceinline__ void init(const FusedP &p, unsigned char *smem) {
        const FusedH &F = p.h[H::ID];
        if constexpr (H::SINK != FS_GLOBAL_AGG) {
            if constexpr (H::W) {
                double2 *d = reinterpret_cast<double2 *>(smem + F.smem_off);
                for (int i = threadIdx.x; i < F.G; i += blockDim.x) d[i] = make_double2(0.0, 0.0);
            } else {
                uint32_t *c = reinterpret_cast<uint32_t *>(smem + F.smem_off);
                for (int i = threadIdx.x; i < F.G; i += blockDim.x) c[i] = 0u;
            }
        }
        if constexpr (H::vm[0] == 1 || H::vm[0] == 3) stage_axes<1>(&F.ax[0], smem);
        if constexpr (H::DIM > 1 && (H::vm[1] == 1 || H::vm[1] == 3)) stage_axes<1>(&F.ax[1], smem);
        if constexpr (H::DIM > 2 && (H::vm[2] == 1 || H::vm[2] == 3)) stage_axes<1>(&F.ax[2], smem);
        Proc<Rest...>::init(p, smem);
    }
    // merge stage: private bins -> global, once per CTA (group threads)
    static __device__ __forceinline__ void flush(const FusedP &p, unsigned char *smem, int tig, int ntg) {
        const FusedH &F = p.h[H::ID];
        if constexpr (H::SINK != FS_GLOBAL_AGG) {
            if constexpr (H::W) {
                const double *d = reinterpret_cast<const double *>(smem + F.smem_off);
                for (int i = tig; i < 2 * F.G; i += ntg)
                    if (d[i] != 0.0) red_f64(F.sw + i, d[i]);
            } else {
                const uint32_t *c = reinterpret_cast<const uint32_t *>(smem + F.smem_off);
                for (int i = tig; i < F.G; i += ntg)
                    if (c[i]) red_u64(F.count + i, (unsigned long long)c[i]);
            }
        }
        Proc<Rest...>::flush(p, smem, tig, ntg);
    }
    // stats, phase 1: each warp's sums (fixed butterfly) -> red[stat][warp of the group]
    static __device__ __forceinline__ void warp_stats(double *red, int wg, int gw, AccT<H, Rest...> &acc) {
        acc.a.finalize_unit();
#pragma unroll
        for (int k = 0; k < H::K; ++k) {
            const double v = warp_sum_fixed(acc.a.s[k]);
            if ((threadIdx.x & 31) == 0) red[k * gw + wg] = v;
        }
        Proc<Rest...>::warp_stats(red + H::K * gw, wg, gw, acc.rest);
    }
    // phase 2: block sums (warp order) -> this cluster's partials of each histogram
    static __device__ __forceinline__ void partials(const FusedP &p, const double *red, int gw, int tig, int ntg,
                                                    int cid, int off) {
        const FusedH &F = p.h[H::ID];
        for (int k = tig - off; k >= 0 && k < H::K; k += ntg) {
            double t = 0.0;
            for (int i = 0; i < gw; ++i) t += red[k * gw + i];
            F.partials[(size_t)cid * H::K + k] = t;
        }
        Proc<Rest...>::partials(p, red + H::K * gw, gw, tig, ntg, cid, off + H::K);
    }
    // phase 3: one ticket per histogram; the last of the role's CTAs gets the flag
    static __device__ __forceinline__ void tickets(const FusedP &p, bool *last, int tig, int j) {
        if (tig == j) last[j] = atomicAdd(p.h[H::ID].counter, 1u) == (unsigned)p.nclusters - 1;
        Proc<Rest...>::tickets(p, last, tig, j + 1);
    }
    // phase 4: the last CTA sums the partials in cluster order (deterministic for a given
    // grid) into the running stats (include-initial) and adds the events
    static __device__ __forceinline__ void last_sum(const FusedP &p, const bool *last, int wg, int gw, int tig, int j) {
        const FusedH &F = p.h[H::ID];
        if (last[j]) {
            const int lane = threadIdx.x & 31;
            for (int k = wg; k < H::K; k += gw) {
                double t = 0.0;
                for (int b = lane; b < p.nclusters; b += 32) t += __ldcg(F.partials + (size_t)b * H::K + k);
                t = warp_sum_fixed(t);
                if (lane == 0) F.stats[k] += t;
            }
            if (tig == 0) {
                *F.entries += (unsigned long long)p.n;
                *F.counter = 0u;
            }
        }
        Proc<Rest...>::last_sum(p, last, wg, gw, tig, j + 1);
    }
};

// The warp groups of a role run in different branches of run_role, so their block and cluster
// barriers are the non-.aligned forms (barriers reached from different code locations; every
// group executes the same number of them).
__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed;\n\tbarrier.cluster.wait;" ::: "memory");
}
__device__ __forceinline__ void block_sync_any() { asm volatile("barrier.sync 0;" ::: "memory"); }

template <class... Hs> __device__ constexpr unsigned grp_cols(Grp<Hs...> *) { return (0u | ... | Hs::colmask); }
template <class... Hs> __device__ constexpr bool grp_w(Grp<Hs...> *) { return (false || ... || Hs::W); }
template <class... Hs> __device__ constexpr int grp_nstats(Grp<Hs...> *) { return (0 + ... + Hs::K); }
template <class... Hs> __device__ constexpr int grp_nh(Grp<Hs...> *) { return (int)sizeof...(Hs); }
template <class... Hs> __device__ __forceinline__ void grp_init(const FusedP &p, unsigned char *smem, Grp<Hs...> *) {
    Proc<Hs...>::init(p, smem);
}

// One warp group: the event loop over the cluster's tiles, then flush and stats.  Every
// group of every CTA in the cluster executes the same number of block and cluster barriers
// (the loop trip count is the cluster's; finishing uses exactly four block barriers).
// red: this group's scratch (stats x warps doubles, then nh flags), carved from the bins'
// shared memory once they are flushed.
template <unsigned SHARED, class... Hs>
__device__ __forceinline__ void run_group(const FusedP &p, unsigned char *smem, unsigned char *red_base, int gi, int ng,
                                          Grp<Hs...> *) {
    using P = Proc<Hs...>;
    constexpr unsigned kCols = (0u | ... | Hs::colmask);
    constexpr bool kW = (false || ... || Hs::W);
    const int nw = blockDim.x >> 5, gw = nw / ng, wg = (threadIdx.x >> 5) - gi * gw;
    const int ntg = gw * 32, tig = (int)threadIdx.x - gi * ntg;
    AccT<Hs...> acc;
    acc.zero();
    unsigned csize;
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
    const int cid = (int)(blockIdx.x / csize);
    const int64_t tile = (int64_t)ntg * BH_FUSED_EPT;
    const int64_t ntiles = (p.n + tile - 1) / tile;
    // the next tile's columns are loaded before the current tile is processed (register
    // double buffer: the loads' latency overlaps the bin updates).  Event indices advance
    // by the grid stride; the cluster barrier is a countdown (no division in the loop).
    struct Buf {
        double x[BH_FUSED_EPT][kFusedMaxCols];
        double w[BH_FUSED_EPT];
    };
    const int64_t stride = (int64_t)p.nclusters * tile;
    auto load = [&](Buf &b, int64_t i0) {
#pragma unroll
        for (int k = 0; k < BH_FUSED_EPT; ++k) {
            const int64_t i = i0 + k * (int64_t)ntg;
            const bool valid = i < p.n;
#pragma unroll
            for (int c = 0; c < kFusedMaxCols; ++c) {
                b.x[k][c] = 0.0;
                if ((kCols >> c) & 1u)
                    if (valid) b.x[k][c] = ((SHARED >> c) & 1u) ? __ldcg(p.cols[c] + i) : __ldcs(p.cols[c] + i);
            }
            b.w[k] = (kW && valid) ? __ldcg(p.w + i) : 1.0;
        }
    };
    Buf cur, nxt;
    int64_t i0 = (int64_t)cid * tile + tig;
    load(cur, i0);
    int sync_left = p.sync_tiles;
    for (int64_t t = cid; t < ntiles; t += p.nclusters) {
        if (csize > 1 && --sync_left == 0) {
            cluster_sync_relaxed();
            sync_left = p.sync_tiles;
        }
        load(nxt, i0 + stride);
#pragma unroll
        for (int k = 0; k < BH_FUSED_EPT; ++k) P::event(p, cur.x[k], cur.w[k], i0 + k * (int64_t)ntg < p.n, smem, acc);
        cur = nxt;
        i0 += stride;
    }
    block_sync_any();                                     // (1) every group done with the bins
    P::flush(p, smem, tig, ntg);
    block_sync_any();                                     // (2) bins flushed: scratch is free
    double *red = reinterpret_cast<double *>(red_base);
    bool *last = reinterpret_cast<bool *>(red + (size_t)P::NSTATS * gw);
    P::warp_stats(red, wg, gw, acc);
    block_sync_any();                                     // (3)
    P::partials(p, red, gw, tig, ntg, cid, 0);
    __threadfence();
    block_sync_any();                                     // (4)
    P::tickets(p, last, tig, 0);
    block_sync_any();                                     // (5)
    __threadfence();
    P::last_sum(p, last, wg, gw, tig, 0);
}

template <unsigned SHARED, class... Gs>
__device__ __forceinline__ void run_role(const FusedP &p, unsigned char *smem, Role<SHARED, Gs...> *) {
    constexpr int NG = sizeof...(Gs);
    static_assert(NG == 2, "a role has exactly two warp groups (all roles walk the same tiles)");
    (grp_init(p, smem, static_cast<Gs *>(nullptr)), ...);
    __syncthreads();
    const int gw = (int)(blockDim.x >> 5) / NG;
    const int gi = (int)(threadIdx.x >> 5) / gw;
    // per-group scratch for the stats: [stats x warps doubles | nh flags], 16-byte aligned
    size_t off = 0;
    int g = 0;
    ((g++ == gi ? run_group<SHARED>(p, smem, smem + off, gi, NG, static_cast<Gs *>(nullptr))
                : void(),
      off += ((size_t)grp_nstats(static_cast<Gs *>(nullptr)) * gw * 8 + grp_nh(static_cast<Gs *>(nullptr)) + 15) &
             ~size_t(15)),
     ...);
}

template <class... Rs>
__global__ void __launch_bounds__(BH_FUSED_THREADS, 1) k_fused(const __grid_constant__ FusedP p) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned rank;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    unsigned r = 0;
    ((rank == r++ ? run_role(p, smem, static_cast<Rs *>(nullptr)) : void()), ...);
}

}  // namespace bh
