// bhist_kernels.cuh — sm_100a device code for bulk histogram filling.
//
// One fused kernel per fill: it streams the coordinate (and weight) columns
// once, runs FindBin per axis, composes the global bin, adds into the bins and
// accumulates the GetStats sums in registers — the three steps of PAPER.md:126
// in a single pass (the paper's CUDA path used one histogram kernel plus one
// reduction kernel per statistic, re-reading the inputs each
// time; the SYCL study found fusing the reductions 1.4-1.9x faster).
// The statistics end in per-CTA partials reduced in a fixed order by the last CTA
// to finish, so they are run-to-run deterministic for a given launch shape.
#pragma once
#ifdef __CUDACC_RTC__          // run-time compiled (NVRTC, bhist_jit.cu): no host headers
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
#ifndef BH_FILL_TU
#define BH_FILL_TU
#endif
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace bh {

constexpr int kMaxDim = 3;
constexpr int kThreadsGlobal = 512;   // GLOBAL sink: kGlobalCtas CTAs/SM
#ifndef BH_GLOBAL_CTAS
#define BH_GLOBAL_CTAS 2
#endif
constexpr int kGlobalCtas = BH_GLOBAL_CTAS;   // k_fill's GLOBAL CTAs per SM (launch bounds + grid)
#ifndef BH_SMEM_THREADS
#define BH_SMEM_THREADS 1024
#endif
constexpr int kThreadsSmem = BH_SMEM_THREADS;   // PRIV / CACHE sinks: 1 CTA/SM owns the SM's shared memory
template <int SINK> struct ThreadsOf {   // SINK_GLOBAL == 1
    static constexpr int v = SINK == 1 ? kThreadsGlobal : kThreadsSmem;
};
// k_fill: the weighted 3-D CACHE fill (11 float64 stats, the register hot bin, warp
// aggregation) spills at 64 registers/thread; 768 threads (80 registers) measured C4w 3.43 ->
// 3.12 ms, while every other shape is faster at 1024 (C4 1.19 vs 1.37 ms)
template <int SINK, int DIM, bool W> struct FillThreads {    // SINK_CACHE == 2
    static constexpr int v = (SINK == 2 && W && DIM == 3) ? 768 : ThreadsOf<SINK>::v;
};

// Streaming (evict-first) loads of the input columns: each byte is read once.
__device__ __forceinline__ double2 ld_stream(const double2 *p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }
__device__ __forceinline__ float4 ld_stream(const float4 *p) { return __ldcs(p); }

// Axis as the kernels see it.  Fixed axes use (xmin, xmax, D = xmax-xmin,
// inv = n/D), all rounded once on the host exactly as the definition rounds them.
// Variable axes use the edges plus a monotone "guide" table.
struct AxisP {
    int32_t n;       // in-range bins
    int32_t var;     // 0 fixed, 1 variable
    double xmin;     // fixed: xmin; variable: e[0]
    double xmax;     // fixed: xmax; variable: e[n]
    double D;        // fixed: RN(xmax - xmin)
    double inv;      // fixed: RN(n / D)
    const double *e;         // variable: n+1 edges (device)
    const uint32_t *guide;   // variable: gcells+1 entries, guide[c] = #{interior i : cell(e_i) < c}
    int32_t gcells;          // variable: number of cells (power of two)
    double gscale;           // variable: gcells / (e[n] - e[0])
    const float *e32;        // variable: RN-to-float32 copy of the edges (device), staged in smem
    int32_t tab_off;         // variable + VSM: byte offset of [e32 | guide] in dynamic smem
    int32_t g16;             // variable + VSM: guide staged as uint32 (0), uint16 (1, n-1 < 65536) or
                             // packed uint16 (2, n-1 < 16384): guide[c] << 2 | min(guide[c+1]-guide[c], 3);
                             // 3: compact table, no float32 edges (see find_bin_var_compact);
                             // 4: the same with log-domain cells (lg > 0)
    const uint4 *tab_img;    // variable: the shared-memory image [e32 | guide in mode g16] (mode 3: the
                             // compact table alone), built at create
    int32_t tab_bytes;       // its size (multiple of 16)
    int32_t lg;              // variable: 0 linear guide cells; > 0 log-domain cells (edges > 0): cell =
    long long kb;            // (bits(x) >> lg) - kb, kb = bits(e[0]) >> lg (positive doubles order as
                             // their bit patterns, so the cell is monotone in x; log-spaced edges get
                             // ~1 edge per cell where linear cells crowd them, e.g. C5's H3)
};

struct FillP {
    int64_t n;               // events in this launch
    const double *x[kMaxDim];
    const double *w;         // nullptr: unit weights
    AxisP ax[kMaxDim];
    int32_t st1, st2;        // strides of axes 1 and 2 in the flat bin index
    int32_t G;               // total bins (flow included)
    int32_t K;               // number of stats
    int32_t peel;            // vector path: leading events handled one by one (alignment)
    int32_t cache_slots;     // CACHE strategy: shared-memory slots (power of two)
    int32_t replicas;        // PRIV strategy: copies of the private bins (warp w uses w % replicas)
    int32_t wc_off;          // weighted PRIV: byte offset of the per-warp hot-bin caches (-1: none,
                             // plain CAS sink; >= 0: collision-adaptive sink SINK_PRIVA)
    unsigned long long *count;   // unit-weight counts [G]
    double *sw;                  // weighted (sum w, sum w^2) of bin g at sw[2g], sw[2g+1]: one 16-byte
                                 // cell per bin, so one warp RED instruction can add both (red_sw_pairs)
    double *partials;            // [gridDim.x * K]
    unsigned int *counter;       // last-CTA ticket
    double *stats;               // [K], running totals
    unsigned long long *entries; // running entries
    int64_t entries_add;         // added to *entries by the last CTA
    const int32_t *gate;         // AUTO's device-side strategy decision: the kernel runs only if
    int32_t gate_run;            // bit mask: run iff gate == nullptr or bit *gate of gate_run is set
                                 // (otherwise every CTA exits at once)
    const unsigned int *win;     // unit CACHE: the probe's dense box (x0, wx, y0, wy) of bins kept as
    int32_t win_off;             // shared-memory u32 counts at byte win_off (nullptr: none)
    int32_t hot_off;             // weighted PRIVA / CACHE: byte offset of the lane window in shared memory
    const struct HotTab *hot;    // the lane-private window of hot cells (nullptr: none)
};

__device__ __forceinline__ bool gated_off(const int32_t *gate, int32_t mask) {
    return gate && !((mask >> (__ldcg(gate) & 31)) & 1);
}
__host__ __device__ constexpr int32_t gate_bit(int v) { return 1 << v; }

// ------------------------------------------------------------------ FindBin
// Fixed axis: b = 1 + floor(n*(x-xmin)/(xmax-xmin)), evaluated as
// the IEEE binary64 expression q = RN(RN(n*RN(x-xmin))/D) (reading R2).  Fast path:
// q' = RN(RN(x-xmin)*inv) with inv = RN(n/D); |q' - q| <= ~4u*q (u = 2^-53).  If
// trunc(q'(1-2^-40)) == trunc(q'(1+2^-40)) (both products rounded, so the computed
// interval still contains q), every value in it -- q included -- truncates to the
// same integer, and the division is skipped; otherwise (~1e-6 of uniform events)
// the exact expression runs.  q >= 0, so truncation == floor.  All operations are
// explicit _rn intrinsics: nvcc may not contract or reorder them.
static __device__ __noinline__ int fixed_exact_quotient(int n, double d, double D) {   // rare path, out of line
    return (int)__ddiv_rn(__dmul_rn((double)n, d), D);
}

__device__ __forceinline__ int find_bin_fixed(const AxisP &a, double x) {
    // branch-free except the rare exact fallback: flow routing by selects
    const bool under = x < a.xmin;
    const bool over = !(x < a.xmax);     // x == xmax and NaN -> overflow (R5)
    const double d = __dsub_rn(x, a.xmin);
    const double q = __dmul_rn(d, a.inv);
    int b = (int)__dmul_rn(q, 1.0 - 0x1p-40);          // cvt.rzi: NaN -> 0, saturating
    if (b != (int)__dmul_rn(q, 1.0 + 0x1p-40) && !under && !over) b = fixed_exact_quotient(a.n, d, a.D);
    b = under ? -1 : (over ? a.n : b);
    return 1 + b;                        // q <= n: bin n+1 is overflow (R4)
}

// Guide cell of a coordinate x >= e[0]: monotone non-decreasing in x (RN is
// monotone, gscale > 0, truncation and min are monotone).  The same function
// builds the table, so the table is exact for it.
__device__ __forceinline__ int guide_cell(const AxisP &a, double x) {
    if (a.lg) {                          // log domain: x >= e[0] > 0, so the key is >= 0
        const long long k = (__double_as_longlong(x) >> a.lg) - a.kb;
        return k < a.gcells - 1 ? (int)k : a.gcells - 1;
    }
    const double t = __dmul_rn(__dsub_rn(x, a.xmin), a.gscale);
    const int c = (int)t;               // cvt.rzi saturates; t >= 0
    return c < a.gcells - 1 ? c : a.gcells - 1;
}

// Variable axis, PAPER.md:126,138 ("binary search"): b = #{edges <= x} (R1).
// Interior edges 1..lo of the cell are < x, lo+1..hi share x's cell, hi+1.. are > x
// (monotonicity of guide_cell), so b = 1 + lo + #{i in (lo, hi] : e_i <= x}; the
// remaining count is a binary search over the (usually 0-3) edges of the cell.
template <typename EdgeLoad>
__device__ __forceinline__ int find_bin_var_impl(const AxisP &a, double x, const uint32_t *guide, EdgeLoad edge) {
    if (x < a.xmin) return 0;
    if (!(x < a.xmax)) return a.n + 1;
    const int c = guide_cell(a, x);
    int lo = (int)guide[c], hi = (int)guide[c + 1];
    while (lo < hi) {                    // largest l in [lo, hi] with l == lo or e[l] <= x
        const int m = (lo + hi + 1) >> 1;
        if (edge(m) <= x) lo = m; else hi = m - 1;
    }
    return 1 + lo;
}

__device__ __forceinline__ int find_bin_var_global(const AxisP &a, double x) {
    return find_bin_var_impl(a, x, a.guide, [&](int i) { return __ldg(a.e + i); });
}

// Shared-memory variant: the guide and a float32 copy of the edges live in smem.
// RN-to-float is monotone, so e32_i < x32 implies e_i < x and e32_i > x32 implies
// e_i > x; only a float tie needs the exact float64 edge (global, ~1e-3 of events
// on the C2 axis).  The result is therefore identical to the float64 search.
template <int GM>   // guide mode: 0 uint32, 1 uint16, 2 packed uint16 (AxisP::g16)
__device__ __forceinline__ int find_bin_var_smem(const AxisP &a, double x, const unsigned char *tab) {
    if (x < a.xmin) return 0;
    if (!(x < a.xmax)) return a.n + 1;
    const float *e32 = reinterpret_cast<const float *>(tab);
    const unsigned char *gt = tab + ((4 * (a.n + 1) + 15) & ~15);
    const int c = guide_cell(a, x);
    int lo, hi;
    if (GM == 2) {                       // one load per event: range start and edge count
        const uint32_t v = reinterpret_cast<const uint16_t *>(gt)[c];
        lo = (int)(v >> 2);
        hi = (v & 3u) < 3u ? lo + (int)(v & 3u) : (int)(reinterpret_cast<const uint16_t *>(gt)[c + 1] >> 2);
    } else if (GM == 1) {
        lo = reinterpret_cast<const uint16_t *>(gt)[c];
        hi = reinterpret_cast<const uint16_t *>(gt)[c + 1];
    } else {
        lo = (int)reinterpret_cast<const uint32_t *>(gt)[c];
        hi = (int)reinterpret_cast<const uint32_t *>(gt)[c + 1];
    }
    const float x32 = __double2float_rn(x);
    while (lo < hi) {
        const int m = (lo + hi + 1) >> 1;
        const float em = e32[m];
        const bool le = em < x32 ? true : (em > x32 ? false : (__ldg(a.e + m) <= x));
        if (le) lo = m; else hi = m - 1;
    }
    return 1 + lo;
}

// Compact mode (g16 == 3, n-1 < 16384): one 32-bit shared-memory word per guide cell and
// no float32 edge array.  With t = RN(RN(x-e0)*gscale) (guide_cell's monotone t) and
// Q(x) = floor(256 t) (exact scaling), the cell is c = Q >> 8 and the quantized position
// inside it q = Q & 255 (clamped to the last cell as guide_cell clamps, with q = 255 there).
// Word c = lo | min(cnt,3) << 14 | q(e_{lo+1}) << 16 | q(e_{lo+2}) << 24, where lo = guide[c]
// and cnt = guide[c+1] - guide[c] interior edges lie in cell c.  (c, q) is monotone in x, so
// q(x) > q(e_i) implies x > e_i and q(x) < q(e_i) implies x < e_i; only an equal q (a tie,
// ~cnt/256 of the events) or a cell of >= 3 edges reads the float64 edges (global, L1/L2
// resident).  One LDS.32 per event instead of the guide load plus the float32 edge search.
template <bool LOG = false>              // LOG: log-domain cells (g16 == 4), a compile-time mode so
__device__ __forceinline__ int compact_cell(const AxisP &a, double x, int &q) {   // C2's kernel carries no log path
    if (LOG) {                           // log domain (lg >= 8): the next 8 bits are the position
        const long long k = (__double_as_longlong(x) >> (a.lg - 8)) - (a.kb << 8);
        int c = (int)(k >> 8);
        q = (int)(k & 255);
        if (k >= ((long long)a.gcells << 8)) { c = a.gcells - 1; q = 255; }
        return c;
    }
    const double t = __dmul_rn(__dsub_rn(x, a.xmin), a.gscale);
    const int qf = (int)__dmul_rn(t, 256.0);         // floor(256 t); t >= 0 and < ~gcells
    int c = qf >> 8;
    q = qf & 255;
    if (c > a.gcells - 1) { c = a.gcells - 1; q = 255; }
    return c;
}

// (the edges by pointer, not the AxisP by reference: a reference into the kernel parameters
// makes nvcc copy the whole FillP to local memory -- measured +9% instructions on C2)
static __device__ __noinline__ int compact_slow(const double *e, double x, const uint32_t *tab, int c, int lo, int cnt) {
    // count the cell's interior edges e[lo+1 .. hi] <= x exactly (ties / >= 3 edges)
    int hi = cnt < 3 ? lo + cnt : (int)(tab[c + 1] & 0x3fffu);
    int l = lo;                                      // largest l in [lo, hi] with l == lo or e[l] <= x
    while (l < hi) {
        const int m = (l + hi + 1) >> 1;
        if (__ldg(e + m) <= x) l = m; else hi = m - 1;
    }
    return 1 + l;
}

template <bool CHECK_RANGE = true, bool LOG = false>
__device__ __forceinline__ int find_bin_var_compact(const AxisP &a, double x, const unsigned char *tabc) {
    if (x < a.xmin) return 0;
    if (!(x < a.xmax)) return a.n + 1;
    const uint32_t *tab = reinterpret_cast<const uint32_t *>(tabc);
    int q;
    const int c = compact_cell<LOG>(a, x, q);
    const uint32_t v = tab[c];
    const int lo = (int)(v & 0x3fffu), cnt = (int)((v >> 14) & 3u);
    const int p1 = (int)((v >> 16) & 255u), p2 = (int)(v >> 24);
    const bool tie = (cnt >= 1 && q == p1) || (cnt >= 2 && q == p2);
    if (tie || cnt == 3) return compact_slow(a.e, x, tab, c, lo, cnt);
    return 1 + lo + (int)(cnt >= 1 && q > p1) + (int)(cnt >= 2 && q > p2);
}

__device__ __forceinline__ int find_bin_var_smem_any(const AxisP &a, double x, const unsigned char *tab) {
    if (a.g16 == 3) return find_bin_var_compact(a, x, tab);
    if (a.g16 == 4) return find_bin_var_compact<true, true>(a, x, tab);
    return a.g16 == 2 ? find_bin_var_smem<2>(a, x, tab)
                      : (a.g16 ? find_bin_var_smem<1>(a, x, tab) : find_bin_var_smem<0>(a, x, tab));
}

// VM (variable-axis mode, a template constant): 0 = every axis fixed (no variable-axis
// code at all), 1 = variable-axis tables staged in shared memory, 2 = tables in global,
// 3 = tables in shared memory and every variable axis in the compact mode (g16 == 3).
// VAR1: the axis is known to be variable (1-D histograms with VM != 0).
template <int VM, bool VAR1 = false>
__device__ __forceinline__ int find_bin(const AxisP &a, double x, const unsigned char *smem) {
#ifdef BH_EXP_NOSEARCH   // experiment only (wrong results): bin from the guide cell alone
    if (a.var) return x < a.xmin ? 0 : (!(x < a.xmax) ? a.n + 1 : 1 + (int)((long long)guide_cell(a, x) * a.n / a.gcells));
#endif
    if (VM == 0 || (!VAR1 && !a.var)) return find_bin_fixed(a, x);
    if (VM == 3) return find_bin_var_compact(a, x, smem + a.tab_off);
    if (VM == 1) {
        return find_bin_var_smem_any(a, x, smem + a.tab_off);
    }
    return find_bin_var_global(a, x);
}

__device__ __forceinline__ int find_bin(const AxisP &a, double x) { return find_bin<2>(a, x, nullptr); }

// Copy each variable axis' table image (float32 edges + guide, built once at create in
// the staged layout) into shared memory: 16-byte loads, four per thread in flight.
template <int DIM>
__device__ __forceinline__ void stage_axes(const AxisP *ax, unsigned char *smem) {
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        if (!ax[a].var) continue;
        const uint4 *src = ax[a].tab_img;
        uint4 *dst = reinterpret_cast<uint4 *>(smem + ax[a].tab_off);
        const int n16 = ax[a].tab_bytes / 16;
        for (int base = 0; base < n16; base += 4 * (int)blockDim.x) {
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = base + k * (int)blockDim.x + (int)threadIdx.x;
                if (i < n16) v[k] = __ldg(src + i);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = base + k * (int)blockDim.x + (int)threadIdx.x;
                if (i < n16) dst[i] = v[k];
            }
        }
    }
}

// ------------------------------------------------------------------ stats
template <int DIM>
struct NStats { static constexpr int K = DIM == 1 ? 4 : DIM == 2 ? 7 : 11; };

// Register accumulator of the GetStats sums (ROOT order, reading R7/R8).
template <int DIM, bool W>
struct Acc {
    static constexpr int K = NStats<DIM>::K;
    double s[K];
    unsigned long long cnt;   // unit weights: in-range count (= sumw = sumw2, exact)
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int k = 0; k < K; ++k) s[k] = 0.0;
        cnt = 0;
    }
    __device__ __forceinline__ void add(const double (&x)[DIM], double w) {
        double wx = W ? w * x[0] : x[0];
        if (W) { s[0] += w; s[1] = fma(w, w, s[1]); } else { ++cnt; }
        s[2] += wx;
        s[3] = fma(wx, x[0], s[3]);
        if (DIM >= 2) {
            const double wy = W ? w * x[1] : x[1];
            s[4] += wy;
            s[5] = fma(wy, x[1], s[5]);
            s[6] = fma(wx, x[1], s[6]);
            if (DIM == 3) {
                const double wz = W ? w * x[2] : x[2];
                s[7] += wz;
                s[8] = fma(wz, x[2], s[8]);
                s[9] = fma(wx, x[2], s[9]);
                s[10] = fma(wy, x[2], s[10]);
            }
        }
    }
    __device__ __forceinline__ void finalize_unit() {
        if (!W) { s[0] = (double)cnt; s[1] = (double)cnt; }
    }
};

__device__ __forceinline__ double warp_sum_fixed(double v) {   // butterfly: same order on every run
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block reduction of the K sums -> partials[blockIdx.x]; the last CTA to arrive
// sums the partials in block order and adds them to the running stats
// (include-initial) and adds the event count to entries.
template <int K>
__device__ __forceinline__ void block_stats_finish(const FillP &p, double (&s)[K]) {
    __shared__ double red[1024 / 32][K];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double v = s[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double t = 0.0;
        const int nw = blockDim.x >> 5;
        for (int i = 0; i < nw; ++i) t += red[i][threadIdx.x];
        p.partials[(size_t)blockIdx.x * K + threadIdx.x] = t;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(p.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // warp k sums statistic k over the blocks: lane-strided loads in flight together, then
    // a fixed butterfly (deterministic for a given grid); small fills are latency-bound
    for (int k = warp; k < K; k += (int)(blockDim.x >> 5)) {   // any blockDim >= 32
        double t = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) t += __ldcg(p.partials + (size_t)b * K + k);
        t = warp_sum_fixed(t);
        if (lane == 0) p.stats[k] += t;
    }
    if (threadIdx.x == 0) {
        *p.entries += (unsigned long long)p.entries_add;
        *p.counter = 0u;
    }
}

// ------------------------------------------------------------------ bin sinks
// SINK_PRIVA: PRIV whose weighted adds adapt to collisions (used with replicas > 1,
// i.e. small bin spaces, where peaked data makes warp-level collisions likely).
enum Sink { SINK_PRIV = 0, SINK_GLOBAL = 1, SINK_CACHE = 2, SINK_PRIVA = 3 };

__device__ __forceinline__ bool cas128_shared(uint32_t addr, unsigned long long cl, unsigned long long ch,
                                              unsigned long long nl, unsigned long long nh,
                                              unsigned long long &ol, unsigned long long &oh) {
    asm volatile(
        "{\n .reg .b128 c, n, o;\n mov.b128 c, {%2, %3};\n mov.b128 n, {%4, %5};\n"
        " atom.shared.cas.b128 o, [%6], c, n;\n mov.b128 {%0, %1}, o;\n}"
        : "=l"(ol), "=l"(oh)
        : "l"(cl), "l"(ch), "l"(nl), "l"(nh), "r"(addr)
        : "memory");
    return ol == cl && oh == ch;
}

__device__ __forceinline__ void exch128_shared(uint32_t addr, unsigned long long il, unsigned long long ih,
                                               unsigned long long &ol, unsigned long long &oh) {
    asm volatile(
        "{\n .reg .b128 d, v;\n mov.b128 v, {%2, %3};\n atom.shared.exch.b128 d, [%4], v;\n mov.b128 {%0, %1}, d;\n}"
        : "=l"(ol), "=l"(oh)
        : "l"(il), "l"(ih), "r"(addr)
        : "memory");
}

// (sumw, sumw2) += (w, w*w) on one 16-byte shared-memory cell (smem float64 add has no
// native atomic on sm_100a; nvcc's atomicAdd(double*) is a CAS loop).  Returns how many
// rounds collided with another thread's add (contention telemetry for PrivSink).
//
// Take-and-return with 128-bit exchanges (ATOMS.EXCH.128), no load and no compare: take the
// cell's pair (leaving +0,+0), add, exchange the sum back; if that exchange brought back a
// pair another thread deposited in the meantime, take the cell again, merge, and repeat.
// Every exchange is atomic, so (cell + the pairs threads hold) always equals the sum of the
// adds made so far, and an add ends when its sum lands in an empty cell (a deposit of +0,+0
// carries nothing).  Measured on 10,002 random cells (tools/microbench/mb4.cu, 1024
// threads/SM): 0.93 adds/clk/SM vs 0.64 for a load + 128-bit CAS loop, and 99 vs 1.2 G
// adds/s when a quarter of the adds hit one cell (a lost CAS re-reads and retries; a
// deposit is merged by whoever finds it).
// BH_SINK_CAS (A/B builds): the round-1 load + ATOMS.CAS.128 loop.
__device__ __forceinline__ int add2_shared_count(double2 *cell, double w, double w2) {
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(cell);
    int lost = 0;
#ifdef BH_SINK_CAS
    double2 cur = *cell;
    while (true) {
        unsigned long long ol, oh;
        if (cas128_shared(addr, __double_as_longlong(cur.x), __double_as_longlong(cur.y),
                          __double_as_longlong(cur.x + w), __double_as_longlong(cur.y + w2), ol, oh))
            return lost;
        ++lost;
        cur = make_double2(__longlong_as_double(ol), __longlong_as_double(oh));
    }
#else
    unsigned long long l, h;
    exch128_shared(addr, 0ull, 0ull, l, h);
    double s1 = __longlong_as_double(l) + w, s2 = __longlong_as_double(h) + w2;
    while (true) {
        exch128_shared(addr, __double_as_longlong(s1), __double_as_longlong(s2), l, h);
        if ((l | h) == 0ull) return lost;
        ++lost;
        unsigned long long l2, h2;
        exch128_shared(addr, 0ull, 0ull, l2, h2);
        s1 = __longlong_as_double(l) + __longlong_as_double(l2);
        s2 = __longlong_as_double(h) + __longlong_as_double(h2);
    }
#endif
}

__device__ __forceinline__ void add2_shared(double2 *cell, double w, double w2) { (void)add2_shared_count(cell, w, w2); }

// Global (sum w, sum w^2) of bin g: sw[2g], sw[2g+1], one 16-byte cell.  The L2 atomic units
// serve one request per 32-byte sector, not per element: two lanes adding the two halves of
// one cell in the SAME warp RED instruction cost one request, the same as one u64 RED
// (tools/microbench/mb6.cu on 1M random cells: 193 G (w, w^2) pairs/s paired vs 96 G/s with
// the halves in two instructions; u64 192 G/s).
// Fire-and-forget float64 add to global memory (RED, no return data; nvcc emitted a returning
// ATOM for atomicAdd in the paired loop below: one 32-byte response per event through the xbar).
__device__ __forceinline__ void red_f64(double *addr, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void red_u64(unsigned long long *addr, unsigned long long v) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void red_sw(double *sw, int g, double a, double b) {
    red_f64(sw + 2 * (size_t)g, a);
    red_f64(sw + 2 * (size_t)g + 1, b);
}

// Warp-cooperative (a, b) adds into the global cells: every lane of `act` calls this; the lanes
// in `ib` (a subset of act) each hold one item (g, a, b).  Participating lanes pair up by rank in
// act -- the even one adds an item's a, the odd one its b, in one RED instruction -- so each
// round adds floor(|act| / 2) items with one sector request each.
__device__ __forceinline__ void red_sw_pairs(unsigned act, unsigned ib, double *sw, int g, double a, double b) {
    if (ib == 0u) return;
    const int lane = (int)(threadIdx.x & 31);
    const int np = __popc(act);
    if (np < 2) {
        if (ib & (1u << lane)) red_sw(sw, g, a, b);
        return;
    }
    const int rank = __popc(act & ((1u << lane) - 1u));
    const int per = np >> 1, half = rank & 1, slot = rank >> 1, k = __popc(ib);
    for (int base = 0; base < k; base += per) {
        const int j = base + slot;
        const bool mine = slot < per && j < k;
        const int src = !mine ? lane : ib == 0xffffffffu ? j : (int)__fns(ib, 0, j + 1);
        const int gg = __shfl_sync(act, g, src);
        const double va = __shfl_sync(act, a, src), vb = __shfl_sync(act, b, src);
        if (mine) red_f64(sw + 2 * (size_t)gg + half, half ? vb : va);
    }
}

// Shared-memory layout of the PRIV sink: unit -> uint32 count[G];
// weighted -> double2 (sumw, sumw2)[G].
// With R > 1 replicas (small bin spaces) warp w adds into replica w % R, so hot
// bins are not contended across warps (R = 32: per-warp private histograms); the
// flush sums the replicas.
//
// SINK_PRIVA (weighted) also gives every warp a private direct-mapped cache of kWC hot
// bins in shared memory: in aggregated mode the leader of a group of >= 2 lanes on one
// bin adds the group's (sum w, sum w^2) to its warp's cache entry with a plain
// read-modify-write (the warp is the only writer), claiming the entry if needed (the
// previous occupant is flushed into the replica).  A peaked weighted histogram thus
// stops serializing all warps of a replica on a few cells (100x100 Cauchy-peaked fill:
// 9 -> see DESIGN.md), while spread data never enters aggregated mode.
#ifndef BH_WC_BITS
#define BH_WC_BITS 5      // 32 entries: C5 5.77 -> 5.62 ms, peaked 100x100 weighted 26 -> 47 G events/s over 16
#endif
constexpr int kWCBits = BH_WC_BITS;                  // 8 / 16 / 32 entries (<= 32: one per lane)
constexpr int kWC = 1 << kWCBits;
constexpr int kWCBytes = kWC * 4 + kWC * 16;         // tags int32[kWC], then (s1, s2) double2[kWC]

// A warp's private direct-mapped cache of hot weighted bins (PRIVA; in front of CACHE's
// slots it measured slower on C4w, 4.36 vs 3.48 ms, and is not used there).
// absorb(): called by every lane of `act` after the group sums; if `act` is the full
// warp, a group leader whose bin is cached adds with a plain read-modify-write (the
// converged warp is the only writer, and one leader per bin); a leader of a group of
// >= 2 that misses claims the entry -- one claimant per entry, the previous occupant
// spilled through `spill(bin, s1, s2)`.  Returns whether this lane's group was absorbed.
struct WarpHot {
    unsigned char *wc;
    __device__ __forceinline__ void init(unsigned char *base) {
        wc = base + (size_t)(threadIdx.x >> 5) * kWCBytes;
        if ((threadIdx.x & 31) < kWC) reinterpret_cast<int32_t *>(wc)[threadIdx.x & 31] = -1;
    }
    template <typename Spill>
    __device__ __forceinline__ bool absorb(unsigned act, bool leader, int gsize, int g, double s1, double s2,
                                           Spill spill) {
        // Plain read-modify-writes are safe only if no other lanes of this warp can be in
        // here at the same time: with independent thread scheduling two diverged subsets
        // of a warp (e.g. the vector loop's last pairs and the scalar tail) may both be
        // adding.  So only a converged full warp uses the cache; partial masks go to the
        // caller's atomic path.
        if (act != 0xffffffffu) return false;
        const int lane = (int)(threadIdx.x & 31);
        int32_t *tags = reinterpret_cast<int32_t *>(wc);
        double2 *vals = reinterpret_cast<double2 *>(wc + kWC * 4);
        const int slot = (int)(((uint32_t)g * 2654435761u) >> (32 - kWCBits));
        bool done = false;
        __syncwarp();                    // earlier cache writes of every lane are visible
        if (leader && tags[slot] == g) {
            double2 v = vals[slot];
            v.x += s1;
            v.y += s2;
            vals[slot] = v;
            done = true;
        }
        __syncwarp(act);
        const bool want = leader && !done && gsize >= 2;
        const unsigned wm = __ballot_sync(act, want);
        if (want) {
            const unsigned sp = __match_any_sync(wm, slot);
            if (lane == __ffs(sp) - 1) {
                const int t = tags[slot];
                if (t >= 0) spill(t, vals[slot].x, vals[slot].y);
                tags[slot] = g;
                vals[slot] = make_double2(s1, s2);
                done = true;
            }
        }
        __syncwarp(act);
        return done;
    }
    template <typename Spill>
    __device__ __forceinline__ void drain(Spill spill) {
        __syncwarp();
        const int lane = (int)(threadIdx.x & 31);
        if (lane < kWC) {
            int32_t *tags = reinterpret_cast<int32_t *>(wc);
            const double2 *vals = reinterpret_cast<const double2 *>(wc + kWC * 4);
            if (tags[lane] >= 0) spill(tags[lane], vals[lane].x, vals[lane].y);
            tags[lane] = -1;
        }
        __syncwarp();
    }
};

// A thread's one-entry register cache of its hot bin (CACHE's weighted sink): adds to the cached
// bin stay in registers; an add to another bin goes to shared memory at once while the
// cached bin is "sticky" (it repeated and keeps >= 1/4 of this thread's recent adds), and
// otherwise replaces the cached bin (whose sums go to shared memory instead).  Either way a
// miss costs one shared-memory add, as without the cache, while a hot bin (C4's 43% of the
// events in one cell, C5's Cauchy-peaked H7) is updated by each thread in registers instead
// of by every thread of the SM on one shared-memory cell.  Per-thread chains stay short
// (<= the events of one thread, ~3e3 at 5e8 events).  BH_LANE_CACHE=0 disables it (A/B).
// Measured: C4w 3.83 -> 3.36 ms.  In front of the PRIV weighted sink it cost more than it
// saved (C2 2.00 -> 2.69 ms, uniform 100x100 weighted 217 -> 146 G events/s: register
// spills at 64 registers/thread; and C5's peaked cells are several warm cells, not one).
#ifndef BH_LANE_CACHE
#define BH_LANE_CACHE 1
#endif
#ifndef BH_CACHE_W_AGG       // CACHE weighted: combine the lanes' items of equal bins before the put
#define BH_CACHE_W_AGG 1     // (0: one put per lane -- C4w 3.36 -> 8.72 ms: the float64 exchanges on
#endif                       // a warm slot serialize, unlike the native u32 atomics of unit counts)
#ifndef BH_LANE_CACHE_U      // the same for CACHE's unit-weight counts (no warp aggregation behind it):
#define BH_LANE_CACHE_U 1    // C4 1.32 -> 1.19 ms, C5 5.47 -> 5.42 ms; uniform C3 forced to CACHE
#endif                       // 1.81 -> 1.99 ms (AUTO runs C3 through SORT)
struct RegHot {
    int g = -1;
    uint32_t n = 0, miss = 0;
    double s1 = 0.0, s2 = 0.0;
    // returns true if (g_, w) was absorbed; otherwise (og, on, o1, o2) is the item to add now
    // (on == 0: nothing to add)
    __device__ __forceinline__ bool step(int g_, double w, int &og, uint32_t &on, double &o1, double &o2) {
        if (g_ == g) {
            ++n;
            s1 += w;
            s2 = fma(w, w, s2);
            return true;
        }
        if (n >= 2 && miss < 4 * n) {            // sticky: the event goes to the sink as is
            ++miss;
            og = g_; on = 1; o1 = w; o2 = w * w;
            return false;
        }
        og = g; on = n; o1 = s1; o2 = s2;         // evict (on == 0 while the cache is empty)
        g = g_; n = 1; miss = 0; s1 = w; s2 = w * w;
        return false;
    }
    // the cached sums, once, before the merge barrier
    __device__ __forceinline__ bool take(int &og, uint32_t &on, double &o1, double &o2) {
        og = g; on = n; o1 = s1; o2 = s2;
        g = -1; n = 0;
        return on != 0;
    }
};

#ifndef BH_AGG_ENTER
#define BH_AGG_ENTER 8       // lanes of one add that lost their CAS -> aggregate the next adds
#endif
#ifndef BH_AGG_STAY
#define BH_AGG_STAY 4        // keep aggregating while some bin holds this many lanes
#endif
// Lane-private window of hot cells (weighted PRIVA; AUTO's hot-cell probe k_hot_probe).  A
// peaked weighted histogram (C5's H7: 50x50 on a Cauchy x Gaussian, ~75% of the events in 8
// cells) serializes every sink on a few shared-memory cells: exchanges collide, the warp
// aggregation walks long peer groups.  With the window, each THREAD owns a private (sum w,
// sum w^2) copy of up to kHotW hot cells in shared memory (cell k of thread t at
// [k * blockDim + t]: consecutive lanes, conflict-free LDS.128/STS.128) and adds its events of
// those cells with plain read-modify-writes -- no atomic, no collision; the other events take
// the PRIVA sink.  A direct-mapped table of kHotSlots slots maps a global bin to its window
// index (one LDS.64 per event).  At the end each warp sums its lanes' copies (shuffles) into
// its replica, before the usual merge.  The probe picks the cells from a sample on the device
// and writes `flag` (1: use the window); the fill launches both kernels gated on it.
constexpr int kHotW = 8;                 // window cells per thread (8 x 16 B x 1024 threads = 128 KB)
constexpr int kHotSlots = 64;
struct HotTab {
    int32_t flag, nwin;                  // flag (gate word): 2 window kernel, 1 GLOBAL, 0 plain; nwin: cells
    int32_t cell[kHotW];                 // global bin of window cell k (-1: none)
    int2 tab[kHotSlots];                 // slot -> {global bin, k}; x = -1 empty
};
constexpr int kHotTabSmem = kHotSlots * 8 + kHotW * 4;     // staged table + cell list (16-byte multiple)
__host__ __device__ constexpr size_t hot_smem_bytes(int threads) { return kHotTabSmem + (size_t)kHotW * 16 * threads; }
__host__ __device__ __forceinline__ int hot_slot(int g) { return (int)(((uint32_t)g * 2654435761u) >> 26); }

#ifndef BH_HOT_COLLECTIVE
#define BH_HOT_COLLECTIVE 1
#endif
#ifndef BH_HOT_PLAIN
#define BH_HOT_PLAIN 0      // 1: C5 4.36 vs 4.33 ms (H7 1.31 vs 1.24): the adaptive sink stays
#endif
template <bool B, class T, class F> struct PickT { using type = T; };   // (NVRTC: no <type_traits>)
template <class T, class F> struct PickT<false, T, F> { using type = F; };
struct NoLaneWindow {
    __device__ __forceinline__ bool add(int, double) { return false; }
    template <typename Spill> __device__ __forceinline__ void drain(Spill) {}
};
struct LaneWindow {
    const int2 *htab = nullptr;          // staged slot table
    const int32_t *hcell = nullptr;      // window cell -> global bin (-1: none)
    double2 *hlane = nullptr;            // this thread's copy of window cell 0 (stride blockDim)
    int hn = 0;                          // window cells (0: no window)
    __device__ __forceinline__ void init(const HotTab *hot, unsigned char *b) {
        int2 *t = reinterpret_cast<int2 *>(b);
        int32_t *c = reinterpret_cast<int32_t *>(b + kHotSlots * 8);
        for (int i = threadIdx.x; i < kHotSlots; i += blockDim.x) t[i] = hot->tab[i];
        if (threadIdx.x < kHotW) c[threadIdx.x] = hot->cell[threadIdx.x];
        hn = hot->nwin;
        htab = t;
        hcell = c;
        hlane = reinterpret_cast<double2 *>(b + kHotTabSmem) + threadIdx.x;
        for (int k = 0; k < kHotW; ++k) hlane[k * blockDim.x] = make_double2(0.0, 0.0);
    }
    // (g, w) of a window cell goes to this thread's private copy: plain read-modify-write
    __device__ __forceinline__ bool add(int g, double w) {
        if (!hn) return false;
        const int2 e = htab[hot_slot(g)];
        if (e.x != g) return false;
        double2 *c = hlane + e.y * blockDim.x;
        double2 v = *c;
        v.x += w;
        v.y = fma(w, w, v.y);
        *c = v;
        return true;
    }
    // every lane of every warp: the warp's lane copies summed by shuffles, lane 0 spills them
    template <typename Spill>
    __device__ __forceinline__ void drain(Spill spill) {
        if (!hn) return;
        __syncwarp();
        for (int k = 0; k < kHotW; ++k) {
            const int g = hcell[k];
            if (g < 0) continue;         // (uniform)
            double2 v = hlane[k * blockDim.x];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
                v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
            }
            if ((threadIdx.x & 31) == 0 && (v.x != 0.0 || v.y != 0.0)) spill(g, v.x, v.y);
        }
        __syncwarp();
    }
};

template <bool W, bool ADAPT>
struct PrivSink {
    uint32_t sm;         // shared-memory address of this warp's replica
    bool agg;            // ADAPT: the warp's previous add collided -> aggregate this one first
    WarpHot hot;         // ADAPT && W: this warp's hot-bin cache
    // lane-private window of hot cells (see HotTab); an empty member unless W && ADAPT (a
    // LaneWindow in the plain sink made nvcc keep the kernel parameters in local memory)
    typename PickT<W && ADAPT, LaneWindow, NoLaneWindow>::type lw;
    __device__ __forceinline__ bool lw_active() const {
        if constexpr (W && ADAPT) return lw.hn != 0;
        else return false;
    }
    static constexpr int kCell = W ? 16 : 4;
    static __device__ __forceinline__ size_t stride_of(int G) { return ((size_t)G * kCell + 15) & ~size_t(15); }
    __device__ __forceinline__ void init(unsigned char *s, int G, int R, int wc_off = -1) {
        const size_t stride = stride_of(G);
        sm = (uint32_t)__cvta_generic_to_shared(s + (size_t)((threadIdx.x >> 5) % R) * stride);
        agg = false;
        if (ADAPT && W) hot.init(s + wc_off);
        if (W) {
            for (int i = threadIdx.x; i < R * (int)(stride / 16); i += blockDim.x)
                reinterpret_cast<double2 *>(s)[i] = make_double2(0.0, 0.0);
        } else {
            for (int i = threadIdx.x; i < R * (int)(stride / 4); i += blockDim.x)
                reinterpret_cast<uint32_t *>(s)[i] = 0u;
        }
    }
    // weighted PRIVA with a hot-cell window (k_fill, p.hot set): stage the table, zero the lane cells
    __device__ __forceinline__ void init_hot(const FillP &p, unsigned char *smem) {
        if (!(W && ADAPT) || !p.hot) return;
        lw.init(p.hot, smem + p.hot_off);
    }
    __device__ __forceinline__ void add(int g, double w) {
#if BH_HOT_COLLECTIVE
        if (W && ADAPT && lw_active()) {
            // a window cell goes to this thread's private copy; the lane still takes part in the
            // warp-collective adaptive add (with no item), so the warp stays converged and the
            // per-warp hot-bin cache (full warps only) keeps absorbing the warm cells
            const bool hit = lw.add(g, w);
            double2 *base = reinterpret_cast<double2 *>(__cvta_shared_to_generic(sm));
            const unsigned act = __activemask();
            const int lane = (int)(threadIdx.x & 31);
            agg = __any_sync(act, agg);
            if (agg) {
                const unsigned peers = __match_any_sync(act, hit ? -1 - lane : g);
                agg = __any_sync(act, !hit && __popc(peers) >= BH_AGG_STAY);
                add_aggregated(base, hit ? -1 - lane : g, hit ? 0.0 : w, hit ? 0.0 : w * w, act, peers, !hit);
            } else {
                const int lost = hit ? 0 : add2_shared_count(base + g, w, w * w);
                agg = __popc(__ballot_sync(act, lost > 0)) >= BH_AGG_ENTER;
            }
            return;
        }
#endif
        if (W && ADAPT && lw.add(g, w)) return;     // a window cell: this thread's private copy
        if (W) {
            double2 *base = reinterpret_cast<double2 *>(__cvta_shared_to_generic(sm));
#ifdef BH_EXP_NOCAS   // experiment only (wrong results): plain read-modify-write instead of CAS
            { double2 v = base[g]; v.x += w; v.y += w * w; base[g] = v; return; }
#endif
            // BH_HOT_PLAIN: with a lane window the remaining (colder) cells take the plain
            // exchange add instead of the collision-adaptive machinery
            if (!ADAPT || (BH_HOT_PLAIN && lw_active())) {
                add2_shared(base + g, w, w * w);
                return;
            }
            // plain CAS while a warp's adds collide little (a lost CAS just retries); once
            // >= 8 lanes of an add lost, the next adds first group equal cells with
            // match.any, and keep doing so while some cell holds >= 4 lanes (peaked data)
            const unsigned act = __activemask();
            // lanes outside an earlier partial mask may carry a stale flag: make it uniform
            agg = __any_sync(act, agg);
            if (agg) {
                const unsigned peers = __match_any_sync(act, g);
                agg = __any_sync(act, __popc(peers) >= BH_AGG_STAY);
                add_aggregated(base, g, w, w * w, act, peers);
            } else {
                agg = __popc(__ballot_sync(act, add2_shared_count(base + g, w, w * w) > 0)) >= BH_AGG_ENTER;
            }
        } else {
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(sm + 4u * (uint32_t)g) : "memory");
        }
    }
    // Aggregated add: group sums by a shuffle walk, then per group leader: hit in the
    // warp's hot-bin cache -> plain add; miss with a group of >= 2 -> claim the entry (one
    // claimant per entry, the old occupant flushed into the replica); else CAS.
    __device__ __forceinline__ void add_aggregated(double2 *base, int g, double w, double w2, unsigned act,
                                                   unsigned peers, bool item = true) {
        const int lane = (int)(threadIdx.x & 31);
        const int rounds = __reduce_max_sync(act, (unsigned)__popc(peers));
        double s1 = 0.0, s2 = 0.0;
        unsigned m = peers;
        for (int k = 0; k < rounds; ++k) {
            const int src = m ? __ffs(m) - 1 : lane;
            const double v1 = __shfl_sync(act, w, src), v2 = __shfl_sync(act, w2, src);
            if (m) { s1 += v1; s2 += v2; m &= m - 1; }
        }
        const bool leader = item && lane == __ffs(peers) - 1;
        const bool done = hot.absorb(act, leader, __popc(peers), g, s1, s2,
                                     [&](int t, double a1, double a2) { add2_shared(base + t, a1, a2); });
        if (leader && !done) add2_shared(base + g, s1, s2);
    }
    // Before the block barrier of the merge stage: hot-bin caches -> this warp's replica.
    __device__ __forceinline__ void drain() {
        if (ADAPT && W) {                // window: the warp's lane copies -> its replica
            double2 *base = reinterpret_cast<double2 *>(__cvta_shared_to_generic(sm));
            lw.drain([&](int g, double a1, double a2) { add2_shared(base + g, a1, a2); });
        }
        if (ADAPT && W) {
            double2 *base = reinterpret_cast<double2 *>(__cvta_shared_to_generic(sm));
            hot.drain([&](int t, double a1, double a2) { add2_shared(base + t, a1, a2); });
        }
    }
    // Merge stage of PAPER.md:162-165: each block adds its local bins (summed over the
    // replicas) to the global ones.
    __device__ __forceinline__ void flush(const FillP &p, const unsigned char *s) {
        const int G = p.G, R = p.replicas;
        const size_t stride = stride_of(G);
        // few bins, many replicas (small fills are latency-bound): S lanes per bin sum
        // interleaved replicas, then a shuffle tree combines them
        int S = 1;
        while (S < 32 && 2 * S <= R && (size_t)2 * S * G <= blockDim.x) S *= 2;
        if (S > 1) {
            const int lane = (int)(threadIdx.x & 31), sub = lane & (S - 1);
            const int bins_per_pass = (int)blockDim.x / S;
            for (int i0 = 0; i0 < G; i0 += bins_per_pass) {
                const int i = i0 + (int)threadIdx.x / S;
                const bool ok = i < G;
                if (W) {
                    double a = 0.0, b = 0.0;
                    for (int r = sub; ok && r < R; r += S) {
                        const double2 u = reinterpret_cast<const double2 *>(s + r * stride)[i];
                        a += u.x;
                        b += u.y;
                    }
                    for (int o = S / 2; o > 0; o >>= 1) {
                        a += __shfl_xor_sync(0xffffffffu, a, o);
                        b += __shfl_xor_sync(0xffffffffu, b, o);
                    }
                    if (ok && sub == 0) red_sw(p.sw, i, a, b);
                } else {
                    uint32_t v = 0;
                    for (int r = sub; ok && r < R; r += S) v += reinterpret_cast<const uint32_t *>(s + r * stride)[i];
                    for (int o = S / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if (ok && sub == 0 && v) red_u64(p.count + i, (unsigned long long)v);
                }
            }
            return;
        }
        if (W) {        // component-wise: a warp's REDs cover 16 contiguous cells (8 sectors)
            for (int i = threadIdx.x; i < 2 * G; i += blockDim.x) {
                double v = reinterpret_cast<const double *>(s)[i];
                for (int r = 1; r < R; ++r) v += reinterpret_cast<const double *>(s + r * stride)[i];
                if (v != 0.0) red_f64(p.sw + i, v);
            }
        } else {
            for (int i = threadIdx.x; i < G; i += blockDim.x) {
                uint32_t v = reinterpret_cast<const uint32_t *>(s)[i];
                for (int r = 1; r < R; ++r) v += reinterpret_cast<const uint32_t *>(s + r * stride)[i];
                if (v) red_u64(p.count + i, (unsigned long long)v);
            }
        }
    }
};

template <bool W>
struct GlobalSink {
    // the global state's pointers, copied out of the kernel parameters (a pointer to the
    // parameters would make nvcc copy them to local memory and emit generic atomics)
    double *sw;
    unsigned long long *count;
    __device__ __forceinline__ void bind(const FillP &p) { sw = p.sw; count = p.count; }
    __device__ __forceinline__ void init(unsigned char *, int) {}
    __device__ __forceinline__ void add(int g, double w) {
        if (W) {
            const unsigned act = __activemask();
            red_sw_pairs(act, act, sw, g, w, w * w);
        } else {
            red_u64(count + g, 1ull);
        }
    }
    __device__ __forceinline__ void drain() {}
    __device__ __forceinline__ void flush(const FillP &, const unsigned char *) {}
};

// CACHE sink: direct-mapped shared-memory cache of global bins.  A slot is
// claimed by the first bin that hashes to it (32-bit CAS, native); hits add in
// shared memory, misses go to global atomics.  Equal bins are first aggregated
// across the warp (match.any; counts by popc, weights by a shuffle walk over the
// peer mask) so the hottest bin costs one atomic per warp instead of up to 32
// serialized ones (hot-bin contention, BASELINE.json config 4).
template <bool W>
struct CacheSink {
    uint32_t *keys;
    unsigned char *vals;
    int S;
    double *sw;                          // the global state (see GlobalSink::bind)
    unsigned long long *count;
    __device__ __forceinline__ void bind(const FillP &p) { sw = p.sw; count = p.count; }
    static constexpr uint32_t kEmpty = 0xffffffffu;
    __device__ __forceinline__ void init(unsigned char *s, int slots) {
        S = slots;
        keys = reinterpret_cast<uint32_t *>(s);
        vals = s + (size_t)S * 4;
        for (int i = threadIdx.x; i < S; i += blockDim.x) keys[i] = kEmpty;
        if (W) {
            double *d = reinterpret_cast<double *>(vals);
            for (int i = threadIdx.x; i < 2 * S; i += blockDim.x) d[i] = 0.0;
        } else {
            uint32_t *c = reinterpret_cast<uint32_t *>(vals);
            for (int i = threadIdx.x; i < S; i += blockDim.x) c[i] = 0u;
        }
    }
    __device__ __forceinline__ int slot_of(uint32_t g) const { return (int)((g * 2654435761u) >> 7) & (S - 1); }
    __device__ __forceinline__ int lookup(uint32_t g) {
        const int sl = slot_of(g);
        uint32_t k = keys[sl];
        if (k == kEmpty) {
            k = atomicCAS(keys + sl, kEmpty, g);
            if (k == kEmpty) k = g;
        }
        return k == g ? sl : -1;
    }
    RegHot lc;        // W: this thread's hot bin (in front of the warp aggregation)
    LaneWindow lw;    // W, AUTO's hot-cell window (k_hot_probe): lane-private copies of the hot cells
    __device__ __forceinline__ void init_hot(const FillP &p, unsigned char *smem) {
        if (W && p.hot) lw.init(p.hot, smem + p.hot_off);
    }
    // unit weights: the thread's hot bin as a register count (same stickiness rule as RegHot);
    // the other events go one by one to their slot or the global count, no warp aggregation
    int ug = -1;
    uint32_t un = 0, umiss = 0;
    // unit weights, AUTO's WINDOW decision (k_part_probe): a dense box of the bin space (1-D: an
    // interval; 2-D: x0 <= b0 < x0+wx, y0 <= b1 < y0+wy) kept as private u32 counts in shared
    // memory, the PAPER.md:138 per-block copy for the part of a large bin space where the
    // events are; the bins outside go through the slots / L2 as before.  C5's H6 (1000x1000 on
    // two Gaussians): a 55K-bin box holds ~2/3 of the events.
    uint32_t wsm = 0;                    // shared-memory address of the box counts (0: none)
    int wx0 = 0, wx = 0, wy0 = 0, wy = 0, wst = 1;
    unsigned long long wmag = 0;         // ceil(2^40 / st1): b1 = (g * wmag) >> 40 exactly (g < 2^24)
    __device__ __forceinline__ void init_win(const FillP &p, unsigned char *smem, int dim) {
        if (W || !p.win) return;
        wx0 = (int)__ldcg(p.win);
        wx = (int)__ldcg(p.win + 1);
        wy0 = (int)__ldcg(p.win + 2);
        wy = (int)__ldcg(p.win + 3);
        if (wx <= 0) return;
        wst = p.st1;
        wmag = dim >= 2 ? ((1ull << 40) + (unsigned long long)p.st1 - 1) / (unsigned long long)p.st1 : 0ull;
        uint32_t *c = reinterpret_cast<uint32_t *>(smem + p.win_off);
        for (int i = threadIdx.x; i < wx * wy; i += blockDim.x) c[i] = 0u;
        wsm = (uint32_t)__cvta_generic_to_shared(c);
    }
    __device__ __forceinline__ void put_count(int g, uint32_t c) {
        if (wsm) {
            const uint32_t by = wmag ? (uint32_t)(((unsigned long long)(uint32_t)g * wmag) >> 40) : 0u;
            const uint32_t ux = (uint32_t)g - by * (uint32_t)wst - (uint32_t)wx0, uy = by - (uint32_t)wy0;
            if (ux < (uint32_t)wx && uy < (uint32_t)wy) {
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(wsm + 4u * (ux + (uint32_t)wx * uy)), "r"(c) : "memory");
                return;
            }
        }
        const int sl = lookup((uint32_t)g);
        if (sl >= 0) atomicAdd(reinterpret_cast<uint32_t *>(vals) + sl, c);
        else red_u64(count + g, (unsigned long long)c);
    }
    __device__ __forceinline__ void add(int g, double w) {
        if (W && lw.add(g, w)) return;
#if BH_LANE_CACHE
        if (W) {
            uint32_t on;
            double o1, o2;
            int og;
            if (lc.step(g, w, og, on, o1, o2)) return;
            add_item(og, on != 0, o1, o2);
            return;
        }
#endif
#if BH_LANE_CACHE_U
        if (!W) {
            if (g == ug) { ++un; return; }
            if (un >= 2 && umiss < 4 * un) { ++umiss; put_count(g, 1u); return; }
            if (un) put_count(ug, un);
            ug = g;
            un = 1;
            umiss = 0;
            return;
        }
#endif
        const unsigned act = __activemask();
        const unsigned peers = __match_any_sync(act, g);
        const int lane = (int)(threadIdx.x & 31);
        const int leader = __ffs(peers) - 1;
        if (W) {
            // each lane sums w and w*w over its peer group (lane order), walking its own
            // peer mask; every lane runs the same number of shuffles (the largest group)
            const int rounds = __reduce_max_sync(act, (unsigned)__popc(peers));
            double s1 = 0.0, s2 = 0.0;
            unsigned m = peers;
            for (int k = 0; k < rounds; ++k) {
                const int src = m ? __ffs(m) - 1 : lane;
                const double v = __shfl_sync(act, w, src);
                if (m) { s1 += v; s2 = fma(v, v, s2); m &= m - 1; }
            }
            if (lane == leader) put(g, s1, s2);
        } else {
            if (lane == leader) {
                const uint32_t c = (uint32_t)__popc(peers);
                const int sl = lookup((uint32_t)g);
                if (sl >= 0) atomicAdd(reinterpret_cast<uint32_t *>(vals) + sl, c);
                else red_u64(count + g, (unsigned long long)c);
            }
        }
    }
    // a weighted item (a lane cache's (sum w, sum w^2) of bin g, or one event) of the lanes
    // with has=true: equal bins of the warp combine first (match.any + a shuffle walk over
    // the peer mask), then the group leader puts the sums
    // group sums that miss the slots go to the global cells with paired-lane REDs
    __device__ __forceinline__ void add_item(int g, bool has, double w1, double w2) {
#if !BH_CACHE_W_AGG
        if (has) put(g, w1, w2);
        return;
#endif
        const unsigned act0 = __activemask();
        const unsigned act = __ballot_sync(act0, has);
        bool glob = false;
        double s1 = 0.0, s2 = 0.0;
        if (has) {
            const unsigned peers = __match_any_sync(act, g);
            const int lane = (int)(threadIdx.x & 31);
            const int rounds = __reduce_max_sync(act, (unsigned)__popc(peers));
            unsigned m = peers;
            for (int k = 0; k < rounds; ++k) {
                const int src = m ? __ffs(m) - 1 : lane;
                const double v1 = __shfl_sync(act, w1, src), v2 = __shfl_sync(act, w2, src);
                if (m) { s1 += v1; s2 += v2; m &= m - 1; }
            }
            if (lane == __ffs(peers) - 1) {
                const int sl = lookup((uint32_t)g);
                if (sl >= 0) add2_shared(reinterpret_cast<double2 *>(vals) + sl, s1, s2);   // (sumw, sumw2) cell
                else glob = true;
            }
        }
        red_sw_pairs(act0, __ballot_sync(act0, glob), sw, g, s1, s2);
    }
    // a weighted group sum into its shared-memory slot, or straight to the global cell
    __device__ __forceinline__ void put(int g, double s1, double s2) {
        const int sl = lookup((uint32_t)g);
        if (sl >= 0) add2_shared(reinterpret_cast<double2 *>(vals) + sl, s1, s2);
        else red_sw(sw, g, s1, s2);
    }
    __device__ __forceinline__ void drain() {
        if (!W && BH_LANE_CACHE_U && un) {
            put_count(ug, un);
            un = 0;
            ug = -1;
        }
        if (W && BH_LANE_CACHE) {
            int og;
            uint32_t on;
            double o1, o2;
            if (lc.take(og, on, o1, o2)) put(og, o1, o2);
        }
        if (W) lw.drain([&](int g, double a1, double a2) { put(g, a1, a2); });
    }
    __device__ __forceinline__ void flush(const FillP &p, const unsigned char *) {
        if (wsm) {                       // the box -> global, once per CTA
            const uint32_t *wc = reinterpret_cast<const uint32_t *>(__cvta_shared_to_generic(wsm));
            for (int i = threadIdx.x; i < wx * wy; i += blockDim.x)
                if (wc[i]) red_u64(p.count + (wx0 + i % wx) + (size_t)wst * (wy0 + i / wx), (unsigned long long)wc[i]);
        }
        for (int i = threadIdx.x; i < S; i += blockDim.x) {
            const uint32_t k = keys[i];
            if (k == kEmpty) continue;
            if (W) {
                const double2 d = reinterpret_cast<const double2 *>(vals)[i];
                red_sw(p.sw, (int)k, d.x, d.y);
            } else {
                const uint32_t v = reinterpret_cast<const uint32_t *>(vals)[i];
                if (v) red_u64(p.count + k, (unsigned long long)v);
            }
        }
    }
};

template <int SINK, bool W> struct SinkOf;
template <bool W> struct SinkOf<SINK_PRIV, W> { using T = PrivSink<W, false>; };
template <bool W> struct SinkOf<SINK_PRIVA, W> { using T = PrivSink<W, true>; };
template <bool W> struct SinkOf<SINK_GLOBAL, W> { using T = GlobalSink<W>; };
template <bool W> struct SinkOf<SINK_CACHE, W> { using T = CacheSink<W>; };

// ------------------------------------------------------------------ the fill kernel
template <int DIM, bool W, int VM, typename S>
__device__ __forceinline__ void do_event(const FillP &p, const double (&x)[DIM], double w, S &sink,
                                         Acc<DIM, W> &acc, const unsigned char *smem) {
    int g = 0, mul = 1;
    bool inr = true;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const int b = find_bin<VM, DIM == 1 && VM != 0>(p.ax[a], x[a], smem);   // step (1), per axis
        inr &= (b >= 1) & (b <= p.ax[a].n);
        g += b * mul;
        if (a + 1 < DIM) mul = (a == 0) ? p.st1 : p.st2;
    }
    sink.add(g, w);                                      // step (2): bin += w, sumw2 += w*w
    if (inr) acc.add(x, w);                              // step (3): stats, in-range only (R6)
}

#ifndef BH_DB_MAX_COLS
#define BH_DB_MAX_COLS 2
#endif
template <int DIM, bool W>
struct Batch {            // U event pairs of every column, held in registers (x2: double-buffered)
    static constexpr int NCOL = DIM + (W ? 1 : 0);
#ifndef BH_U_TWO_COLS
#define BH_U_TWO_COLS 1
#endif
#ifndef BH_U_ONE_COL
#define BH_U_ONE_COL 4      // 4 measured 4% faster than 2 on C1S (1.28 vs 1.33 ms)
#endif
    static constexpr int U = NCOL == 1 ? BH_U_ONE_COL : NCOL == 2 ? BH_U_TWO_COLS : 1;   // <= 64 registers at 1024 threads
    static constexpr bool DB = NCOL <= BH_DB_MAX_COLS;   // prefetch the next batch (register double buffer)
    double2 x[U][DIM];
    double2 w[U];
};

// Shared-memory layout: [sink | variable-axis tables (VSM)]; the tables start at
// each axis' tab_off.  VEC: columns are read as double2 (LDG.E.128) after `peel`
// leading events; the next batch is loaded before the current one is processed
// (register double-buffering) so each thread keeps 2*U*ncol 16-byte loads in flight.
template <int DIM, bool W, int SINK, bool VEC, int VM>
__global__ void __launch_bounds__((FillThreads<SINK, DIM, W>::v), SINK == SINK_GLOBAL ? kGlobalCtas : 1) k_fill(FillP p) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (gated_off(p.gate, p.gate_run)) return;          // (uniform: the whole grid exits)
    using Sink_t = typename SinkOf<SINK, W>::T;
    Sink_t sink;
    if constexpr (SINK == SINK_GLOBAL || SINK == SINK_CACHE) sink.bind(p);
    if constexpr (SINK == SINK_CACHE) sink.init(smem, p.cache_slots);
    else if constexpr (SINK == SINK_PRIV || SINK == SINK_PRIVA) sink.init(smem, p.G, p.replicas, p.wc_off);
    else sink.init(smem, p.G);
    if constexpr (SINK == SINK_PRIVA && W) sink.init_hot(p, smem);
    if constexpr (SINK == SINK_CACHE && !W && DIM <= 2) sink.init_win(p, smem, DIM);
    if constexpr (SINK == SINK_CACHE && W) sink.init_hot(p, smem);
    if constexpr (VM == 1 || VM == 3) stage_axes<DIM>(p.ax, smem);
    if constexpr (SINK != SINK_GLOBAL || VM == 1 || VM == 3) __syncthreads();

    Acc<DIM, W> acc;
    acc.zero();
    // one launch covers <= 2^30 events (host split), so pair and event indices fit in int32
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nth = gridDim.x * blockDim.x;

    if constexpr (VEC) {
        using B = Batch<DIM, W>;
        constexpr int U = B::U;
        const int base = p.peel;
        const int n = (int)p.n;
        const int npair = (n - base) >> 1;
        const double2 *xs[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) xs[a] = reinterpret_cast<const double2 *>(p.x[a] + base);
        const double2 *ws = W ? reinterpret_cast<const double2 *>(p.w + base) : nullptr;
        auto load = [&](B &bt, int q0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = q0 + u * nth;
                if (q < npair) {
#pragma unroll
                    for (int a = 0; a < DIM; ++a) bt.x[u][a] = ld_stream(xs[a] + q);
                    if (W) bt.w[u] = ld_stream(ws + q);
                }
            }
        };
        // SINK_PRIVA's warp hot-bin caches need converged full warps: with warp-uniform
        // trip counts (below) every lane reaches these reconvergence points
        constexpr bool kConverge = SINK == SINK_PRIVA;
        auto process = [&](const B &bt, int q0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = q0 + u * nth < npair;
                double x0[DIM], x1[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) { x0[a] = bt.x[u][a].x; x1[a] = bt.x[u][a].y; }
                if (kConverge) __syncwarp();
                if (ok) do_event<DIM, W, VM>(p, x0, W ? bt.w[u].x : 1.0, sink, acc, smem);
                if (kConverge) __syncwarp();
                if (ok) do_event<DIM, W, VM>(p, x1, W ? bt.w[u].y : 1.0, sink, acc, smem);
            }
        };
        const int step = U * nth;
        // Warp-uniform trip counts (load/process predicate each lane's pairs) and an explicit
        // reconvergence per batch: data-dependent branches (the variable-axis search, rare
        // exact FindBin decisions) must not leave lanes issuing the next batch's loads on
        // their own -- partial-warp loads of evict-first lines re-read DRAM (measured 2x
        // traffic and 4.5x time on C2 when the compiler dropped a reconvergence point).
        const int lane0 = tid & 31;
        if constexpr (B::DB) {
            // register double buffer: load the next batch, then process the current one
            // (a two-buffer ping-pong unroll measured 25% slower on C1S: more live registers)
            B cur, nxt;
            int q0 = tid;
            load(cur, q0);
            for (; q0 - lane0 < npair; q0 += step) {
                load(nxt, q0 + step);
                process(cur, q0);
                cur = nxt;
                __syncwarp();
            }
        } else {
            B cur;
            // per-lane trips (uniform trips + __syncwarp measured 2-3% slower on C4), except
            // for SINK_PRIVA, whose reconvergence points need every lane
            for (int q0 = tid; kConverge ? q0 - lane0 < npair : q0 < npair; q0 += step) {
                load(cur, q0);       // 3-4 columns: 48-64 B per thread in flight already
                process(cur, q0);
            }
        }
        // leading peeled events and the odd tail
        const int tail0 = base + 2 * npair;
        const int nscalar = base + (n - tail0);
        if (tid < nscalar) {
            const int i = tid < base ? tid : tail0 + (tid - base);
            double x[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) x[a] = p.x[a][i];
            do_event<DIM, W, VM>(p, x, W ? p.w[i] : 1.0, sink, acc, smem);
        }
    } else {
        for (int i = tid; i < (int)p.n; i += nth) {
            double x[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) x[a] = ld_stream(p.x[a] + i);
            do_event<DIM, W, VM>(p, x, W ? ld_stream(p.w + i) : 1.0, sink, acc, smem);
        }
    }

    if constexpr (SINK != SINK_GLOBAL) {
        sink.drain();
        __syncthreads();
        sink.flush(p, smem);
    }
    acc.finalize_unit();
    block_stats_finish<Acc<DIM, W>::K>(p, acc.s);
}

// ------------------------------------------------------------------ float32 input columns (NEXT-2)
// Same three steps on float32 coordinates/weights (RDataFrame's TH1F-style inputs,
// "different ... input data types"): each value is widened exactly to
// float64 and the float64 path follows, so the result equals bh_fill on the widened
// columns; the columns cost 4 B/event instead of 8.  Columns sharing a 16-byte phase are
// read as float4 (4 events per LDG.128) after `peel` (0-3) leading events; p.peel < 0
// selects the scalar loop (mixed phases).  CT = float or int32_t: int32 coordinate columns
// (e.g. multiplicities) widen exactly to float64 too; weights are float32 in both.
template <typename CT> struct Vec4Of;
template <> struct Vec4Of<float> { using T = float4; };
template <> struct Vec4Of<int32_t> { using T = int4; };

template <int DIM, bool W, int SINK, int VM, typename CT>
__global__ void __launch_bounds__((ThreadsOf<SINK>::v), SINK == SINK_GLOBAL ? 2 : 1) k_fill_f32(FillP p) {
    extern __shared__ __align__(16) unsigned char smem[];
    using Sink_t = typename SinkOf<SINK, W>::T;
    Sink_t sink;
    if constexpr (SINK == SINK_GLOBAL || SINK == SINK_CACHE) sink.bind(p);
    if constexpr (SINK == SINK_CACHE) sink.init(smem, p.cache_slots);
    else if constexpr (SINK == SINK_PRIV || SINK == SINK_PRIVA) sink.init(smem, p.G, p.replicas, p.wc_off);
    else sink.init(smem, p.G);
    if constexpr (VM == 1) stage_axes<DIM>(p.ax, smem);
    if constexpr (SINK != SINK_GLOBAL || VM == 1) __syncthreads();
    Acc<DIM, W> acc;
    acc.zero();
    using CV = typename Vec4Of<CT>::T;
    const CT *xs[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) xs[a] = reinterpret_cast<const CT *>(p.x[a]);
    const float *ws = reinterpret_cast<const float *>(p.w);
    const int n = (int)p.n;                       // host splits launches at 2^30 events
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    auto one = [&](int i) {
        double x[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) x[a] = (double)xs[a][i];
        do_event<DIM, W, VM>(p, x, W ? (double)ws[i] : 1.0, sink, acc, smem);
    };
    if (p.peel < 0) {
        for (int i = tid; i < n; i += nth) one(i);
    } else {
        const int base = p.peel, nq = (n - base) >> 2;
        // 16-byte vectors per column per thread in flight: one column 4, more columns 2
        // (measured: C1F 654 / 764 / 850 G events/s at 1 / 2 / 4; C2F best at 2)
#ifdef BH_F32_U
        constexpr int UF = BH_F32_U;
#else
        constexpr int UF = DIM + (W ? 1 : 0) == 1 ? 4 : 2;
#endif
        for (int q0 = tid; q0 - (tid & 31) < nq; q0 += UF * nth) {   // warp-uniform trips (see k_fill)
            __syncwarp();
            CV xv[UF][DIM];
            float4 wv[UF];
#pragma unroll
            for (int u = 0; u < UF; ++u) {
                const int q = q0 + u * nth;
                if (q < nq) {
#pragma unroll
                    for (int a = 0; a < DIM; ++a) xv[u][a] = __ldcs(reinterpret_cast<const CV *>(xs[a] + base) + q);
                    if (W) wv[u] = ld_stream(reinterpret_cast<const float4 *>(ws + base) + q);
                }
            }
#pragma unroll
            for (int u = 0; u < UF; ++u) {
                if (q0 + u * nth >= nq) continue;
                const CT *xf[DIM];
#pragma unroll
                for (int a = 0; a < DIM; ++a) xf[a] = reinterpret_cast<const CT *>(&xv[u][a]);
                const float *wf = reinterpret_cast<const float *>(&wv[u]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    double x[DIM];
#pragma unroll
                    for (int a = 0; a < DIM; ++a) x[a] = (double)xf[a][j];
                    do_event<DIM, W, VM>(p, x, W ? (double)wf[j] : 1.0, sink, acc, smem);
                }
            }
        }
        const int tail0 = base + 4 * nq, nscalar = base + (n - tail0);
        if (tid < nscalar) one(tid < base ? tid : tail0 + (tid - base));
    }
    if constexpr (SINK != SINK_GLOBAL) {
        sink.drain();
        __syncthreads();
        sink.flush(p, smem);
    }
    acc.finalize_unit();
    block_stats_finish<Acc<DIM, W>::K>(p, acc.s);
}

// ------------------------------------------------------------------ fused Filter + Define (NEXT-1)
// RDataFrame's own example filters events and defines a derived column
// before the histogram action.  Instead of materializing the derived column (a write and
// a re-read of 8 B/event), a short register program runs inside the fill: r[0..ncols) hold
// the event's columns, each op writes one register, then the axes read r[axis_reg[a]],
// the weight r[weight_reg] and the event passes iff r[filter_reg] != 0.  Only IEEE
// correctly-rounded operations exist (+ - * / sqrt, comparisons, min/max, logic), so a
// derived coordinate is bit-identical to the same expression evaluated anywhere.
constexpr int kExprRegs = 16;
constexpr int kExprOps = 32;
enum ExprOp : int32_t {
    EX_CONST = 0, EX_COPY, EX_ADD, EX_SUB, EX_MUL, EX_DIV, EX_SQRT, EX_ABS, EX_NEG, EX_MIN, EX_MAX,
    EX_LT, EX_LE, EX_GT, EX_GE, EX_EQ, EX_NE, EX_AND, EX_OR, EX_NOT, EX_SELECT, EX_COUNT
};
struct ExprIns { int32_t op, dst, a, b, c, pad; double imm; };
struct ExprP {
    int32_t ncols, nops, weight_reg, filter_reg;
    int32_t axis_reg[kMaxDim];
    const double *cols[kExprRegs];
    ExprIns ins[kExprOps];
};

__device__ __forceinline__ void run_expr(const ExprP &e, double (&r)[kExprRegs]) {
    for (int k = 0; k < e.nops; ++k) {          // uniform across the warp: no divergence
        const ExprIns I = e.ins[k];
        const double a = r[I.a], b = r[I.b];
        double v;
        switch (I.op) {
        case EX_CONST: v = I.imm; break;
        case EX_COPY: v = a; break;
        case EX_ADD: v = __dadd_rn(a, b); break;
        case EX_SUB: v = __dsub_rn(a, b); break;
        case EX_MUL: v = __dmul_rn(a, b); break;
        case EX_DIV: v = __ddiv_rn(a, b); break;
        case EX_SQRT: v = __dsqrt_rn(a); break;
        case EX_ABS: v = fabs(a); break;
        case EX_NEG: v = -a; break;
        case EX_MIN: v = fmin(a, b); break;
        case EX_MAX: v = fmax(a, b); break;
        case EX_LT: v = a < b; break;
        case EX_LE: v = a <= b; break;
        case EX_GT: v = a > b; break;
        case EX_GE: v = a >= b; break;
        case EX_EQ: v = a == b; break;
        case EX_NE: v = a != b; break;
        case EX_AND: v = (a != 0.0) && (b != 0.0); break;
        case EX_OR: v = (a != 0.0) || (b != 0.0); break;
        case EX_NOT: v = !(a != 0.0); break;
        default: v = (a != 0.0) ? b : r[I.c]; break;   // EX_SELECT
        }
        r[I.dst] = v;
    }
}

// Same sinks and stats as k_fill; entries += number of events that pass the filter.
template <int DIM, bool W, int SINK, int VM>
__global__ void __launch_bounds__(ThreadsOf<SINK>::v, SINK == SINK_GLOBAL ? 2 : 1)
    k_fill_expr(FillP p, const __grid_constant__ ExprP e) {
    extern __shared__ __align__(16) unsigned char smem[];
    using Sink_t = typename SinkOf<SINK, W>::T;
    Sink_t sink;
    if constexpr (SINK == SINK_GLOBAL || SINK == SINK_CACHE) sink.bind(p);
    if constexpr (SINK == SINK_CACHE) sink.init(smem, p.cache_slots);
    else if constexpr (SINK == SINK_PRIV || SINK == SINK_PRIVA) sink.init(smem, p.G, p.replicas, p.wc_off);
    else sink.init(smem, p.G);
    if constexpr (VM == 1) stage_axes<DIM>(p.ax, smem);
    if constexpr (SINK != SINK_GLOBAL || VM == 1) __syncthreads();
    Acc<DIM, W> acc;
    acc.zero();
    unsigned int passed = 0;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += nth) {
        double r[kExprRegs];
#pragma unroll
        for (int c = 0; c < kExprRegs; ++c) r[c] = c < e.ncols ? ld_stream(e.cols[c] + i) : 0.0;
        run_expr(e, r);
        if (e.filter_reg >= 0 && !(r[e.filter_reg] != 0.0)) continue;   // Filter
        ++passed;
        double x[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) x[a] = r[e.axis_reg[a]];
        do_event<DIM, W, VM>(p, x, W ? r[e.weight_reg] : 1.0, sink, acc, smem);
    }
    // entries: passing events (order-independent integer adds)
    for (int o = 16; o > 0; o >>= 1) passed += __shfl_xor_sync(0xffffffffu, passed, o);
    if ((threadIdx.x & 31) == 0 && passed) atomicAdd(p.entries, (unsigned long long)passed);
    if constexpr (SINK != SINK_GLOBAL) {
        sink.drain();
        __syncthreads();
        sink.flush(p, smem);
    }
    acc.finalize_unit();
    block_stats_finish<Acc<DIM, W>::K>(p, acc.s);   // p.entries_add == 0 here
}

// ------------------------------------------------------------------ exact, deterministic weighted mode (NEXT-3)
// Per launch: E = exponent of max|w| (finite weights), then every weight becomes the
// integer m = RN(w * 2^(96-E)) (|m| < 2^96; exact unless |w| < 2^(E-43)), split into four
// signed 24-bit chunks.  Lanes of a warp holding the same bin sum their chunks exactly
// with __reduce_add_sync (|group sum| < 2^29), and the group leader adds them with integer
// RED.64 into per-bin int64 limbs (weights 2^0, 2^24, 2^48, 2^72) -- order independent, so
// the per-bin sums are bitwise reproducible -- and the limbs are folded back once per
// launch: sumw[g] += RN(sum m) * 2^(E-96), the correctly rounded value of the exact sum
// of the scaled weights.  Same for w*w with its own exponent.  A launch has <= 2^30
// events, so a limb stays below 2^54.  Non-finite weights take the ordinary float64
// atomics (NaN/inf propagate as in any float sum).
constexpr int kLimbs = 4;                      // per quantity; 8 per bin (sumw, sumw2)

#ifndef BH_FILL_TU   // kernels below the fill templates are compiled once, in bhist.cu

__global__ void k_wmax(const double *__restrict__ w, int64_t n, unsigned long long *maxbits) {
    unsigned long long m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double a = fabs(w[i]);
        if (a <= 1.7976931348623157e308) m = max(m, (unsigned long long)__double_as_longlong(a));   // finite
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(maxbits, m);      // |w| bit patterns order like values
}

__device__ __forceinline__ int exact_exp(unsigned long long maxbits) {   // max|w| < 2^E
    int e = 0;
    if (maxbits) frexp(__longlong_as_double((long long)maxbits), &e);
    return e;
}

// the four signed 24-bit chunks of RN(v * 2^(96-e)), low first
__device__ __forceinline__ void exact_chunks(double v, int e, int (&c)[kLimbs]) {
    double r = ldexp(v, 96 - e);
#pragma unroll
    for (int k = kLimbs - 1; k >= 1; --k) {
        const double hk = trunc(ldexp(r, -24 * k));
        r -= ldexp(hk, 24 * k);                  // exact: removes the top bits of r's expansion
        c[k] = (int)hk;
    }
    c[0] = (int)rint(r);                         // the only rounding (weights < 2^(e-43))
}

template <int DIM>
__global__ void __launch_bounds__(512, 2) k_fill_exact(FillP p, long long *limbs, const unsigned long long *maxbits) {
    const int e1 = exact_exp(*maxbits);
    const int e2 = 2 * e1 + 1;                      // max RN(w*w) < 2^(2 e1) <= 2^e2
    Acc<DIM, true> acc;
    acc.zero();
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = ((p.n + nth - 1) / nth) * nth;     // whole warps run every iteration
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += nth) {
        const bool valid = i < p.n;
        double x[DIM];
        int g = 0, mul = 1;
        bool inr = valid;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            x[a] = valid ? ld_stream(p.x[a] + i) : 0.0;
            const int b = find_bin(p.ax[a], x[a]);
            inr &= (b >= 1) & (b <= p.ax[a].n);
            g += b * mul;
            if (a + 1 < DIM) mul = (a == 0) ? p.st1 : p.st2;
        }
        const double w = valid ? ld_stream(p.w + i) : 0.0, w2 = w * w;
        const bool fin = fabs(w) <= 1.7976931348623157e308 && fabs(w2) <= 1.7976931348623157e308;
        if (valid && !fin) {
            atomicAdd(p.sw + 2 * (size_t)g, w);
            atomicAdd(p.sw + 2 * (size_t)g + 1, w2);
        }
        const bool use = valid && fin;
        const unsigned act = __ballot_sync(0xffffffffu, use);
        if (use) {
            int c1[kLimbs], c2[kLimbs];
            exact_chunks(w, e1, c1);
            exact_chunks(w2, e2, c2);
            const unsigned peers = __match_any_sync(act, g);
            const bool dup = __any_sync(act, __popc(peers) > 1);
            const bool leader = (int)(threadIdx.x & 31) == __ffs(peers) - 1;
            long long *lb = limbs + 2 * kLimbs * (size_t)g;
#pragma unroll
            for (int k = 0; k < kLimbs; ++k) {
                int s1 = c1[k], s2 = c2[k];
                if (dup) {                               // equal bins in the warp: exact group sums
                    s1 = (int)__reduce_add_sync(peers, (unsigned)c1[k]);
                    s2 = (int)__reduce_add_sync(peers, (unsigned)c2[k]);
                }
                if (leader) {
                    if (s1) atomicAdd(reinterpret_cast<unsigned long long *>(lb + k), (unsigned long long)(long long)s1);
                    if (s2) atomicAdd(reinterpret_cast<unsigned long long *>(lb + kLimbs + k),
                                      (unsigned long long)(long long)s2);
                }
            }
        }
        if (inr) acc.add(x, w);
    }
    block_stats_finish<Acc<DIM, true>::K>(p, acc.s);
}

__device__ __forceinline__ double fold_limbs(long long *l, int e) {
    __int128 v = 0;
#pragma unroll
    for (int k = kLimbs - 1; k >= 0; --k) v = (v << 24) + (__int128)l[k];
#pragma unroll
    for (int k = 0; k < kLimbs; ++k) l[k] = 0;
    return ldexp((double)v, e - 96);
}

__global__ void k_exact_fold(int G, long long *limbs, const unsigned long long *maxbits, double *sw) {
    const int e1 = exact_exp(*maxbits), e2 = 2 * e1 + 1;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
        long long *l = limbs + 2 * kLimbs * (size_t)g;
        if (l[0] | l[1] | l[2] | l[3]) sw[2 * (size_t)g] += fold_limbs(l, e1);
        if (l[4] | l[5] | l[6] | l[7]) sw[2 * (size_t)g + 1] += fold_limbs(l + kLimbs, e2);
    }
}

#endif  // BH_FILL_TU

// ------------------------------------------------------------------ fused multi-histogram fill (C5)
// One pass over a set of columns feeding several histograms (the paper's future
// work "multiple histograms from different columns in one pass"; RDataFrame
// runs all actions of a dataframe in one event loop).  Each column byte is
// read once per pass; each histogram runs the same three steps as k_fill.  The host
// planner (bh_fill_multi) puts histograms whose private state is large in passes of
// their own (k_fill) and fuses the small ones here: all their bins are privatized in
// shared memory (u32 counts / double2 (sumw, sumw2) with 128-bit CAS), equal bins
// are aggregated across the warp first (hot bins, e.g. a Cauchy-peaked column), and
// each thread keeps its statistics in a private shared-memory column
// (acc[stat][thread], conflict-free), since up to 8 x 11 sums do not fit in registers.
constexpr int kMaxHist = 8;
constexpr int kMaxCols = 8;
constexpr int kMultiThreads = 1024;

struct MultiH {
    int32_t dim;
    int32_t weighted;
    int32_t col[kMaxDim];
    AxisP ax[kMaxDim];
    int32_t st1, st2;
    int32_t G, K;
    int32_t stat_off;                    // first index of this histogram's stats in the flat list
    int32_t smem_off;                    // byte offset of the privatized bins
    unsigned long long *count;
    double *sw, *stats, *partials;      // sw: interleaved (sum w, sum w^2) [2G]
    unsigned long long *entries;
};

struct MultiP {
    int64_t n;
    int32_t nh, ncols, nstats;
    int32_t acc_off;                     // byte offset of acc[nstats][blockDim.x]
    int32_t agg_unit;                    // aggregate equal bins across the warp for unit weights too
    const double *cols[kMaxCols];
    const double *w;
    unsigned int *counter;               // ticket of histogram 0
    MultiH h[kMaxHist];
};

#ifndef BH_FILL_TU
__device__ __forceinline__ double pick(const double (&x)[kMaxCols], int c) {
    double v = x[0];
#pragma unroll
    for (int k = 1; k < kMaxCols; ++k) v = (c == k) ? x[k] : v;   // selects, no local memory
    return v;
}

// Bin add for one event of histogram H with warp aggregation: lanes with equal bins
// elect a leader that adds the group's count (popc) or (sum w, sum w*w) once.
__device__ __forceinline__ void multi_add(const MultiH &H, unsigned char *smem, bool valid, int g, double w,
                                          bool agg_unit) {
    if (!H.weighted && !agg_unit) {          // native u32 ATOMS; the hardware serializes equal addresses
        if (valid) atomicAdd(reinterpret_cast<uint32_t *>(smem + H.smem_off) + g, 1u);
        return;
    }
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const unsigned peers = __match_any_sync(act, g);
    const int lane = (int)(threadIdx.x & 31);
    const int leader = __ffs(peers) - 1;
    if (H.weighted) {
        const int rounds = __reduce_max_sync(act, (unsigned)__popc(peers));
        double s1 = 0.0, s2 = 0.0;
        unsigned m = peers;
        for (int k = 0; k < rounds; ++k) {
            const int src = m ? __ffs(m) - 1 : lane;
            const double v = __shfl_sync(act, w, src);
            if (m) { s1 += v; s2 = fma(v, v, s2); m &= m - 1; }
        }
        if (lane == leader) add2_shared(reinterpret_cast<double2 *>(smem + H.smem_off) + g, s1, s2);
    } else if (lane == leader) {
        atomicAdd(reinterpret_cast<uint32_t *>(smem + H.smem_off) + g, (uint32_t)__popc(peers));
    }
}

__global__ void __launch_bounds__(1024, 1) k_fill_multi(const __grid_constant__ MultiP p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ bool last;
    double *acc = reinterpret_cast<double *>(smem + p.acc_off);     // acc[k * blockDim.x + tid]
    const int T = blockDim.x;
    for (int hh = 0; hh < p.nh; ++hh) {
        const MultiH &H = p.h[hh];
        if (H.weighted) {
            double2 *d = reinterpret_cast<double2 *>(smem + H.smem_off);
            for (int i = threadIdx.x; i < H.G; i += T) d[i] = make_double2(0.0, 0.0);
        } else {
            uint32_t *c = reinterpret_cast<uint32_t *>(smem + H.smem_off);
            for (int i = threadIdx.x; i < H.G; i += T) c[i] = 0u;
        }
        for (int a = 0; a < H.dim; ++a)
            if (H.ax[a].var && H.ax[a].tab_off >= 0) stage_axes<1>(&H.ax[a], smem);
    }
    for (int k = 0; k < p.nstats; ++k) acc[k * T + threadIdx.x] = 0.0;
    __syncthreads();

    const int64_t nth = (int64_t)gridDim.x * T;
    const int64_t n_round = ((p.n + nth - 1) / nth) * nth;     // every lane runs every iteration
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n_round; i += nth) {
        const bool valid = i < p.n;
        double x[kMaxCols];
#pragma unroll
        for (int c = 0; c < kMaxCols; ++c) x[c] = (c < p.ncols && valid) ? ld_stream(p.cols[c] + i) : 0.0;
        const double wv = (valid && p.w) ? ld_stream(p.w + i) : 1.0;
        for (int hh = 0; hh < p.nh; ++hh) {
            const MultiH &H = p.h[hh];
            const double w = H.weighted ? wv : 1.0;
            double xa[kMaxDim] = {0.0, 0.0, 0.0};
            int g = 0, mul = 1;
            bool inr = true;
            for (int a = 0; a < H.dim; ++a) {
                xa[a] = pick(x, H.col[a]);
                const AxisP &A = H.ax[a];
                int b;
                if (!A.var) b = find_bin_fixed(A, xa[a]);
                else if (A.tab_off >= 0)
                    b = find_bin_var_smem_any(A, xa[a], smem + A.tab_off);
                else b = find_bin_var_global(A, xa[a]);
                inr &= (b >= 1) & (b <= A.n);
                g += b * mul;
                mul = (a == 0) ? H.st1 : H.st2;
            }
            multi_add(H, smem, valid, g, w, p.agg_unit != 0);   // step (2)
            if (valid && inr) {                              // step (3)
                double *ac = acc + (size_t)H.stat_off * T + threadIdx.x;
                const double wx = w * xa[0];
                ac[0] += w;
                ac[T] = fma(w, w, ac[T]);
                ac[2 * T] += wx;
                ac[3 * T] = fma(wx, xa[0], ac[3 * T]);
                if (H.dim >= 2) {
                    const double wy = w * xa[1];
                    ac[4 * T] += wy;
                    ac[5 * T] = fma(wy, xa[1], ac[5 * T]);
                    ac[6 * T] = fma(wx, xa[1], ac[6 * T]);
                    if (H.dim == 3) {
                        const double wz = w * xa[2];
                        ac[7 * T] += wz;
                        ac[8 * T] = fma(wz, xa[2], ac[8 * T]);
                        ac[9 * T] = fma(wx, xa[2], ac[9 * T]);
                        ac[10 * T] = fma(wy, xa[2], ac[10 * T]);
                    }
                }
            }
        }
    }

    // merge stage: privatized bins -> global
    __syncthreads();
    for (int hh = 0; hh < p.nh; ++hh) {
        const MultiH &H = p.h[hh];
        if (H.weighted) {
            const double *d = reinterpret_cast<const double *>(smem + H.smem_off);
            for (int i = threadIdx.x; i < 2 * H.G; i += T)
                if (d[i] != 0.0) red_f64(H.sw + i, d[i]);
        } else {
            const uint32_t *c = reinterpret_cast<const uint32_t *>(smem + H.smem_off);
            for (int i = threadIdx.x; i < H.G; i += T)
                if (c[i]) red_u64(H.count + i, (unsigned long long)c[i]);
        }
    }
    // stats: per-thread columns -> block partials (fixed order) -> last CTA, fixed order
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = T >> 5;
    for (int k = warp; k < p.nstats; k += nw) {
        double t = 0.0;
        for (int j = lane; j < T; j += 32) t += acc[k * T + j];
        t = warp_sum_fixed(t);
        if (lane == 0) {
            int hh = 0;
            while (hh + 1 < p.nh && p.h[hh + 1].stat_off <= k) ++hh;
            const MultiH &H = p.h[hh];
            H.partials[(size_t)blockIdx.x * H.K + (k - H.stat_off)] = t;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(p.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x < p.nstats) {
        int hh = 0;
        while (hh + 1 < p.nh && p.h[hh + 1].stat_off <= (int)threadIdx.x) ++hh;
        const MultiH &H = p.h[hh];
        const int k = threadIdx.x - H.stat_off;
        double t = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(H.partials + (size_t)b * H.K + k);
        H.stats[k] += t;
    }
    if (threadIdx.x < p.nh) *p.h[threadIdx.x].entries += (unsigned long long)p.n;
    if (threadIdx.x == 0) *p.counter = 0u;
}

// ------------------------------------------------------------------ auxiliary kernels
// guide[c] = #{interior i in [1, n-1] : cell(e_i) < c}, c = 0..gcells (cell is monotone in i).
__global__ void k_build_guide(AxisP a, uint32_t *guide) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > a.gcells) return;
    int lo = 1, hi = a.n;            // first interior i with cell(e_i) >= c, in [1, n]
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (guide_cell(a, a.e[m]) < c) lo = m + 1; else hi = m;
    }
    guide[c] = (uint32_t)(lo - 1);
}

__global__ void k_edges_f32(const double *e, int n, float *e32) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) e32[i] = __double2float_rn(e[i]);
}

// Shared-memory image of a variable axis: [e32 (n+1 floats, padded to 16 B) | guide in
// mode a.g16]; the packed mode stores guide[c] << 2 | min(guide[c+1] - guide[c], 3).
__global__ void k_table_image(AxisP a, const uint32_t *guide, unsigned char *img) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (a.g16 >= 3) {                    // compact: one word per cell, no float32 edges
        if (i <= a.gcells) {
            const uint32_t lo = guide[i];
            const uint32_t cnt = i < a.gcells ? guide[i + 1] - lo : 0u;
            uint32_t v = lo | (cnt < 3u ? cnt : 3u) << 14;
            int q;
            auto qpos = [&](double e) { if (a.g16 == 4) compact_cell<true>(a, e, q); else compact_cell<false>(a, e, q); };
            if (cnt >= 1) { qpos(a.e[lo + 1]); v |= (uint32_t)q << 16; }
            if (cnt >= 2) { qpos(a.e[lo + 2]); v |= (uint32_t)q << 24; }
            reinterpret_cast<uint32_t *>(img)[i] = v;
        }
        return;
    }
    float *e32 = reinterpret_cast<float *>(img);
    if (i <= a.n) e32[i] = __double2float_rn(a.e[i]);
    unsigned char *gt = img + ((4 * (a.n + 1) + 15) & ~15);
    if (i <= a.gcells) {
        const uint32_t g0 = guide[i];
        if (a.g16 == 2) {
            const uint32_t d = i < a.gcells ? guide[i + 1] - g0 : 0u;
            reinterpret_cast<uint16_t *>(gt)[i] = (uint16_t)((g0 << 2) | (d < 3u ? d : 3u));
        } else if (a.g16 == 1) {
            reinterpret_cast<uint16_t *>(gt)[i] = (uint16_t)g0;
        } else {
            reinterpret_cast<uint32_t *>(gt)[i] = g0;
        }
    }
}

#endif  // BH_FILL_TU

// Per-event global bins through the same FindBin code the fills run: VM 1 / 3 stage the
// variable-axis tables in shared memory exactly as k_fill does (float32-edge or compact
// search), VM 2 searches the float64 edges in global memory, VM 0 has fixed axes only.
template <int DIM, int VM>
__global__ void k_find_bins(FillP p, int32_t *out) {
    extern __shared__ __align__(16) unsigned char smem[];
    if constexpr (VM == 1 || VM == 3) {
        stage_axes<DIM>(p.ax, smem);
        __syncthreads();
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
        int g = 0, mul = 1;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            g += find_bin<VM, DIM == 1 && VM != 0>(p.ax[a], p.x[a][i], smem) * mul;
            if (a + 1 < DIM) mul = (a == 0) ? p.st1 : p.st2;
        }
        out[i] = g;
    }
}

#ifndef BH_FILL_TU
// bh_reset: bins, sums of w^2, stats and entries to zero in ONE launch (five memsets cost
// ~2-3 us of launch overhead each, a third of a 1e6-event fill step); 16-byte stores.
__global__ void k_reset(int G, unsigned long long *count, double *sw, double *stats,
                        unsigned long long *entries) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t h = G / 2;                  // the arrays are 16-byte aligned (cudaMalloc)
    for (int64_t i = t0; i < h; i += stride) {
        reinterpret_cast<ulonglong2 *>(count)[i] = make_ulonglong2(0ull, 0ull);
        reinterpret_cast<double2 *>(sw)[2 * i] = make_double2(0.0, 0.0);
        reinterpret_cast<double2 *>(sw)[2 * i + 1] = make_double2(0.0, 0.0);
    }
    if (t0 == 0 && (G & 1)) {
        count[G - 1] = 0ull;
        reinterpret_cast<double2 *>(sw)[G - 1] = make_double2(0.0, 0.0);
    }
    if (t0 < 16) stats[t0] = 0.0;
    if (t0 == 0) *entries = 0ull;
}

// packed = [content | sumw2 | stats | entries], content = count + sumw.
__global__ void k_pack(int G, int K, const unsigned long long *count, const double *sw,
                       const double *stats, const unsigned long long *entries, double *out) {
    const int64_t tot = 2 * (int64_t)G + K + 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        double v;
        if (i < G) v = (double)count[i] + sw[2 * i];
        else if (i < 2 * (int64_t)G) v = (double)count[i - G] + sw[2 * (i - G) + 1];
        else if (i < 2 * (int64_t)G + K) v = stats[i - 2 * G];
        else v = (double)*entries;
        out[i] = v;
    }
}

__global__ void k_unpack(int G, int K, unsigned long long *count, double *sw, double *stats,
                         unsigned long long *entries, const double *in) {
    const int64_t tot = 2 * (int64_t)G + K + 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = in[i];
        if (i < G) { count[i] = 0ull; sw[2 * i] = v; }
        else if (i < 2 * (int64_t)G) sw[2 * (i - G) + 1] = v;
        else if (i < 2 * (int64_t)G + K) stats[i - 2 * G] = v;
        else *entries = (unsigned long long)v;
    }
}

// bh_read_as: the packed float64 [content | sumw2] of bh_pack narrowed once (reading R18):
// float32 by round-to-nearest, int32 (unit-weight counts) saturated at INT32_MAX.
// (Unit-weight contents are integers < 2^53, exact in the packed float64.)
__global__ void k_narrow(int G, int type, const double *packed, void *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * (int64_t)G;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = packed[i];
        if (type == 1) reinterpret_cast<float *>(out)[i] = __double2float_rn(v);
        else reinterpret_cast<int32_t *>(out)[i] = v >= 2147483647.0 ? 2147483647 : (int32_t)v;
    }
}

// Several histograms packed into one buffer for ONE collective per step:
// histogram i occupies [off_i, off_i + len_i) with the bh_pack layout, or, when unit_i is
// set (a unit-weight-only state: sumw2 == content), [content(G) | stats(K) | entries].
struct PackDesc {
    int64_t off;
    int32_t G, K, unit;
    unsigned long long *count;
    double *sw, *stats;                          // sw: interleaved (sum w, sum w^2) [2G]
    unsigned long long *entries;
};
constexpr int kMaxPack = 8;
struct PackMultiP {
    int32_t nh;
    int64_t total;
    PackDesc d[kMaxPack];
};

__device__ __forceinline__ int pack_find(const PackMultiP &p, int64_t i) {
    int k = 0;
    while (k + 1 < p.nh && p.d[k + 1].off <= i) ++k;
    return k;
}

__global__ void k_pack_multi(const __grid_constant__ PackMultiP p, double *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.total; i += (int64_t)gridDim.x * blockDim.x) {
        const PackDesc &D = p.d[pack_find(p, i)];
        const int64_t j = i - D.off, G = D.G;
        const int64_t s2 = D.unit ? 0 : G;           // length of the sumw2 section
        double v;
        if (j < G) v = (double)D.count[j] + D.sw[2 * j];
        else if (j < G + s2) v = (double)D.count[j - G] + D.sw[2 * (j - G) + 1];
        else if (j < G + s2 + D.K) v = D.stats[j - G - s2];
        else v = (double)*D.entries;
        out[i] = v;
    }
}

__global__ void k_unpack_multi(const __grid_constant__ PackMultiP p, const double *in) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.total; i += (int64_t)gridDim.x * blockDim.x) {
        const PackDesc &D = p.d[pack_find(p, i)];
        const int64_t j = i - D.off, G = D.G;
        const int64_t s2 = D.unit ? 0 : G;
        const double v = in[i];
        if (j < G) {
            D.count[j] = 0ull;
            D.sw[2 * j] = v;
            if (D.unit) D.sw[2 * j + 1] = v;         // unit weights: sum w^2 == count
        } else if (j < G + s2) D.sw[2 * (j - G) + 1] = v;
        else if (j < G + s2 + D.K) D.stats[j - G - s2] = v;
        else *D.entries = (unsigned long long)v;
    }
}

#endif  // BH_FILL_TU

}  // namespace bh
