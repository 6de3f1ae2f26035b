// bhist.cu — host side of libbhist: the C ABI of include/bhist.h.
//
// Owns per-histogram device state (RHnCUDA analogue: "keeps track of
// device allocations and contains a Fill method"), validates axes, builds the
// variable-axis guide tables, chooses the fill strategy and launch shape, and
// runs the pinned double-buffered host->device path.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/bhist.h"
#include "bhist_launch.cuh"
#include "bhist_state.h"

using namespace bh;

namespace {

thread_local std::string g_err;

bh_status fail(bh_status st, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
bh_status fail(bh_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) return fail(BH_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                           __FILE__, __LINE__);                                    \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace



namespace {

size_t align16(size_t b);
size_t axis_table_bytes(const AxisP &a);
#ifndef BH_SORT_PB_UNIT
#define BH_SORT_PB_UNIT 15
#endif
int sort_pb(bool weighted) { return weighted ? 13 : BH_SORT_PB_UNIT; }   // 2^pb bins = 128 KB of shared memory
int64_t sort_partitions(const bh_hist *h, bool weighted) {
    return (h->G + (int64_t(1) << sort_pb(weighted)) - 1) >> sort_pb(weighted);
}
constexpr size_t kStaticSmemReserve = 4096;   // block_stats_finish scratch + driver reserve

// AUTO: privatize the bins in shared memory whenever they fit next to the reserve
// (variable-axis tables then go to smem only if they also fit); otherwise CACHE.
int resolve_strategy(const bh_hist *h, bool weighted) {
    // EXACT only changes weighted fills of bh_fill / bh_fill_host (fill_exact below)
    if (h->strategy == BH_STRATEGY_SORT)     // weighted partitions are 4x smaller
        return sort_partitions(h, weighted) <= kPartMaxP ? BH_STRATEGY_SORT : BH_STRATEGY_CACHE;
    const size_t priv = (weighted ? 16 : 4) * (size_t)h->G;
    // forced PRIV is accepted when the unit-weight bins fit (bh_set_strategy); weighted
    // cells are 4x larger, so a weighted fill that cannot hold them uses CACHE instead
    if (h->strategy == BH_STRATEGY_PRIV && priv + kStaticSmemReserve > h->smem_optin) return BH_STRATEGY_CACHE;
    if (h->strategy != BH_STRATEGY_AUTO && h->strategy != BH_STRATEGY_EXACT) return h->strategy;
    if (priv + kStaticSmemReserve <= h->smem_optin) return BH_STRATEGY_PRIV;
    // large bin spaces: shared-memory cache of the hottest bins in front of L2 atomics
    // (as fast as plain GLOBAL on uniform data, 30x faster on the peaked C4 shape).
    // SORT is faster on uniform data but not on peaked data, so it is opt-in.
    return BH_STRATEGY_CACHE;
}

// kernels without a SORT variant (float32 columns, fill_expr) use CACHE instead
int resolve_one_pass(const bh_hist *h, bool weighted) {
    const int s = resolve_strategy(h, weighted);
    return s == BH_STRATEGY_SORT ? BH_STRATEGY_CACHE : s;
}

int cache_slots_for(bool weighted) {
    if (const char *env = getenv(weighted ? "BHIST_CACHE_SLOTS_W" : "BHIST_CACHE_SLOTS_U")) return atoi(env);  // A/B
    return weighted ? 8192 : 16384;      // measured: C3w 3.82 -> 3.43 ms from 4096 weighted slots
}

size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

size_t sink_bytes(const bh_hist *h, int strategy, bool weighted, int slots = 0) {
    if (strategy == BH_STRATEGY_PRIV) return align16(weighted ? 16 * (size_t)h->G : 4 * (size_t)h->G);
    if (strategy == BH_STRATEGY_CACHE) {
        const size_t S = slots > 0 ? slots : cache_slots_for(weighted);
        return S * 4 + (weighted ? 16 * S : 4 * S);
    }
    return 0;
}

// Bytes of shared memory the variable-axis tables take (float32 edges + guide).
size_t axis_table_bytes(const AxisP &a) {
    if (!a.var) return 0;
    if (a.g16 >= 3) return align16(4 * (size_t)(a.gcells + 1));
    return align16(4 * (size_t)(a.n + 1)) + align16((a.g16 ? 2 : 4) * (size_t)(a.gcells + 1));
}


FillP make_params(const bh_hist *h, int64_t n, const double *const *coords, const double *w) {
    FillP p{};
    p.n = n;
    for (int a = 0; a < h->dim; ++a) { p.x[a] = coords[a]; p.ax[a] = h->ax[a]; }
    p.w = w;
    p.st1 = h->st1;
    p.st2 = h->st2;
    p.G = (int32_t)h->G;
    p.K = h->K;
    p.count = h->count;
    p.sw = h->sw;
    p.partials = h->partials;
    p.counter = h->counter;
    p.stats = h->stats;
    p.entries = h->entries;
    p.entries_add = n;
    p.wc_off = -1;
    p.hot = nullptr;
    p.hot_off = -1;
    p.win = nullptr;
    p.win_off = -1;
    return p;
}

int threads_of(int strategy, bool weighted, int dim = 0) {     // dim: k_fill's FillThreads rule
    if (strategy == BH_STRATEGY_CACHE && weighted && dim == 3) return 768;
    return strategy == BH_STRATEGY_GLOBAL ? kThreadsGlobal : kThreadsSmem;
}
int resident_blocks(int strategy) { return strategy == BH_STRATEGY_GLOBAL ? kGlobalCtas : 1; }

// Shared-memory plan of one fill: strategy, variable-axis tables (VSM), PRIV replicas.
struct FillPlan {
    LaunchCfg c{};
    AxisP ax[kMaxDim];
    int replicas = 1;
    int wc_off = -1;     // weighted PRIV: per-warp hot-bin caches (collision-adaptive sink)
};

// Small fills (e.g. the paper's 32768-event bulks) cannot amortize PRIV's
// per-CTA zeroing and flushing of all G bins: below ~2 G events per SM, AUTO sends them
// through CACHE (warp-aggregated, hot-bin safe) instead.
bool small_fill(const bh_hist *h, int64_t n) { return n < 2 * h->G * (int64_t)h->nsm; }

bh_status plan_fill(const bh_hist *h, bool weighted, FillPlan &pl, int64_t n, size_t reserve = 0, int force = -1,
                    int slots = 0) {
    LaunchCfg &c = pl.c;
    c.weighted = weighted;
    c.strategy = force >= 0 ? force : resolve_one_pass(h, c.weighted);
    if (force < 0 && c.strategy == BH_STRATEGY_PRIV && (h->strategy == BH_STRATEGY_AUTO || h->strategy == BH_STRATEGY_EXACT) &&
        small_fill(h, n))
        c.strategy = BH_STRATEGY_CACHE;
    size_t sink = sink_bytes(h, c.strategy, c.weighted, slots);
    // variable-axis tables go to shared memory behind the sink when they fit
    size_t tabs = 0;
    for (int a = 0; a < h->dim; ++a) {
        pl.ax[a] = h->ax[a];
        if (pl.ax[a].var) {
            pl.ax[a].tab_off = (int32_t)(sink + tabs);
            tabs += axis_table_bytes(pl.ax[a]);
        }
    }
    c.vsm = tabs > 0 && sink + tabs + reserve + kStaticSmemReserve <= h->smem_optin;
    c.vm = tabs == 0 ? 0 : (c.vsm ? 1 : 2);
    if (c.vm == 1) {                     // every variable axis compact: the specialized search
        bool all3 = true;
        for (int a = 0; a < h->dim; ++a) all3 &= !h->ax[a].var || h->ax[a].g16 == 3;
        if (all3) c.vm = 3;
    }
    // PRIV: replicate the private bins into the spare shared memory (up to one copy
    // per warp) so hot bins are not contended across warps
    pl.replicas = 1;
    pl.wc_off = -1;
    size_t wcb = 0;
    if (c.strategy == BH_STRATEGY_PRIV) {
        if (sink + reserve + kStaticSmemReserve > h->smem_optin)
            return fail(BH_EINVAL, "strategy %d needs %zu B of shared memory (device max %zu)", c.strategy,
                        sink + reserve, h->smem_optin);
        size_t spare = h->smem_optin - kStaticSmemReserve - reserve - (c.vsm ? tabs : 0);
        const int cap = threads_of(c.strategy, c.weighted) / 32;
        // weighted fills get the collision-adaptive sink with per-warp hot-bin caches when
        // they fit, except a single replica next to variable-axis tables (C2's shape: the
        // spread-out fill measured fastest with the plain CAS sink)
        bool has_var = false;
        for (int a = 0; a < h->dim; ++a) has_var |= h->ax[a].var != 0;
        const size_t reps0 = spare / std::max<size_t>(sink, 1);
        const size_t wc_need = (size_t)kWCBytes * cap;
        if (c.weighted && spare >= sink + wc_need && (reps0 > 1 || !has_var) && !getenv("BHIST_NO_WARP_CACHE")) {
            wcb = wc_need;
            spare -= wcb;
        }
        pl.replicas = (int)std::max<size_t>(1, std::min<size_t>(cap, spare / std::max<size_t>(sink, 1)));
        const char *env = getenv("BHIST_PRIV_REPLICAS");
        if (env) pl.replicas = std::max(1, std::min(pl.replicas, atoi(env)));
        // the variable-axis tables sit behind all replicas
        for (int a = 0; a < h->dim; ++a)
            if (pl.ax[a].var) pl.ax[a].tab_off += (int32_t)((pl.replicas - 1) * sink);
        sink *= pl.replicas;
        if (wcb) pl.wc_off = (int)(sink + (c.vsm ? tabs : 0));     // behind replicas and tables
    }
    c.smem = sink + (c.vsm ? tabs : 0) + wcb;
    if (c.smem + reserve + kStaticSmemReserve > h->smem_optin)
        return fail(BH_EINVAL, "strategy %d needs %zu B of shared memory (device max %zu)", c.strategy, c.smem,
                    h->smem_optin);
    return BH_OK;
}

// Persistent grid (resident CTAs on every SM), but each block should see enough events
// to amortize zeroing + flushing its private bins.
int grid_for(const bh_hist *h, const LaunchCfg &c, int64_t m) {
    const int nt = threads_of(c.strategy, c.weighted, h->dim);
    // small fills are latency-bound: spread them over many SMs (>= 2 events per thread);
    // PRIV blocks must still amortize zeroing + flushing their private bins (>= 8 events
    // per thread and >= 4 G per block: measured best for C1's 1e6 events)
    int64_t want_per_block = (int64_t)nt * 2;
    if (c.strategy == BH_STRATEGY_PRIV) {
        static const int ept = getenv("BHIST_PRIV_EPT") ? std::max(1, atoi(getenv("BHIST_PRIV_EPT"))) : 8;  // A/B
        want_per_block = std::max<int64_t>((int64_t)nt * ept, 4 * h->G);
    }
    int64_t grid = (m + want_per_block - 1) / want_per_block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(grid, (int64_t)h->nsm * resident_blocks(c.strategy)));
}

// EXACT weighted fill: max|w| -> integer-limb RED.64 fill -> fold (see k_fill_exact).
bh_status fill_exact(bh_hist *h, int64_t n, const double *const *coords, const double *w, cudaStream_t s) {
    if (!h->limbs) {
        if (cudaMalloc(reinterpret_cast<void **>(&h->limbs), sizeof(long long) * 2 * kLimbs * h->G) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void **>(&h->maxbits), sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            return fail(BH_ENOMEM, "exact-mode limbs allocation failed");
        }
        CUDA_TRY(cudaMemsetAsync(h->limbs, 0, sizeof(long long) * 2 * kLimbs * h->G, s));
    }
    const int64_t kMaxLaunch = int64_t(1) << 30;   // limb sums stay below 2^54
    for (int64_t off = 0; off < n; off += kMaxLaunch) {
        const int64_t m = std::min(kMaxLaunch, n - off);
        const double *cs[kMaxDim] = {};
        for (int a = 0; a < h->dim; ++a) cs[a] = coords[a] + off;
        FillP p = make_params(h, m, cs, w + off);
        CUDA_TRY(cudaMemsetAsync(h->maxbits, 0, sizeof(unsigned long long), s));
        const int g1 = (int)std::min<int64_t>((m + 255) / 256, (int64_t)h->nsm * 8);
        k_wmax<<<g1, 256, 0, s>>>(w + off, m, h->maxbits);
        const int g2 = (int)std::min<int64_t>((m + 511) / 512, (int64_t)h->nsm * 2);
        switch (h->dim) {
        case 1: k_fill_exact<1><<<g2, 512, 0, s>>>(p, h->limbs, h->maxbits); break;
        case 2: k_fill_exact<2><<<g2, 512, 0, s>>>(p, h->limbs, h->maxbits); break;
        default: k_fill_exact<3><<<g2, 512, 0, s>>>(p, h->limbs, h->maxbits); break;
        }
        const int g3 = (int)std::min<int64_t>((h->G + 255) / 256, (int64_t)h->nsm * 8);
        k_exact_fold<<<g3, 256, 0, s>>>((int)h->G, h->limbs, h->maxbits, h->sw);
        CUDA_TRY(cudaGetLastError());
        h->launches += 3;
    }
    return BH_OK;
}

// ---- SORT strategy (bhist_sort.cuh): pass 1 scatter -> plan -> pass 2 reduce, per chunk
// pad segments to RC records (pass 2 reads aligned chunks) while that costs little
int sort_rc(bool weighted, int P) { return weighted ? (P <= 512 ? 4 : 1) : (P <= 256 ? 8 : 1); }
int sort_ts(int tile, int P, int rc) { return (tile + P * (rc - 1) + 7) / 8 * 8; }

template <bool W, int RC>
cudaError_t launch_part2(const FillP &p, const PartP &q, int grid, cudaStream_t s) {
    auto kern = k_part_reduce<W, RC>;
    const int smem = ((W ? 16 : 4) << sort_pb(W)) + 4 * (2 * kReduceBatch + 1 + 32);
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void *>(kern), (size_t)smem)) return e;
    kern<<<grid, kReduceThreads, smem, s>>>(p, q);
    return cudaGetLastError();
}

// Scratch for chunks of `ev` events (grow-only; the stream is synchronized before a
// buffer that kernels may still read is freed).
bh_status part_scratch(bh_hist *h, int64_t ev, bool weighted, int P, cudaStream_t s) {
    const int tile = kPartThreads * part_ev(h->dim, weighted);
    const int64_t tiles = (ev + tile - 1) / tile;
    const int64_t nl = tiles * sort_ts(tile, P, sort_rc(weighted, P)), no = tiles * (P + 1);
    const bool grow = nl > h->part_cap_l || (weighted && nl > h->part_cap_w) || no > h->part_cap_offs || P > h->part_P;
    if (!grow) return BH_OK;
    CUDA_TRY(cudaStreamSynchronize(s));
    auto realloc = [&](void **ptr, size_t bytes) -> bool {
        if (*ptr) cudaFree(*ptr);
        *ptr = nullptr;
        if (cudaMalloc(ptr, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
        return true;
    };
    if (nl > h->part_cap_l) {
        if (!realloc(reinterpret_cast<void **>(&h->part_l), sizeof(uint16_t) * nl)) { h->part_cap_l = 0; return fail(BH_ENOMEM, "SORT scratch"); }
        h->part_cap_l = nl;
    }
    if (weighted && nl > h->part_cap_w) {
        if (!realloc(reinterpret_cast<void **>(&h->part_w), sizeof(double) * nl)) { h->part_cap_w = 0; return fail(BH_ENOMEM, "SORT scratch"); }
        h->part_cap_w = nl;
    }
    if (no > h->part_cap_offs) {
        if (!realloc(reinterpret_cast<void **>(&h->part_offs), sizeof(uint32_t) * no)) { h->part_cap_offs = 0; return fail(BH_ENOMEM, "SORT scratch"); }
        h->part_cap_offs = no;
    }
    if (P > h->part_P) {
        if (!realloc(reinterpret_cast<void **>(&h->part_cnt), sizeof(unsigned long long) * P) ||
            !realloc(reinterpret_cast<void **>(&h->part_cp), sizeof(unsigned long long) * (P + 1))) {
            h->part_P = 0;
            return fail(BH_ENOMEM, "SORT scratch");
        }
        CUDA_TRY(cudaMemsetAsync(h->part_cnt, 0, sizeof(unsigned long long) * P, s));
        h->part_P = P;
    }
    return BH_OK;
}

bh_status fill_sort(bh_hist *h, int64_t n, const double *const *coords, const double *w, cudaStream_t s,
                    const int32_t *gate = nullptr) {
    const bool W = w != nullptr;
    const int pb = sort_pb(W);
    const int P = (int)sort_partitions(h, W);
    // chunk: bounds the scratch (2 or 10 B per event) and keeps pass 2's merge traffic
    // (about (#SM + P) partitions x 2^pb bins per chunk) small next to the events
    int64_t chunk = W ? (int64_t(1) << 26) : (int64_t(1) << 28);   // unit 2^28: C3 in one chunk (+3%)
    if (const char *env = getenv("BHIST_SORT_CHUNK")) chunk = std::max<int64_t>(1, atoll(env));   // tests: many chunks
    if (bh_status r = part_scratch(h, std::min(n, chunk), W, P, s)) return r;
    // pass-1 shared memory: staging + counters, then the variable-axis tables if they fit
    const int tile = kPartThreads * part_ev(h->dim, W);
    const int rc = sort_rc(W, P), ts = sort_ts(tile, P, rc);
    const size_t stages = (size_t)kPartStages * (h->dim + (W ? 1 : 0)) * tile * 8 + 8 * kPartStages;
    const size_t base = align16(stages + (W ? 8 * (size_t)ts : 0) + 2 * (size_t)ts + 4 * (2 * (size_t)P + 1));
    AxisP ax[kMaxDim];
    size_t tabs = 0;
    for (int a = 0; a < h->dim; ++a) {
        ax[a] = h->ax[a];
        if (ax[a].var) { ax[a].tab_off = (int32_t)(base + tabs); tabs += axis_table_bytes(ax[a]); }
    }
    const size_t per_cta = h->smem_optin - kStaticSmemReserve;        // one pass-1 CTA per SM
    const int vm = tabs == 0 ? 0 : (base + tabs <= per_cta ? 1 : 2);
    const size_t smem1 = vm == 1 ? base + tabs : base;
    if (smem1 > per_cta) return fail(BH_EINVAL, "SORT pass 1 needs %zu B of shared memory", smem1);
    for (int64_t off = 0; off < n; off += chunk) {
        const int64_t m = std::min(chunk, n - off);
        const double *cs[kMaxDim] = {};
        for (int a = 0; a < h->dim; ++a) cs[a] = coords[a] + off;
        FillP p = make_params(h, m, cs, W ? w + off : nullptr);
        for (int a = 0; a < h->dim; ++a) p.ax[a] = ax[a];
        PartP q{};
        q.gate = gate;
        q.rec_l = h->part_l;
        q.rec_w = h->part_w;
        q.offs = h->part_offs;
        q.cnt = h->part_cnt;
        q.cp = h->part_cp;
        q.P = P;
        q.pb = pb;
        q.tile = tile;
        q.ts = ts;
        q.ntiles = (int)((m + tile - 1) / tile);
        const int g1 = std::max(1, std::min(q.ntiles, h->nsm));
        cudaError_t e;
        switch (h->dim * 2 + (W ? 1 : 0)) {
        case 2: e = fill_launch_part1<1, false>(p, q, vm, rc, g1, smem1, s); break;
        case 3: e = fill_launch_part1<1, true>(p, q, vm, rc, g1, smem1, s); break;
        case 4: e = fill_launch_part1<2, false>(p, q, vm, rc, g1, smem1, s); break;
        case 5: e = fill_launch_part1<2, true>(p, q, vm, rc, g1, smem1, s); break;
        case 6: e = fill_launch_part1<3, false>(p, q, vm, rc, g1, smem1, s); break;
        default: e = fill_launch_part1<3, true>(p, q, vm, rc, g1, smem1, s); break;
        }
        if (e != cudaSuccess) return fail(BH_ECUDA, "SORT pass 1 launch: %s", cudaGetErrorString(e));
        k_part_plan<<<1, 32, 0, s>>>(q);
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail(BH_ECUDA, "SORT plan launch: %s", cudaGetErrorString(e));
        const int g2 = h->nsm * kReduceCtas;
        e = W ? (rc == 1 ? launch_part2<true, 1>(p, q, g2, s) : launch_part2<true, 4>(p, q, g2, s))
              : (rc == 1 ? launch_part2<false, 1>(p, q, g2, s) : launch_part2<false, 8>(p, q, g2, s));
        if (e != cudaSuccess) return fail(BH_ECUDA, "SORT pass 2 launch: %s", cudaGetErrorString(e));
        h->launches += 3;
    }
    return BH_OK;
}

// AUTO for bin spaces that do not fit PRIV (measured: SORT 1.45x faster than CACHE on
// spread-out unit-weight data, several times slower with a hot partition or weights, and its
// per-chunk merge only amortizes over >= ~8 x #SM x 2^pb events; for weights, GLOBAL's
// paired-lane REDs are 1.6x faster than CACHE on spread-out data (C3w 2.0 vs 3.2 ms) and
// ~40x slower on a hot bin (C4w), whose same-address REDs serialize in L2).  The first large
// fill after create/reset launches k_part_probe on a strided sample of its own events; the
// probe writes both decisions to device memory (unit weights: SORT if no partition holds
// > 5% of the sample and no hashed bin bucket > 1%; weights: GLOBAL if no bucket holds
// > 0.2%), and that fill and every later eligible one launch BOTH paths, each gated on the
// device flag (the other exits at once).  The choice therefore depends on the data only,
// never on host timing, and the host never waits for it.  Returns the device flag of this
// fill's choice (1: SORT / GLOBAL), or nullptr (plain CACHE).
constexpr int kProbeSamples = 1 << 14;     // one CTA: ~40 us, once per histogram and reset

// Unit-weight WINDOW plan (probe decision 2, see k_part_probe): CACHE with kWinSlots slots,
// its tables, then the box counts at `off`, as many as the rest of shared memory holds (amax).
constexpr int kWinSlots = 1024;
bool win_plan(const bh_hist *h, int64_t n, FillPlan &pw, size_t &off, int &amax) {
    if (h->dim > 2 || plan_fill(h, false, pw, n, 0, BH_STRATEGY_CACHE, kWinSlots) != BH_OK) {
        g_err.clear();
        return false;
    }
    off = align16(pw.c.smem);
    const size_t room = h->smem_optin > off + kStaticSmemReserve ? h->smem_optin - off - kStaticSmemReserve : 0;
    amax = (int)std::min<size_t>(room / 4, (size_t)1 << 20);
    return amax >= 1024;
}

// Identity of a fill's inputs for AUTO's decisions: the column pointers and the size.
uint64_t input_key(const bh_hist *h, int64_t n, const double *const *coords) {
    uint64_t k = 1469598103934665603ull ^ (uint64_t)n;
    for (int a = 0; a < h->dim; ++a) k = (k ^ reinterpret_cast<uintptr_t>(coords[a])) * 1099511628211ull;
    return k;
}
// After bh_reset (state 2) a decision stands for the same inputs, else it is made again.
void rearm(int &state, uint64_t &stored, uint64_t key) {
    if (state == 2) state = key == stored ? 1 : 0;
    if (state == 0) stored = key;
}

// Smallest fill the AUTO probes look at: `dflt`, or BHIST_AUTO_MIN_EVENTS (sanitizer runs and
// tests of the decisions on small inputs); never below two probe samples per event run.
int64_t auto_min_events(int64_t dflt) {
    const char *e = getenv("BHIST_AUTO_MIN_EVENTS");
    return std::max<int64_t>(e ? atoll(e) : dflt, 2 * (int64_t)kProbeSamples);
}

const int32_t *auto_gate(bh_hist *h, int64_t n, const double *const *coords, bool weighted, cudaStream_t s) {
    if (h->strategy != BH_STRATEGY_AUTO || resolve_strategy(h, weighted) != BH_STRATEGY_CACHE) return nullptr;
    const int P = (int)sort_partitions(h, false);
    if (P > kPartMaxP || n < auto_min_events(8LL * h->nsm * (1LL << sort_pb(false)))) return nullptr;
    if (getenv(weighted ? "BHIST_NO_AUTO_GLOBAL" : "BHIST_NO_AUTO_SORT")) return nullptr;
    if (!h->probe_dev) {
        if (cudaMalloc(reinterpret_cast<void **>(&h->probe_dev), 8 * sizeof(unsigned int)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;                                  // no probe: stay on CACHE
        }
    }
    rearm(h->probe_state, h->probe_key, input_key(h, n, coords));
    if (h->probe_state == 0) {
        FillP p = make_params(h, n, coords, nullptr);
        if (cudaMemsetAsync(h->probe_dev, 0, 8 * sizeof(unsigned int), s) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        FillPlan pw;
        size_t woff = 0;
        int amax = 0;
        if (getenv("BHIST_NO_AUTO_WINDOW") || !win_plan(h, n, pw, woff, amax)) amax = 0;
        const size_t sm = sizeof(unsigned int) * (P + kProbeHash + 4 * kProbeMarg + 2 + kProbeSamples);
        cudaError_t e;
        switch (h->dim) {
        case 1:
            e = cudaFuncSetAttribute(k_part_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e == cudaSuccess) k_part_probe<1><<<1, 1024, sm, s>>>(p, sort_pb(false), P, kProbeSamples, amax, h->probe_dev);
            break;
        case 2:
            e = cudaFuncSetAttribute(k_part_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e == cudaSuccess) k_part_probe<2><<<1, 1024, sm, s>>>(p, sort_pb(false), P, kProbeSamples, amax, h->probe_dev);
            break;
        default:
            e = cudaFuncSetAttribute(k_part_probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e == cudaSuccess) k_part_probe<3><<<1, 1024, sm, s>>>(p, sort_pb(false), P, kProbeSamples, 0, h->probe_dev);
            break;
        }
        if (e != cudaSuccess) { cudaGetLastError(); return nullptr; }
        if (cudaGetLastError() != cudaSuccess) return nullptr;
        h->launches++;
        h->probe_state = 1;                                   // decided (on the device)
    }
    return reinterpret_cast<const int32_t *>(h->probe_dev + (weighted ? 3 : 2));
}

// AUTO's lane-private window of hot cells (see HotTab) for large weighted PRIVA and CACHE
// fills: the first such fill after create/reset launches k_hot_probe on a strided sample of
// its events; that fill and every later one launch the window kernel and the plain one (and,
// for CACHE, the GLOBAL one of k_part_probe's decision `gdec`), gated on the probe's device
// word.  Returns the device table, or nullptr (no window).
constexpr int64_t kHotMinEvents = int64_t(1) << 22;
constexpr int kHotCacheSlots = 4096;       // CACHE's slots next to the lane window
const HotTab *auto_hot(bh_hist *h, int64_t n, const double *const *coords, const FillPlan &pl,
                       const int32_t *gdec, cudaStream_t s) {
    const bool priva = pl.c.strategy == BH_STRATEGY_PRIV && pl.wc_off >= 0;
    if (h->strategy != BH_STRATEGY_AUTO || !(priva || pl.c.strategy == BH_STRATEGY_CACHE) || n < auto_min_events(kHotMinEvents) ||
        getenv("BHIST_NO_HOT_WINDOW"))
        return nullptr;
    if (!h->hot_dev) {
        if (cudaMalloc(reinterpret_cast<void **>(&h->hot_dev), sizeof(HotTab)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    }
    rearm(h->hot_state, h->hot_key, input_key(h, n, coords));
    if (h->hot_state == 0) {
        FillP p = make_params(h, n, coords, nullptr);
        const unsigned int *gd = reinterpret_cast<const unsigned int *>(gdec);
        switch (h->dim) {
        case 1: k_hot_probe<1><<<1, 1024, 0, s>>>(p, kProbeSamples, gd, h->hot_dev); break;
        case 2: k_hot_probe<2><<<1, 1024, 0, s>>>(p, kProbeSamples, gd, h->hot_dev); break;
        default: k_hot_probe<3><<<1, 1024, 0, s>>>(p, kProbeSamples, gd, h->hot_dev); break;
        }
        if (cudaGetLastError() != cudaSuccess) return nullptr;
        h->launches++;
        h->hot_state = 1;
    }
    return h->hot_dev;
}

// One fill over device-resident columns, split into launches of <= 2^30 events.
bh_status fill_device(bh_hist *h, int64_t n, const double *const *coords, const double *w, cudaStream_t s) {
    if (w) h->weighted_content = true;
    if (w && h->strategy == BH_STRATEGY_EXACT) return fill_exact(h, n, coords, w, s);
    if (resolve_strategy(h, w != nullptr) == BH_STRATEGY_SORT) return fill_sort(h, n, coords, w, s);
    const int32_t *gate = auto_gate(h, n, coords, w != nullptr, s);
    if (gate && !w)                                           // SORT, run iff the device flag says so
        if (bh_status r = fill_sort(h, n, coords, w, s, gate)) return r;
    FillPlan pl, pg;                                          // pg: weighted GLOBAL, run iff the flag says so
    if (bh_status r = plan_fill(h, w != nullptr, pl, n)) return r;
    if (gate && w)
        if (bh_status r = plan_fill(h, true, pg, n, 0, BH_STRATEGY_GLOBAL)) return r;
    // unit weights: the WINDOW variant of CACHE (probe decision 2)
    FillPlan pwin;
    size_t win_off = 0;
    int win_amax = 0;
    const bool winp = gate && !w && !getenv("BHIST_NO_AUTO_WINDOW") && win_plan(h, n, pwin, win_off, win_amax);
    // weighted PRIVA / CACHE: the hot-cell window variant, run iff the probe's word says 2
    const HotTab *hot = w ? auto_hot(h, n, coords, pl, gate, s) : nullptr;
    FillPlan phot;
    const bool hot_cache = pl.c.strategy == BH_STRATEGY_CACHE;
    const size_t hot_bytes = hot_smem_bytes(threads_of(pl.c.strategy, true, h->dim));
    if (hot && (hot_cache ? plan_fill(h, true, phot, n, hot_bytes, BH_STRATEGY_CACHE, kHotCacheSlots) != BH_OK
                          : plan_fill(h, true, phot, n, hot_bytes) != BH_OK || phot.c.strategy != BH_STRATEGY_PRIV ||
                                phot.wc_off < 0)) {
        hot = nullptr;
        g_err.clear();
    }
    LaunchCfg &c = pl.c;
    const int64_t kMaxLaunch = int64_t(1) << 30;   // in-kernel event indices are int32
    for (int64_t off = 0; off < n; off += kMaxLaunch) {
        const int64_t m = std::min(kMaxLaunch, n - off);
        const double *cs[kMaxDim] = {};
        for (int a = 0; a < h->dim; ++a) cs[a] = coords[a] + off;
        const double *ws = c.weighted ? w + off : nullptr;
        FillP p = make_params(h, m, cs, ws);
        for (int a = 0; a < h->dim; ++a) p.ax[a] = pl.ax[a];
        p.gate = gate;                                        // CACHE, run iff the flag is 0
        p.gate_run = gate_bit(0);
        // vector path: every column must share the same 16-byte phase
        const uintptr_t ph = reinterpret_cast<uintptr_t>(cs[0]) & 15;
        c.vec = (ph % 8) == 0;
        for (int a = 1; a < h->dim; ++a) c.vec &= (reinterpret_cast<uintptr_t>(cs[a]) & 15) == ph;
        if (c.weighted) c.vec &= (reinterpret_cast<uintptr_t>(ws) & 15) == ph;
        p.peel = c.vec && ph ? 1 : 0;
        if (p.peel > m) p.peel = (int32_t)m;
        p.cache_slots = cache_slots_for(c.weighted);
        p.replicas = pl.replicas;
        p.wc_off = pl.wc_off;
        c.grid = grid_for(h, c, m);
        cudaError_t e;
        if (winp) {                                           // unit: the gated WINDOW kernel
            FillP pq = p;
            for (int a = 0; a < h->dim; ++a) pq.ax[a] = pwin.ax[a];
            pq.cache_slots = kWinSlots;
            pq.win = h->probe_dev + 4;
            pq.win_off = (int32_t)win_off;
            pq.gate_run = gate_bit(2);
            LaunchCfg cw = pwin.c;
            cw.smem = win_off + 4 * (size_t)win_amax;
            cw.vec = c.vec;
            cw.grid = grid_for(h, cw, m);
            e = h->dim == 1 ? fill_launch<1, false>(pq, cw, s) : fill_launch<2, false>(pq, cw, s);
            if (e != cudaSuccess) return fail(BH_ECUDA, "fill launch: %s", cudaGetErrorString(e));
            ++h->launches;
        }
        if (hot) {                                            // gated window kernel, then the plain one
            FillP pq = p;
            for (int a = 0; a < h->dim; ++a) pq.ax[a] = phot.ax[a];
            pq.replicas = phot.replicas;
            pq.wc_off = phot.wc_off;
            if (hot_cache) pq.cache_slots = kHotCacheSlots;
            pq.hot = hot;
            pq.hot_off = (int32_t)align16(phot.c.smem);
            pq.gate = &hot->flag;
            pq.gate_run = gate_bit(2);
            LaunchCfg ch = phot.c;
            ch.smem = pq.hot_off + hot_bytes;
            ch.vec = c.vec;
            ch.grid = grid_for(h, ch, m);
            switch (h->dim) {
            case 1: e = fill_launch<1, true>(pq, ch, s); break;
            case 2: e = fill_launch<2, true>(pq, ch, s); break;
            default: e = fill_launch<3, true>(pq, ch, s); break;
            }
            if (e != cudaSuccess) return fail(BH_ECUDA, "fill launch: %s", cudaGetErrorString(e));
            ++h->launches;
            p.gate = &hot->flag;
            // the plain sink also runs for every word whose kernel this fill does not launch (the
            // probe decided once, on an earlier fill that may have had other candidates)
            p.gate_run = gate_bit(0) | (gate && w ? 0 : gate_bit(1));
        }
        if (gate && w) {                                      // weighted AUTO: the gated GLOBAL fill first
            FillP pq = p;
            for (int a = 0; a < h->dim; ++a) pq.ax[a] = pg.ax[a];
            pq.gate_run = gate_bit(1);
            LaunchCfg &cg = pg.c;
            cg.vec = c.vec;
            cg.grid = grid_for(h, cg, m);
            switch (h->dim) {
            case 1: e = fill_launch<1, true>(pq, cg, s); break;
            case 2: e = fill_launch<2, true>(pq, cg, s); break;
            default: e = fill_launch<3, true>(pq, cg, s); break;
            }
            if (e != cudaSuccess) return fail(BH_ECUDA, "fill launch: %s", cudaGetErrorString(e));
            ++h->launches;
        }
        switch (h->dim) {
        case 1: e = c.weighted ? fill_launch<1, true>(p, c, s) : fill_launch<1, false>(p, c, s); break;
        case 2: e = c.weighted ? fill_launch<2, true>(p, c, s) : fill_launch<2, false>(p, c, s); break;
        default: e = c.weighted ? fill_launch<3, true>(p, c, s) : fill_launch<3, false>(p, c, s); break;
        }
        if (e != cudaSuccess) return fail(BH_ECUDA, "fill launch: %s", cudaGetErrorString(e));
        ++h->launches;
    }
    return BH_OK;
}

// float32 columns (see k_fill_f32); EXACT is not offered for float32 weights (uses AUTO).
// 4-byte columns: float32 or (is_int) int32 coordinates, float32 weights.
bh_status fill_device_f32(bh_hist *h, int64_t n, const float *const *coords, const float *w, cudaStream_t s,
                          bool is_int = false) {
    if (w) h->weighted_content = true;
    FillPlan pl;
    if (bh_status r = plan_fill(h, w != nullptr, pl, n)) return r;
    LaunchCfg &c = pl.c;
    const int64_t kMaxLaunch = int64_t(1) << 30;
    for (int64_t off = 0; off < n; off += kMaxLaunch) {
        const int64_t m = std::min(kMaxLaunch, n - off);
        const double *cs[kMaxDim] = {};
        for (int a = 0; a < h->dim; ++a) cs[a] = reinterpret_cast<const double *>(coords[a] + off);
        const double *ws = w ? reinterpret_cast<const double *>(w + off) : nullptr;
        FillP p = make_params(h, m, cs, ws);
        for (int a = 0; a < h->dim; ++a) p.ax[a] = pl.ax[a];
        const uintptr_t ph = reinterpret_cast<uintptr_t>(cs[0]) & 15;
        bool vec = (ph % 4) == 0;
        for (int a = 1; a < h->dim; ++a) vec &= (reinterpret_cast<uintptr_t>(cs[a]) & 15) == ph;
        if (w) vec &= (reinterpret_cast<uintptr_t>(ws) & 15) == ph;
        p.peel = vec ? (int32_t)std::min<int64_t>(ph ? (16 - ph) / 4 : 0, m) : -1;
        p.cache_slots = cache_slots_for(c.weighted);
        p.replicas = pl.replicas;
        p.wc_off = pl.wc_off;
        c.grid = grid_for(h, c, m);
        cudaError_t e;
        if (is_int) {
            switch (h->dim) {
            case 1: e = c.weighted ? fill_launch_i32<1, true>(p, c, s) : fill_launch_i32<1, false>(p, c, s); break;
            case 2: e = c.weighted ? fill_launch_i32<2, true>(p, c, s) : fill_launch_i32<2, false>(p, c, s); break;
            default: e = c.weighted ? fill_launch_i32<3, true>(p, c, s) : fill_launch_i32<3, false>(p, c, s); break;
            }
        } else {
            switch (h->dim) {
            case 1: e = c.weighted ? fill_launch_f32<1, true>(p, c, s) : fill_launch_f32<1, false>(p, c, s); break;
            case 2: e = c.weighted ? fill_launch_f32<2, true>(p, c, s) : fill_launch_f32<2, false>(p, c, s); break;
            default: e = c.weighted ? fill_launch_f32<3, true>(p, c, s) : fill_launch_f32<3, false>(p, c, s); break;
            }
        }
        if (e != cudaSuccess) return fail(BH_ECUDA, "fill_f32 launch: %s", cudaGetErrorString(e));
        ++h->launches;
    }
    return BH_OK;
}

bh_status check_hist(const bh_hist *h) {
    if (!h) return fail(BH_EINVAL, "NULL histogram");
    return BH_OK;
}

// calls that touch the state or its stream may not run while a persistent bulk consumer
// (bh_bulk_begin .. bh_bulk_end) owns the histogram
bh_status bulk_check(const bh_hist *h) {
    if (check_hist(h)) return BH_EINVAL;
    if (h->bulk_active) return fail(BH_EINVAL, "a bulk session (bh_bulk_begin) is active on this histogram");
    return BH_OK;
}

}  // namespace

namespace bh {
bh_status set_error(bh_status st, const char *msg) { return fail(st, "%s", msg); }
size_t axis_table_bytes_of(const AxisP &a) { return axis_table_bytes(a); }
}  // namespace bh

extern "C" {

int32_t bh_version(void) { return 10000; }

const char *bh_last_error(void) { return g_err.c_str(); }

bh_status bh_create(int32_t dim, const bh_axis *axes, int32_t device, bh_hist **out) {
    if (!out) return fail(BH_EINVAL, "out is NULL");
    *out = nullptr;
    if (dim < 1 || dim > 3) return fail(BH_EINVAL, "dim must be 1, 2 or 3 (got %d)", dim);
    if (!axes) return fail(BH_EINVAL, "axes is NULL");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(BH_EDEVICE, "no CUDA device");
    }
    if (device < 0 || device >= ndev) return fail(BH_EDEVICE, "device %d out of range [0,%d)", device, ndev);
    // validate axes (all on the host, before any allocation)
    int64_t G = 1;
    for (int a = 0; a < dim; ++a) {
        const bh_axis &A = axes[a];
        if (A.nbins < 1) return fail(BH_EINVAL, "axis %d: nbins must be >= 1", a);
        if (A.edges) {
            for (int i = 0; i <= A.nbins; ++i)
                if (!std::isfinite(A.edges[i])) return fail(BH_EINVAL, "axis %d: edge %d not finite", a, i);
            for (int i = 0; i < A.nbins; ++i)
                if (!(A.edges[i] < A.edges[i + 1])) return fail(BH_EINVAL, "axis %d: edges not strictly increasing at %d", a, i);
            if (!std::isfinite(A.edges[A.nbins] - A.edges[0])) return fail(BH_EINVAL, "axis %d: edge range overflows", a);
        } else {
            if (!std::isfinite(A.xmin) || !std::isfinite(A.xmax) || !(A.xmin < A.xmax))
                return fail(BH_EINVAL, "axis %d: need finite xmin < xmax", a);
            const double D = A.xmax - A.xmin;
            if (!std::isfinite(D) || !std::isfinite((double)A.nbins * D) || !std::isfinite((double)A.nbins / D))
                return fail(BH_EINVAL, "axis %d: nbins*(xmax-xmin) not finite", a);
        }
        G *= (int64_t)A.nbins + 2;
        if (G >= (int64_t(1) << 31)) return fail(BH_EINVAL, "total bins (with flow) must be < 2^31");
    }
    DeviceGuard dg(device);
    if (!dg.ok) return fail(BH_EDEVICE, "cudaSetDevice(%d) failed", device);
    bh_hist *h = new bh_hist();
    h->device = device;
    h->dim = dim;
    h->G = G;
    h->K = dim == 1 ? 4 : dim == 2 ? 7 : 11;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) { delete h; return fail(BH_ECUDA, "cudaGetDeviceProperties"); }
    h->nsm = prop.multiProcessorCount;
    h->smem_optin = prop.sharedMemPerBlockOptin;
    h->max_grid = h->nsm * 4;
    h->st1 = axes[0].nbins + 2;
    h->st2 = dim > 2 ? (axes[0].nbins + 2) * (axes[1].nbins + 2) : 1;
    auto cleanup = [&](bh_status st) { bh_destroy(h); return st; };
#define ALLOC(ptr, bytes)                                                                          \
    do {                                                                                           \
        if (cudaMalloc(reinterpret_cast<void **>(&(ptr)), (bytes)) != cudaSuccess) {               \
            cudaGetLastError();                                                                    \
            return cleanup(fail(BH_ENOMEM, "cudaMalloc(%zu) failed", (size_t)(bytes)));            \
        }                                                                                          \
    } while (0)
    ALLOC(h->count, sizeof(unsigned long long) * G);
    ALLOC(h->sw, 2 * sizeof(double) * G);
    ALLOC(h->stats, sizeof(double) * 16);
    ALLOC(h->entries, sizeof(unsigned long long));
    ALLOC(h->partials, sizeof(double) * 16 * h->max_grid);
    ALLOC(h->counter, sizeof(unsigned int));
    ALLOC(h->pack_buf, sizeof(double) * (2 * G + h->K + 1));
    if (cudaMallocHost(reinterpret_cast<void **>(&h->pack_host), sizeof(double) * (2 * G + h->K + 1)) != cudaSuccess) {
        cudaGetLastError();
        return cleanup(fail(BH_ENOMEM, "cudaMallocHost failed"));
    }
    for (int a = 0; a < dim; ++a) {
        const bh_axis &A = axes[a];
        AxisP &P = h->ax[a];
        P.n = A.nbins;
        if (!A.edges) {
            P.var = 0;
            P.xmin = A.xmin;
            P.xmax = A.xmax;
            P.D = A.xmax - A.xmin;            // RN, as the definition rounds it
            P.inv = (double)A.nbins / P.D;    // RN(n/D): fast-path multiplier
        } else {
            P.var = 1;
            P.xmin = A.edges[0];
            P.xmax = A.edges[A.nbins];
            // guide cells: a power of two, up to 64 per bin (fewer edges per cell for
            // non-uniform edges, e.g. log-spaced) while the shared-memory tables (float32
            // edges + uint16 guide) stay <= 56 KB; at least ~n/2 cells
            int gc = 1;
            while (2 * gc < A.nbins && gc < (1 << 22)) gc <<= 1;
            while (gc < 64 * A.nbins && 4 * (size_t)(A.nbins + 1) + 2 * (size_t)(2 * gc + 1) <= 56 * 1024) gc <<= 1;
            // compact mode (g16 == 3): one 32-bit word per cell, no float32 edges, as many cells
            // as fit in 56 KB (<= 64 per bin); taken when <= 2% of the interior edges share a
            // cell with two others (those cells search the float64 edges), e.g. C2's 10,000
            // near-uniform bins: 8192 cells, 0.3% of the edges
            int gc3 = 1;
            while (2 * gc3 <= 64 * A.nbins && 4 * (size_t)(2 * gc3 + 1) <= 56 * 1024) gc3 <<= 1;
            bool compact = (A.nbins - 1) < 16384 && 2 * gc3 >= A.nbins && !getenv("BHIST_NO_COMPACT");
            if (compact) {
                const double sc = (double)gc3 / (A.edges[A.nbins] - A.edges[0]);
                std::vector<int> cnt(gc3, 0);
                std::vector<int> cell(A.nbins + 1, 0);
                for (int i = 1; i < A.nbins; ++i) {
                    const double t = (A.edges[i] - A.edges[0]) * sc;
                    cell[i] = std::min((int)t, gc3 - 1);
                    ++cnt[cell[i]];
                }
                int crowded = 0;
                for (int i = 1; i < A.nbins; ++i) crowded += cnt[cell[i]] >= 3;
                compact = crowded <= 0.02 * std::max(1, A.nbins - 1);
            }
            // log-domain compact cells (positive edges, e.g. log-spaced): cell = (bits(x) >> lg)
            // - (bits(e0) >> lg), the finest lg whose cells fit the table; taken when the linear
            // cells crowd too many edges and these do not
            int lgc = 0, lcells = 0;
            if (!compact && A.edges[0] > 0.0 && (A.nbins - 1) < 16384 && !getenv("BHIST_NO_LOG_GUIDE") &&
                !getenv("BHIST_NO_COMPACT")) {
                auto bits = [](double v) { long long b; memcpy(&b, &v, 8); return b; };
                const long long b0 = bits(A.edges[0]), bn = bits(A.edges[A.nbins]);
                const int maxc = (56 * 1024) / 4 - 1;
                for (int lg = 8; lg < 62; ++lg) {
                    const long long cells = (bn >> lg) - (b0 >> lg) + 1;
                    if (cells > maxc) continue;
                    std::vector<int> cnt((size_t)cells, 0), cell(A.nbins + 1, 0);
                    for (int i = 1; i < A.nbins; ++i) {
                        cell[i] = (int)((bits(A.edges[i]) >> lg) - (b0 >> lg));
                        ++cnt[cell[i]];
                    }
                    int crowded = 0;
                    for (int i = 1; i < A.nbins; ++i) crowded += cnt[cell[i]] >= 3;
                    if (crowded <= 0.02 * std::max(1, A.nbins - 1)) { lgc = lg; lcells = (int)cells; }
                    break;                   // the finest lg that fits decides
                }
            }
            if (compact) gc = gc3;
            if (lgc) { compact = true; gc = lcells; }
            P.gcells = gc;
            P.gscale = (double)gc / (P.xmax - P.xmin);
            P.lg = lgc;
            P.kb = 0;
            if (lgc) { long long b0; memcpy(&b0, &A.edges[0], 8); P.kb = b0 >> lgc; }
            if (!std::isfinite(P.gscale) || !(P.gscale > 0)) return cleanup(fail(BH_EINVAL, "axis %d: edge range too small", a));
            double *de = nullptr;
            uint32_t *dg2 = nullptr;
            ALLOC(de, sizeof(double) * (A.nbins + 1));
            h->axis_mem.push_back(de);
            ALLOC(dg2, sizeof(uint32_t) * (gc + 1));
            h->axis_mem.push_back(dg2);
            if (cudaMemcpy(de, A.edges, sizeof(double) * (A.nbins + 1), cudaMemcpyHostToDevice) != cudaSuccess)
                return cleanup(fail(BH_ECUDA, "edge upload failed"));
            float *de32 = nullptr;
            ALLOC(de32, sizeof(float) * (A.nbins + 1));
            h->axis_mem.push_back(de32);
            P.e = de;
            P.guide = dg2;
            P.e32 = de32;
            P.g16 = compact ? (lgc ? 4 : 3) : (A.nbins - 1) < 16384 ? 2 : ((A.nbins - 1) < 65536 ? 1 : 0);
            k_build_guide<<<(gc + 1 + 255) / 256, 256>>>(P, dg2);
            k_edges_f32<<<(A.nbins + 1 + 255) / 256, 256>>>(de, A.nbins + 1, de32);
            unsigned char *img = nullptr;
            P.tab_bytes = (int32_t)axis_table_bytes(P);
            ALLOC(img, P.tab_bytes);
            h->axis_mem.push_back(img);
            cudaMemset(img, 0, P.tab_bytes);
            k_table_image<<<(std::max(A.nbins, gc) + 1 + 255) / 256, 256>>>(P, dg2, img);
            P.tab_img = reinterpret_cast<const uint4 *>(img);
            if (cudaGetLastError() != cudaSuccess) return cleanup(fail(BH_ECUDA, "guide build launch failed"));
        }
    }
#undef ALLOC
    if (cudaMemset(h->count, 0, sizeof(unsigned long long) * G) != cudaSuccess ||
        cudaMemset(h->sw, 0, 2 * sizeof(double) * G) != cudaSuccess ||
        cudaMemset(h->stats, 0, sizeof(double) * 16) != cudaSuccess ||
        cudaMemset(h->entries, 0, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(h->counter, 0, sizeof(unsigned int)) != cudaSuccess)
        return cleanup(fail(BH_ECUDA, "initial memset failed"));
    if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(fail(BH_ECUDA, "create: %s", cudaGetErrorString(cudaGetLastError())));
    *out = h;
    return BH_OK;
}

bh_status bh_destroy(bh_hist *h) {
    if (!h) return BH_OK;
    DeviceGuard dg(h->device);
    if (h->bulk_active) bh_bulk_end(h);      // let the persistent consumer finish before freeing
    cudaDeviceSynchronize();
    if (h->bulk_ctl) cudaFreeHost(h->bulk_ctl);
    if (h->bulk_kstream) cudaStreamDestroy(h->bulk_kstream);
    for (cudaEvent_t ev : h->bulk_ev)
        if (ev) cudaEventDestroy(ev);
    cudaFree(h->bulk_dev);
    for (int i = 0; i < kBulkRing; ++i)
        if (h->bulk_stage[i]) cudaFreeHost(h->bulk_stage[i]);
    cudaFree(h->count);
    cudaFree(h->sw);
    cudaFree(h->stats);
    cudaFree(h->entries);
    cudaFree(h->partials);
    cudaFree(h->counter);
    cudaFree(h->limbs);
    cudaFree(h->maxbits);
    cudaFree(h->pack_buf);
    cudaFree(h->part_l);
    cudaFree(h->part_w);
    cudaFree(h->part_offs);
    cudaFree(h->part_cnt);
    cudaFree(h->part_cp);
    cudaFree(h->probe_dev);
    cudaFree(h->hot_dev);
    cudaFree(h->narrow_buf);
    if (h->narrow_host) cudaFreeHost(h->narrow_host);
    if (h->pack_host) cudaFreeHost(h->pack_host);
    for (void *p : h->axis_mem) cudaFree(p);
    for (int i = 0; i < kStageSlots; ++i) {
        if (h->stage[i]) cudaFree(h->stage[i]);
        if (h->copied[i]) cudaEventDestroy(h->copied[i]);
        if (h->consumed[i]) cudaEventDestroy(h->consumed[i]);
    }
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    delete h;
    return BH_OK;
}

bh_status bh_reset(bh_hist *h, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(s);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((h->G / 2 + 255) / 256, (int64_t)h->nsm * 8));
    k_reset<<<grid, 256, 0, st>>>((int)h->G, h->count, h->sw, h->stats, h->entries);
    CUDA_TRY(cudaGetLastError());
    ++h->launches;
    h->weighted_content = false;
    // AUTO re-decides on the next large fill unless it reads the same input buffers (state 2)
    if (h->probe_state) h->probe_state = 2;
    if (h->hot_state) h->hot_state = 2;
    return BH_OK;
}

bh_status bh_fill(bh_hist *h, int64_t n, const double *const *coords, const double *w, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (n < 0) return fail(BH_EINVAL, "n < 0");
    if (n == 0) return BH_OK;
    if (!coords) return fail(BH_EINVAL, "coords is NULL");
    for (int a = 0; a < h->dim; ++a)
        if (!coords[a]) return fail(BH_EINVAL, "coords[%d] is NULL", a);
    DeviceGuard dg(h->device);
    return fill_device(h, n, coords, w, static_cast<cudaStream_t>(s));
}

bh_status bh_fill_f32(bh_hist *h, int64_t n, const float *const *coords, const float *w, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (n < 0) return fail(BH_EINVAL, "n < 0");
    if (n == 0) return BH_OK;
    if (!coords) return fail(BH_EINVAL, "coords is NULL");
    for (int a = 0; a < h->dim; ++a)
        if (!coords[a]) return fail(BH_EINVAL, "coords[%d] is NULL", a);
    DeviceGuard dg(h->device);
    return fill_device_f32(h, n, coords, w, static_cast<cudaStream_t>(s));
}

bh_status bh_fill_i32(bh_hist *h, int64_t n, const int32_t *const *coords, const float *w, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (n < 0) return fail(BH_EINVAL, "n < 0");
    if (n == 0) return BH_OK;
    if (!coords) return fail(BH_EINVAL, "coords is NULL");
    for (int a = 0; a < h->dim; ++a)
        if (!coords[a]) return fail(BH_EINVAL, "coords[%d] is NULL", a);
    DeviceGuard dg(h->device);
    return fill_device_f32(h, n, reinterpret_cast<const float *const *>(coords), w, static_cast<cudaStream_t>(s), true);
}

}  // extern "C"

namespace {
// Host columns -> device staging ring (copy stream) -> the device fill of column type CT
// (double: bh_fill path; float / int32_t: the 4-byte path with float32 weights).
template <typename CT, typename WT>
bh_status fill_host_impl(bh_hist *h, int64_t n, const CT *const *coords, const WT *w, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (n < 0) return fail(BH_EINVAL, "n < 0");
    if (n == 0) return BH_OK;
    if (!coords) return fail(BH_EINVAL, "coords is NULL");
    for (int a = 0; a < h->dim; ++a)
        if (!coords[a]) return fail(BH_EINVAL, "coords[%d] is NULL", a);
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(s);
    // lazily create the copy stream, events and the device double buffer
    if (!h->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    if (h->stage_chunk != h->chunk) {
        CUDA_TRY(cudaStreamSynchronize(h->copy_stream));
        for (int i = 0; i < kStageSlots; ++i) {
            if (h->consumed[i]) CUDA_TRY(cudaEventSynchronize(h->consumed[i]));
            if (h->stage[i]) cudaFree(h->stage[i]);
            h->stage[i] = nullptr;
            if (cudaMalloc(reinterpret_cast<void **>(&h->stage[i]), sizeof(double) * (kMaxDim + 1) * h->chunk) != cudaSuccess) {
                cudaGetLastError();
                h->stage_chunk = 0;
                return fail(BH_ENOMEM, "staging allocation failed");
            }
            if (!h->copied[i]) CUDA_TRY(cudaEventCreateWithFlags(&h->copied[i], cudaEventDisableTiming));
            if (!h->consumed[i]) CUDA_TRY(cudaEventCreateWithFlags(&h->consumed[i], cudaEventDisableTiming));
            h->slot_used[i] = false;       // fresh buffer: nothing reads it yet
        }
        h->stage_chunk = h->chunk;
    }
    // a slot holds (dim + 1) columns of `chunk` float64 values: 2x `chunk` 4-byte values
    const int64_t C = h->stage_chunk * (int64_t)(sizeof(double) / sizeof(CT));
    for (int64_t off = 0; off < n; off += C) {
        const int slot = h->next_slot;
        h->next_slot = (slot + 1) % kStageSlots;
        const int64_t m = std::min(C, n - off);
        CT *buf = reinterpret_cast<CT *>(h->stage[slot]);
        // the slot may be overwritten only after the fill that read it has run:
        // that fill may belong to an earlier bh_fill_host call whose kernels are still queued
        // on a stream (this function returns once the HOST bytes are consumed, not the slots)
        if (h->slot_used[slot]) CUDA_TRY(cudaStreamWaitEvent(h->copy_stream, h->consumed[slot], 0));
        const CT *dcols[kMaxDim] = {};
        for (int a = 0; a < h->dim; ++a) {
            CUDA_TRY(cudaMemcpyAsync(buf + a * C, coords[a] + off, sizeof(CT) * m, cudaMemcpyHostToDevice, h->copy_stream));
            dcols[a] = buf + a * C;
        }
        const WT *dw = nullptr;
        if (w) {
            WT *wb = reinterpret_cast<WT *>(buf + h->dim * C);
            CUDA_TRY(cudaMemcpyAsync(wb, w + off, sizeof(WT) * m, cudaMemcpyHostToDevice, h->copy_stream));
            dw = wb;
        }
        CUDA_TRY(cudaEventRecord(h->copied[slot], h->copy_stream));
        if (!(h->debug & BH_DEBUG_SKIP_COPY_WAIT)) CUDA_TRY(cudaStreamWaitEvent(st, h->copied[slot], 0));
        bh_status r;
        if constexpr (sizeof(CT) == 8) r = fill_device(h, m, dcols, dw, st);
        else r = fill_device_f32(h, m, reinterpret_cast<const float *const *>(dcols), dw, st,
                                 std::is_same<CT, int32_t>::value);
        if (r != BH_OK) return r;
        CUDA_TRY(cudaEventRecord(h->consumed[slot], st));
        h->slot_used[slot] = true;
    }
    // every host byte has been read once the last copy has completed
    CUDA_TRY(cudaStreamSynchronize(h->copy_stream));
    return BH_OK;
}
}  // namespace

extern "C" {

bh_status bh_fill_host(bh_hist *h, int64_t n, const double *const *coords, const double *w, bh_stream s) {
    return fill_host_impl<double, double>(h, n, coords, w, s);
}

bh_status bh_fill_host_f32(bh_hist *h, int64_t n, const float *const *coords, const float *w, bh_stream s) {
    return fill_host_impl<float, float>(h, n, coords, w, s);
}

bh_status bh_fill_host_i32(bh_hist *h, int64_t n, const int32_t *const *coords, const float *w, bh_stream s) {
    return fill_host_impl<int32_t, float>(h, n, coords, w, s);
}

// ---------------------------------------------------------------- persistent bulk consumer
// (bhist_bulk.cuh).  The host side of the descriptor ring: post a bulk (plain stores of its
// fields, then its sequence number with release semantics) and wait for the device's "done".

}  // extern "C"

namespace {
// bulk `seq` is consumed once the done word of its ring slot has reached it
bool bulk_is_done(const bh_hist *h, long long seq) {
    if (seq <= 0) return true;
    return *reinterpret_cast<volatile long long *>(&h->bulk_ctl->done[(seq - 1) % kBulkRing]) >= seq;
}

// wait until the device has consumed bulk `seq` (false on timeout or device-side abort)
bool bulk_wait_done(const bh_hist *h, long long seq) {
    if (bulk_is_done(h, seq)) return true;
    const auto t0 = std::chrono::steady_clock::now();
    const auto limit = std::chrono::nanoseconds(h->bulk_timeout_ns + 2000000000LL);
    for (uint64_t spin = 0;; ++spin) {
        if (bulk_is_done(h, seq)) {
            std::atomic_thread_fence(std::memory_order_acquire);
            return true;
        }
        if ((spin & 1023) == 0) {
            if (*reinterpret_cast<volatile long long *>(&h->bulk_ctl->status) != 0) return false;
            if (std::chrono::steady_clock::now() - t0 > limit) return false;
        }
    }
}

void bulk_post(bh_hist *h, long long seq, int64_t n, const double *const *x, const double *w) {
    BulkDesc *d = &h->bulk_ctl->ring[(seq - 1) % kBulkRing];
    d->n = n;
    for (int a = 0; a < kMaxDim; ++a) d->x[a] = a < h->dim && x ? x[a] : nullptr;
    d->w = w;
    std::atomic_thread_fence(std::memory_order_release);
    *reinterpret_cast<volatile long long *>(&d->seq) = seq;
}

}  // namespace

extern "C" {

bh_status bh_bulk_begin(bh_hist *h, int32_t weighted, int32_t timeout_ms, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (timeout_ms < 0) return fail(BH_EINVAL, "timeout_ms < 0");
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(s);
    if (!h->bulk_ctl) {
        void *p = nullptr;
        if (cudaHostAlloc(&p, sizeof(BulkCtl), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return fail(BH_ENOMEM, "pinned bulk descriptor ring");
        }
        h->bulk_ctl = static_cast<BulkCtl *>(p);
        CUDA_TRY(cudaMalloc(reinterpret_cast<void **>(&h->bulk_dev), sizeof(BulkDev)));
    }
    if (!h->bulk_stage[0]) {          // pinned staging for pageable bulks (kBulkRing slots)
        const int64_t cap = 1 << 16;
        for (int i = 0; i < kBulkRing; ++i)
            if (cudaHostAlloc(reinterpret_cast<void **>(&h->bulk_stage[i]), sizeof(double) * (kMaxDim + 1) * cap,
                              cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                return fail(BH_ENOMEM, "pinned bulk staging");
            }
        h->bulk_stage_cap = cap;
    }
    // the resident kernel runs on a non-blocking stream of the histogram's own, ordered after
    // the caller's earlier work on s; bh_bulk_end orders s after it.  (On the caller's stream
    // it would hold back everything queued behind it -- with the legacy default stream, every
    // blocking stream of the process.)
    if (!h->bulk_kstream) CUDA_TRY(cudaStreamCreateWithFlags(&h->bulk_kstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i)
        if (!h->bulk_ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&h->bulk_ev[i], cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(h->bulk_ev[0], st));
    CUDA_TRY(cudaStreamWaitEvent(h->bulk_kstream, h->bulk_ev[0], 0));
    memset(h->bulk_ctl, 0, sizeof(BulkCtl));
    std::atomic_thread_fence(std::memory_order_seq_cst);
    BulkCtl *dctl = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dctl), h->bulk_ctl, 0));
    CUDA_TRY(cudaMemsetAsync(h->bulk_dev, 0, sizeof(BulkDev), h->bulk_kstream));
    // the plan of a large fill: the kernel lives for the whole sequence, so PRIV's zeroing and
    // flushing of the private bins is paid once, not per bulk
    const bool W = weighted != 0;
    if (W) h->weighted_content = true;
    const int strategy = resolve_one_pass(h, W);
    if (strategy != BH_STRATEGY_PRIV && strategy != BH_STRATEGY_CACHE && strategy != BH_STRATEGY_GLOBAL)
        return fail(BH_EINVAL, "bulk sessions support the PRIV, CACHE and GLOBAL strategies");
    // shared memory for the TMA staging of bulks (two tiles of te events per column), as
    // much as the plan leaves; none: the threads read the host columns directly
    const int ncol = h->dim + (W ? 1 : 0);
    auto stage_bytes = [&](int te) {      // kBulkStages stages + full/empty barriers + tile records
        return align16((size_t)kBulkStages * ncol * (te + 4) * 8 + 16 * kBulkStages + sizeof(BulkTile) * kBulkStages +
                       sizeof(BulkDesc) + 16);
    };
    FillPlan pl;
    int te = 0;
    if (!getenv("BHIST_BULK_NO_TMA"))
        for (int t : {1024, 512, 256, 128}) {
            FillPlan q;
            if (plan_fill(h, W, q, int64_t(1) << 40, stage_bytes(t)) == BH_OK) { pl = q; te = t; break; }
        }
    if (te == 0)
        if (bh_status r = plan_fill(h, W, pl, int64_t(1) << 40)) return r;
    LaunchCfg &c = pl.c;
    const int stage_off = (int)align16(c.smem);
    if (te) c.smem = stage_off + stage_bytes(te);
    const double *none[kMaxDim] = {};
    FillP p = make_params(h, 0, none, nullptr);
    for (int a = 0; a < h->dim; ++a) p.ax[a] = pl.ax[a];
    p.entries_add = 0;                     // entries are added per bulk by the kernel
    p.cache_slots = cache_slots_for(W);
    p.replicas = pl.replicas;
    p.wc_off = pl.wc_off;
    c.grid = h->nsm;                  // x the resident CTAs per SM (launch_bulk_s, occupancy query)
    const long long tmo = (long long)(timeout_ms ? timeout_ms : 10000) * 1000000LL;
    cudaError_t e;
    switch (h->dim) {
    case 1: e = W ? fill_launch_bulk<1, true>(p, c, dctl, h->bulk_dev, tmo, stage_off, te, h->bulk_kstream) : fill_launch_bulk<1, false>(p, c, dctl, h->bulk_dev, tmo, stage_off, te, h->bulk_kstream); break;
    case 2: e = W ? fill_launch_bulk<2, true>(p, c, dctl, h->bulk_dev, tmo, stage_off, te, h->bulk_kstream) : fill_launch_bulk<2, false>(p, c, dctl, h->bulk_dev, tmo, stage_off, te, h->bulk_kstream); break;
    default: e = W ? fill_launch_bulk<3, true>(p, c, dctl, h->bulk_dev, tmo, stage_off, te, h->bulk_kstream) : fill_launch_bulk<3, false>(p, c, dctl, h->bulk_dev, tmo, stage_off, te, h->bulk_kstream); break;
    }
    if (e != cudaSuccess) return fail(BH_ECUDA, "bulk kernel launch: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaEventRecord(h->bulk_ev[1], h->bulk_kstream));
    ++h->launches;
    h->bulk_active = true;
    h->bulk_weighted = W;
    h->bulk_seq = 0;
    h->bulk_timeout_ns = tmo;
    h->bulk_stream = st;
    return BH_OK;
}

bh_status bh_bulk_submit(bh_hist *h, int64_t n, const double *const *coords, const double *w, int64_t *ticket) {
    if (check_hist(h)) return BH_EINVAL;
    if (!h->bulk_active) return fail(BH_EINVAL, "no bulk session (bh_bulk_begin)");
    if (n < 0 || n > (int64_t(1) << 31)) return fail(BH_EINVAL, "bulk size %lld out of [0, 2^31]", (long long)n);
    if (n > 0 && (w != nullptr) != h->bulk_weighted) return fail(BH_EINVAL, "weights must be given iff the session is weighted");
    if (n > 0) {
        if (!coords) return fail(BH_EINVAL, "coords is NULL");
        for (int a = 0; a < h->dim; ++a)
            if (!coords[a]) return fail(BH_EINVAL, "coords[%d] is NULL", a);
    }
    DeviceGuard dg(h->device);
    // pinned columns are read in place (zero-copy); pageable ones are copied, in pieces of at
    // most bulk_stage_cap events, into the pinned staging area of the ring slot (allocated at
    // bh_bulk_begin: no allocation may run while the consumer kernel is resident)
    const double *src[kMaxDim + 1] = {};
    for (int a = 0; a < h->dim && n > 0; ++a) src[a] = coords[a];
    if (n > 0) src[h->dim] = w;
    const double *dev[kMaxDim + 1] = {};
    bool pinned = true;
    for (int a = 0; a <= h->dim && n > 0; ++a) {
        if (!src[a]) continue;
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, src[a]) != cudaSuccess) { cudaGetLastError(); at.type = cudaMemoryTypeUnregistered; }
        if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged)
            return fail(BH_EINVAL, "bh_bulk_submit takes HOST columns (use bh_fill for device columns)");
        if (at.type == cudaMemoryTypeHost && at.devicePointer) dev[a] = static_cast<const double *>(at.devicePointer);
        else pinned = false;
    }
    const int64_t piece = pinned ? std::max<int64_t>(n, 1) : h->bulk_stage_cap;
    int64_t off = 0;
    do {
        const int64_t m = std::min<int64_t>(piece, n - off);
        const long long seq = h->bulk_seq + 1;
        // the ring slot is free once the bulk posted kBulkRing earlier is consumed
        if (!bulk_wait_done(h, seq - kBulkRing)) return fail(BH_ECUDA, "bulk consumer not responding (timed out or aborted)");
        const double *dx[kMaxDim] = {};
        const double *dw = nullptr;
        if (m > 0) {
            const double *col[kMaxDim + 1] = {};
            if (pinned) {
                for (int a = 0; a <= h->dim; ++a) col[a] = dev[a];
            } else {
                double *buf = h->bulk_stage[(seq - 1) % kBulkRing];
                for (int a = 0; a <= h->dim; ++a) {
                    if (!src[a]) continue;
                    double *slotcol = buf + (size_t)a * h->bulk_stage_cap;
                    memcpy(slotcol, src[a] + off, sizeof(double) * m);
                    double *d = nullptr;
                    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void **>(&d), slotcol, 0));
                    col[a] = d - off;                     // indexed from `off` below
                }
            }
            for (int a = 0; a < h->dim; ++a) dx[a] = col[a] + off;
            dw = w ? col[h->dim] + off : nullptr;
        }
        bulk_post(h, seq, m, dx, dw);
        h->bulk_seq = seq;
        off += m;
    } while (off < n);
    if (ticket) *ticket = h->bulk_seq;
    return BH_OK;
}

bh_status bh_bulk_wait(bh_hist *h, int64_t ticket) {
    if (check_hist(h)) return BH_EINVAL;
    if (!h->bulk_active) return fail(BH_EINVAL, "no bulk session (bh_bulk_begin)");
    if (ticket > h->bulk_seq) return fail(BH_EINVAL, "ticket %lld was not issued", (long long)ticket);
    if (!bulk_wait_done(h, ticket)) return fail(BH_ECUDA, "bulk consumer not responding (timed out or aborted)");
    return BH_OK;
}

bh_status bh_bulk_fill(bh_hist *h, int64_t n, const double *const *coords, const double *w) {
    int64_t t = 0;
    if (bh_status r = bh_bulk_submit(h, n, coords, w, &t)) return r;
    return bh_bulk_wait(h, t);
}

bh_status bh_bulk_end(bh_hist *h) {
    if (check_hist(h)) return BH_EINVAL;
    if (!h->bulk_active) return fail(BH_EINVAL, "no bulk session (bh_bulk_begin)");
    DeviceGuard dg(h->device);
    const long long seq = h->bulk_seq + 1;
    bool ok = bulk_wait_done(h, seq - kBulkRing);
    if (ok) {
        bulk_post(h, seq, -1, nullptr, nullptr);
        ok = bulk_wait_done(h, seq);                 // every CTA has flushed its bins and stats
    }
    ok = ok && *reinterpret_cast<volatile long long *>(&h->bulk_ctl->status) == 0;
    h->bulk_active = false;
    h->bulk_seq = seq;
    CUDA_TRY(cudaStreamWaitEvent(h->bulk_stream, h->bulk_ev[1], 0));    // s after the session
    if (!ok) {
        // the kernel has left (or will leave) on its own after its timeout
        cudaStreamSynchronize(h->bulk_kstream);
        cudaGetLastError();
        return fail(BH_ECUDA, "bulk consumer not responding (timed out or aborted); the session's fills are lost");
    }
    return BH_OK;
}

bh_status bh_fill_multi(bh_hist *const *hs, int32_t nh, const int32_t *col_of_axis, const uint8_t *weighted,
                        int64_t n, const double *const *cols, int32_t ncols, const double *w, bh_stream s) {
    if (!hs || nh < 1 || nh > kMaxHist) return fail(BH_EINVAL, "need 1..%d histograms", kMaxHist);
    if (!col_of_axis || !weighted || !cols) return fail(BH_EINVAL, "NULL argument");
    if (ncols < 1 || ncols > kMaxCols) return fail(BH_EINVAL, "need 1..%d columns", kMaxCols);
    if (n < 0) return fail(BH_EINVAL, "n < 0");
    for (int c = 0; c < ncols; ++c)
        if (!cols[c]) return fail(BH_EINVAL, "cols[%d] is NULL", c);
    int nstats = 0;
    for (int i = 0; i < nh; ++i) {
        if (!hs[i]) return fail(BH_EINVAL, "histogram %d is NULL", i);
        if (bulk_check(hs[i])) return BH_EINVAL;
        if (hs[i]->device != hs[0]->device) return fail(BH_EMISMATCH, "histograms live on different devices");
        for (int j = 0; j < i; ++j)
            if (hs[j] == hs[i]) return fail(BH_EINVAL, "histogram %d appears twice", i);
        if (weighted[i] && !w) return fail(BH_EINVAL, "histogram %d is weighted but w is NULL", i);
        for (int a = 0; a < hs[i]->dim; ++a) {
            const int c = col_of_axis[3 * i + a];
            if (c < 0 || c >= ncols) return fail(BH_EINVAL, "histogram %d axis %d: column %d out of range", i, a, c);
        }
        nstats += hs[i]->K;
    }
    if (n == 0) return BH_OK;
    for (int i = 0; i < nh; ++i)
        if (weighted[i]) hs[i]->weighted_content = true;
    DeviceGuard dg(hs[0]->device);
    cudaStream_t st = static_cast<cudaStream_t>(s);
    // ---- one pass for every histogram (bhist_jit.cu): a kernel specialized to this set,
    // compiled at run time; EXACT / forced-SORT histograms keep passes of their own
    std::vector<int> jit_idx, rest_idx;
    for (int i = 0; i < nh; ++i) {
        const int st = hs[i]->strategy;
        if ((st == BH_STRATEGY_EXACT && weighted[i]) || st == BH_STRATEGY_SORT) rest_idx.push_back(i);
        else jit_idx.push_back(i);
    }
    const bool one_pass = hs[0]->multi_mode == BH_MULTI_ONE_PASS || (hs[0]->debug & BH_DEBUG_REQUIRE_JIT) ||
                          getenv("BHIST_MULTI_ONE_PASS");
    if (one_pass && jit_idx.size() >= 2) {
        bool done = false;
        if (bh_status r = fused_fill(hs, jit_idx.data(), (int)jit_idx.size(), col_of_axis, weighted, n, cols, ncols, w,
                                     st, &done))
            return r;
        if (done) {
            for (int i : rest_idx) {
                const double *cs[kMaxDim] = {};
                for (int a = 0; a < hs[i]->dim; ++a) cs[a] = cols[col_of_axis[3 * i + a]];
                if (bh_status r = fill_device(hs[i], n, cs, weighted[i] ? w : nullptr, st)) return r;
            }
            return BH_OK;
        }
        if (hs[0]->debug & BH_DEBUG_REQUIRE_JIT)
            return fail(BH_ECUDA, "fused one-pass fill unavailable: %s", g_err.c_str());
    }
    // ---- fallback plan.  The single-histogram kernel (k_fill, fully templated) is faster per
    // histogram than the generic fused kernel, and the fill is bound by the bin updates,
    // not by HBM; so fusing only pays when histograms read the SAME columns (e.g. one
    // variable with several binnings): then the fused pass reads them once.  Histograms
    // with a small private state and an identical column set (+ weight flag) are packed
    // into fused passes (k_fill_multi) whose privatized bins, variable-axis tables and
    // per-thread statistics columns fit in shared memory; all others get solo passes.
    const size_t kFuseLimit = 64 * 1024;
    const char *env_t = getenv("BHIST_MULTI_THREADS");
    const int mthreads = env_t ? std::max(128, std::min(1024, atoi(env_t))) / 32 * 32 : kMultiThreads;
    const char *env_s = getenv("BHIST_MULTI_SOLO");
    const bool fuse_off = env_s && atoi(env_s) != 0;
    const char *env_a = getenv("BHIST_MULTI_AGG_UNIT");
    const int agg_unit = env_a ? atoi(env_a) : 0;
    const size_t budget = hs[0]->smem_optin - kStaticSmemReserve;
    struct Cand { int i; size_t bytes; std::vector<int> key; };
    std::vector<int> solo;
    std::vector<Cand> small;
    for (int i = 0; i < nh; ++i) {
        const bh_hist *H = hs[i];
        size_t b = align16((weighted[i] ? 16 : 4) * (size_t)H->G);
        for (int a = 0; a < H->dim; ++a) b += axis_table_bytes(H->ax[a]);
        std::vector<int> key;
        for (int a = 0; a < H->dim; ++a) key.push_back(col_of_axis[3 * i + a]);
        std::sort(key.begin(), key.end());
        key.push_back(weighted[i] ? 1 : 0);
        const bool exact = weighted[i] && H->strategy == BH_STRATEGY_EXACT;
        if (b > kFuseLimit || fuse_off || exact) solo.push_back(i); else small.push_back({i, b, key});
    }
    std::stable_sort(small.begin(), small.end(), [](const Cand &x, const Cand &y) {
        return x.key != y.key ? x.key < y.key : x.bytes < y.bytes; });
    std::vector<std::vector<int>> fused;
    {
        std::vector<int> cur;
        std::vector<int> cur_key;
        size_t used = 0;
        int stats = 0;
        for (const Cand &c : small) {
            const int k = hs[c.i]->K;
            if (!cur.empty() && (c.key != cur_key ||
                                 used + c.bytes + (size_t)(stats + k) * mthreads * 8 > budget)) {
                fused.push_back(cur);
                cur.clear();
                used = 0;
                stats = 0;
            }
            cur.push_back(c.i);
            cur_key = c.key;
            used += c.bytes;
            stats += k;
        }
        if (!cur.empty()) fused.push_back(cur);
    }
    for (auto it = fused.begin(); it != fused.end();) {
        if (it->size() == 1) { solo.push_back((*it)[0]); it = fused.erase(it); } else ++it;
    }
    // ---- solo passes: the single-histogram kernel on this histogram's own columns
    for (int i : solo) {
        const double *cs[kMaxDim] = {};
        for (int a = 0; a < hs[i]->dim; ++a) cs[a] = cols[col_of_axis[3 * i + a]];
        bh_status r = fill_device(hs[i], n, cs, weighted[i] ? w : nullptr, st);
        if (r != BH_OK) return r;
    }
    // ---- fused passes
    for (const std::vector<int> &pass : fused) {
        MultiP p{};
        p.nh = (int32_t)pass.size();
        p.ncols = ncols;
        p.counter = hs[pass[0]]->counter;
        size_t used = 0;
        int stat_off = 0;
        for (int j = 0; j < p.nh; ++j) {
            const int i = pass[j];
            const bh_hist *H = hs[i];
            MultiH &M = p.h[j];
            M.dim = H->dim;
            M.weighted = weighted[i] ? 1 : 0;
            for (int a = 0; a < 3; ++a) M.col[a] = a < H->dim ? col_of_axis[3 * i + a] : 0;
            M.st1 = H->st1;
            M.st2 = H->st2;
            M.G = (int32_t)H->G;
            M.K = H->K;
            M.stat_off = stat_off;
            stat_off += H->K;
            M.smem_off = (int32_t)used;
            used += align16((weighted[i] ? 16 : 4) * (size_t)H->G);
            for (int a = 0; a < H->dim; ++a) {
                M.ax[a] = H->ax[a];
                M.ax[a].tab_off = -1;
                if (M.ax[a].var) {
                    M.ax[a].tab_off = (int32_t)used;
                    used += axis_table_bytes(M.ax[a]);
                }
            }
            M.count = H->count;
            M.sw = H->sw;
            M.stats = H->stats;
            M.partials = H->partials;
            M.entries = H->entries;
        }
        p.nstats = stat_off;
        p.agg_unit = agg_unit;
        p.acc_off = (int32_t)used;
        used += (size_t)stat_off * mthreads * sizeof(double);
        if (used > budget) return fail(BH_EINVAL, "fused pass needs %zu B of shared memory", used);
        auto kern = k_fill_multi;
        CUDA_TRY(ensure_smem(reinterpret_cast<const void *>(kern), used));
        const int64_t kMaxLaunch = int64_t(1) << 30;   // in-kernel event indices are int32
        for (int64_t off = 0; off < n; off += kMaxLaunch) {
            const int64_t m = std::min(kMaxLaunch, n - off);
            p.n = m;
            for (int c = 0; c < ncols; ++c) p.cols[c] = cols[c] + off;
            p.w = w ? w + off : nullptr;
            int64_t grid = (m + mthreads * 4 - 1) / (mthreads * 4);
            grid = std::max<int64_t>(1, std::min<int64_t>(grid, hs[0]->nsm));
            kern<<<(int)grid, mthreads, used, st>>>(p);
            CUDA_TRY(cudaGetLastError());
            hs[pass[0]]->launches++;      // one launch, counted once
        }
    }
    return BH_OK;
}

bh_status bh_fill_expr(bh_hist *h, int64_t n, const double *const *cols, int32_t ncols, const bh_op *prog,
                       int32_t nops, const int32_t *axis_reg, int32_t weight_reg, int32_t filter_reg, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (n < 0) return fail(BH_EINVAL, "n < 0");
    if (ncols < 0 || ncols > kExprRegs) return fail(BH_EINVAL, "need 0..%d columns", kExprRegs);
    if (nops < 0 || nops > kExprOps) return fail(BH_EINVAL, "need 0..%d ops", kExprOps);
    if (nops > 0 && !prog) return fail(BH_EINVAL, "prog is NULL");
    if (!axis_reg) return fail(BH_EINVAL, "axis_reg is NULL");
    if (ncols > 0 && !cols) return fail(BH_EINVAL, "cols is NULL");
    for (int c = 0; c < ncols; ++c)
        if (!cols[c]) return fail(BH_EINVAL, "cols[%d] is NULL", c);
    auto reg_ok = [](int r) { return r >= 0 && r < kExprRegs; };
    ExprP e{};
    e.ncols = ncols;
    e.nops = nops;
    for (int k = 0; k < nops; ++k) {
        const bh_op &o = prog[k];
        if (o.op < 0 || o.op >= EX_COUNT) return fail(BH_EINVAL, "op %d: unknown opcode %d", k, o.op);
        if (!reg_ok(o.dst) || !reg_ok(o.a) || !reg_ok(o.b) || !reg_ok(o.c))
            return fail(BH_EINVAL, "op %d: register out of range [0,%d)", k, kExprRegs);
        e.ins[k] = ExprIns{o.op, o.dst, o.a, o.b, o.c, 0, o.imm};
    }
    for (int a = 0; a < h->dim; ++a) {
        if (!reg_ok(axis_reg[a])) return fail(BH_EINVAL, "axis_reg[%d] out of range", a);
        e.axis_reg[a] = axis_reg[a];
    }
    if (weight_reg >= kExprRegs || filter_reg >= kExprRegs) return fail(BH_EINVAL, "register out of range");
    e.weight_reg = weight_reg < 0 ? -1 : weight_reg;
    if (e.weight_reg >= 0 && n > 0) h->weighted_content = true;
    e.filter_reg = filter_reg < 0 ? -1 : filter_reg;
    if (n == 0) return BH_OK;
    DeviceGuard dg(h->device);
    FillPlan pl;
    if (bh_status r = plan_fill(h, e.weight_reg >= 0, pl, n)) return r;
    LaunchCfg &c = pl.c;
    const int64_t kMaxLaunch = int64_t(1) << 30;
    for (int64_t off = 0; off < n; off += kMaxLaunch) {
        const int64_t m = std::min(kMaxLaunch, n - off);
        for (int k = 0; k < ncols; ++k) e.cols[k] = cols[k] + off;
        const double *none[kMaxDim] = {};
        FillP p = make_params(h, m, none, nullptr);
        for (int a = 0; a < h->dim; ++a) p.ax[a] = pl.ax[a];
        p.entries_add = 0;                 // the kernel adds the passing events itself
        p.cache_slots = cache_slots_for(c.weighted);
        p.replicas = pl.replicas;
        p.wc_off = pl.wc_off;
        c.grid = grid_for(h, c, m);
        cudaError_t r;
        switch (h->dim) {
        case 1: r = c.weighted ? fill_launch_expr<1, true>(p, e, c, static_cast<cudaStream_t>(s))
                           : fill_launch_expr<1, false>(p, e, c, static_cast<cudaStream_t>(s)); break;
        case 2: r = c.weighted ? fill_launch_expr<2, true>(p, e, c, static_cast<cudaStream_t>(s))
                           : fill_launch_expr<2, false>(p, e, c, static_cast<cudaStream_t>(s)); break;
        default: r = c.weighted ? fill_launch_expr<3, true>(p, e, c, static_cast<cudaStream_t>(s))
                           : fill_launch_expr<3, false>(p, e, c, static_cast<cudaStream_t>(s)); break;
        }
        if (r != cudaSuccess) return fail(BH_ECUDA, "fill_expr launch: %s", cudaGetErrorString(r));
        ++h->launches;
    }
    return BH_OK;
}

bh_status bh_find_bins(const bh_hist *h, int64_t n, const double *const *coords, int32_t *out, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (n < 0) return fail(BH_EINVAL, "n < 0");
    if (n == 0) return BH_OK;
    if (!coords || !out) return fail(BH_EINVAL, "NULL pointer");
    for (int a = 0; a < h->dim; ++a)
        if (!coords[a]) return fail(BH_EINVAL, "coords[%d] is NULL", a);
    DeviceGuard dg(h->device);
    FillP p = make_params(h, n, coords, nullptr);
    // the variable-axis search the fills use: tables in shared memory when they fit
    // (BH_DEBUG_FIND_BINS_GLOBAL forces the float64 global-memory search instead)
    size_t tabs = 0;
    bool all3 = true;
    for (int a = 0; a < h->dim; ++a) {
        if (!h->ax[a].var) continue;
        p.ax[a].tab_off = (int32_t)tabs;
        tabs += axis_table_bytes(h->ax[a]);
        all3 &= h->ax[a].g16 == 3;
    }
    int vm = tabs == 0 ? 0 : (tabs + kStaticSmemReserve <= h->smem_optin ? (all3 ? 3 : 1) : 2);
    if (vm && (h->debug & BH_DEBUG_FIND_BINS_GLOBAL)) vm = 2;
    const size_t smem = (vm == 1 || vm == 3) ? tabs : 0;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)h->nsm * (smem ? 2 : 16));
    cudaStream_t st = static_cast<cudaStream_t>(s);
    auto launch = [&](auto kern) -> cudaError_t {
        if (cudaError_t e = ensure_smem(reinterpret_cast<const void *>(kern), smem)) return e;
        kern<<<grid, 256, smem, st>>>(p, out);
        return cudaGetLastError();
    };
    cudaError_t e;
#define BH_FB(D) (vm == 0 ? launch(k_find_bins<D, 0>) : vm == 1 ? launch(k_find_bins<D, 1>) \
                  : vm == 3 ? launch(k_find_bins<D, 3>) : launch(k_find_bins<D, 2>))
    switch (h->dim) {
    case 1: e = BH_FB(1); break;
    case 2: e = BH_FB(2); break;
    default: e = BH_FB(3); break;
    }
#undef BH_FB
    if (e != cudaSuccess) return fail(BH_ECUDA, "find_bins launch: %s", cudaGetErrorString(e));
    const_cast<bh_hist *>(h)->launches++;
    return BH_OK;
}

bh_status bh_info(const bh_hist *h, int32_t *dim, int64_t *nbins_total, int32_t *nstats) {
    if (check_hist(h)) return BH_EINVAL;
    if (dim) *dim = h->dim;
    if (nbins_total) *nbins_total = h->G;
    if (nstats) *nstats = h->K;
    return BH_OK;
}

bh_status bh_packed_size(const bh_hist *h, int64_t *n_doubles) {
    if (check_hist(h)) return BH_EINVAL;
    if (!n_doubles) return fail(BH_EINVAL, "NULL output");
    *n_doubles = 2 * h->G + h->K + 1;
    return BH_OK;
}

bh_status bh_pack(const bh_hist *h, double *dev_out, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (!dev_out) return fail(BH_EINVAL, "NULL output");
    DeviceGuard dg(h->device);
    const int64_t tot = 2 * h->G + h->K + 1;
    const int grid = (int)std::min<int64_t>((tot + 255) / 256, (int64_t)h->nsm * 8);
    k_pack<<<grid, 256, 0, static_cast<cudaStream_t>(s)>>>((int)h->G, h->K, h->count, h->sw, h->stats,
                                                            h->entries, dev_out);
    CUDA_TRY(cudaGetLastError());
    const_cast<bh_hist *>(h)->launches++;
    return BH_OK;
}

bh_status bh_unpack(bh_hist *h, const double *dev_in, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    if (!dev_in) return fail(BH_EINVAL, "NULL input");
    DeviceGuard dg(h->device);
    const int64_t tot = 2 * h->G + h->K + 1;
    const int grid = (int)std::min<int64_t>((tot + 255) / 256, (int64_t)h->nsm * 8);
    k_unpack<<<grid, 256, 0, static_cast<cudaStream_t>(s)>>>((int)h->G, h->K, h->count, h->sw, h->stats,
                                                              h->entries, dev_in);
    CUDA_TRY(cudaGetLastError());
    h->launches++;
    h->weighted_content = true;          // sumw2 now comes from the buffer
    return BH_OK;
}

}  // extern "C"

namespace {
bh_status pack_plan(bh_hist *const *hs, int32_t nh, const uint8_t *unit, PackMultiP &p, bool packing) {
    if (!hs || nh < 1 || nh > kMaxPack) return fail(BH_EINVAL, "need 1..%d histograms", kMaxPack);
    p = PackMultiP{};
    p.nh = nh;
    int64_t off = 0;
    for (int i = 0; i < nh; ++i) {
        bh_hist *h = hs[i];
        if (!h) return fail(BH_EINVAL, "histogram %d is NULL", i);
        if (h->device != hs[0]->device) return fail(BH_EMISMATCH, "histograms live on different devices");
        const bool u = unit && unit[i];
        if (u && packing && h->weighted_content)
            return fail(BH_EINVAL, "histogram %d holds weighted fills: it cannot be packed without sumw2", i);
        PackDesc &D = p.d[i];
        D.off = off;
        D.G = (int32_t)h->G;
        D.K = h->K;
        D.unit = u ? 1 : 0;
        D.count = h->count;
        D.sw = h->sw;
        D.stats = h->stats;
        D.entries = h->entries;
        off += (u ? 1 : 2) * h->G + h->K + 1;
    }
    p.total = off;
    return BH_OK;
}
}  // namespace

extern "C" {

bh_status bh_packed_size_multi(bh_hist *const *hs, int32_t nh, const uint8_t *unit, int64_t *n_doubles) {
    if (!n_doubles) return fail(BH_EINVAL, "NULL output");
    PackMultiP p;
    if (bh_status r = pack_plan(hs, nh, unit, p, false)) return r;
    *n_doubles = p.total;
    return BH_OK;
}

bh_status bh_pack_multi(bh_hist *const *hs, int32_t nh, const uint8_t *unit, double *dev_out, bh_stream s) {
    if (!dev_out) return fail(BH_EINVAL, "NULL output");
    PackMultiP p;
    if (bh_status r = pack_plan(hs, nh, unit, p, true)) return r;
    DeviceGuard dg(hs[0]->device);
    const int grid = (int)std::min<int64_t>((p.total + 255) / 256, (int64_t)hs[0]->nsm * 8);
    k_pack_multi<<<grid, 256, 0, static_cast<cudaStream_t>(s)>>>(p, dev_out);
    CUDA_TRY(cudaGetLastError());
    hs[0]->launches++;
    return BH_OK;
}

bh_status bh_unpack_multi(bh_hist *const *hs, int32_t nh, const uint8_t *unit, const double *dev_in, bh_stream s) {
    if (!dev_in) return fail(BH_EINVAL, "NULL input");
    PackMultiP p;
    if (bh_status r = pack_plan(hs, nh, unit, p, false)) return r;
    DeviceGuard dg(hs[0]->device);
    const int grid = (int)std::min<int64_t>((p.total + 255) / 256, (int64_t)hs[0]->nsm * 8);
    k_unpack_multi<<<grid, 256, 0, static_cast<cudaStream_t>(s)>>>(p, dev_in);
    CUDA_TRY(cudaGetLastError());
    hs[0]->launches++;
    for (int i = 0; i < nh; ++i)
        if (!(unit && unit[i])) hs[i]->weighted_content = true;
    return BH_OK;
}

bh_status bh_read(const bh_hist *h, double *contents, double *sumw2, double *stats, int64_t *entries, bh_stream s) {
    if (bulk_check(h)) return BH_EINVAL;
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(s);
    bh_status r = bh_pack(h, h->pack_buf, s);
    if (r != BH_OK) return r;
    const int64_t tot = 2 * h->G + h->K + 1;
    CUDA_TRY(cudaMemcpyAsync(h->pack_host, h->pack_buf, sizeof(double) * tot, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (contents) memcpy(contents, h->pack_host, sizeof(double) * h->G);
    if (sumw2) memcpy(sumw2, h->pack_host + h->G, sizeof(double) * h->G);
    if (stats) memcpy(stats, h->pack_host + 2 * h->G, sizeof(double) * h->K);
    if (entries) *entries = (int64_t)h->pack_host[2 * h->G + h->K];
    return BH_OK;
}

bh_status bh_read_as(const bh_hist *h, int32_t type, void *contents, void *sumw2, double *stats, int64_t *entries,
                     bh_stream s) {
    if (type == BH_CONTENT_F64)
        return bh_read(h, static_cast<double *>(contents), static_cast<double *>(sumw2), stats, entries, s);
    if (type != BH_CONTENT_F32 && type != BH_CONTENT_I32) return fail(BH_EINVAL, "unknown content type %d", type);
    if (bulk_check(h)) return BH_EINVAL;
    if (type == BH_CONTENT_I32 && h->weighted_content)
        return fail(BH_EINVAL, "int32 (TH1I) contents need unit-weight fills only: this histogram holds weighted sums");
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(s);
    bh_status r = bh_pack(h, h->pack_buf, s);
    if (r != BH_OK) return r;
    const int64_t G = h->G, tot = 2 * G + h->K + 1;
    // the narrowed [content | sumw2] (8 B per bin) goes to lazily allocated device + pinned buffers
    bh_hist *hm = const_cast<bh_hist *>(h);
    if (!hm->narrow_buf) {
        if (cudaMalloc(reinterpret_cast<void **>(&hm->narrow_buf), 8 * (size_t)G) != cudaSuccess ||
            cudaMallocHost(reinterpret_cast<void **>(&hm->narrow_host), 8 * (size_t)G) != cudaSuccess) {
            cudaGetLastError();
            return fail(BH_ENOMEM, "narrow read buffers (%lld B)", (long long)(8 * G));
        }
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((2 * G + 255) / 256, (int64_t)h->nsm * 8));
    k_narrow<<<grid, 256, 0, st>>>((int)G, type, h->pack_buf, hm->narrow_buf);
    CUDA_TRY(cudaGetLastError());
    hm->launches++;
    CUDA_TRY(cudaMemcpyAsync(hm->narrow_host, hm->narrow_buf, 8 * (size_t)G, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h->pack_host + 2 * G, h->pack_buf + 2 * G, sizeof(double) * (h->K + 1),
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (contents) memcpy(contents, hm->narrow_host, 4 * (size_t)G);
    if (sumw2) memcpy(sumw2, hm->narrow_host + 4 * (size_t)G, 4 * (size_t)G);
    if (stats) memcpy(stats, h->pack_host + 2 * G, sizeof(double) * h->K);
    if (entries) *entries = (int64_t)h->pack_host[tot - 1];
    return BH_OK;
}

bh_status bh_set_strategy(bh_hist *h, int32_t strategy) {
    if (bulk_check(h)) return BH_EINVAL;
    if (strategy < BH_STRATEGY_AUTO || strategy > BH_STRATEGY_SORT) return fail(BH_EINVAL, "unknown strategy %d", strategy);
    if (strategy == BH_STRATEGY_PRIV && 4 * (size_t)h->G + kStaticSmemReserve > h->smem_optin)
        return fail(BH_EINVAL, "PRIV cannot hold %lld bins in shared memory", (long long)h->G);
    if (strategy == BH_STRATEGY_SORT && sort_partitions(h, false) > kPartMaxP)
        return fail(BH_EINVAL, "SORT supports at most %d partitions of 2^%d bins", kPartMaxP, sort_pb(false));
    h->strategy = strategy;
    return BH_OK;
}

bh_status bh_get_strategy(const bh_hist *h, int32_t weighted, int32_t *strategy) {
    if (check_hist(h)) return BH_EINVAL;
    if (!strategy) return fail(BH_EINVAL, "NULL output");
    *strategy = (weighted && h->strategy == BH_STRATEGY_EXACT) ? BH_STRATEGY_EXACT : resolve_strategy(h, weighted != 0);
    // AUTO's large fills after the probe decided (on the device) for SORT (unit weights) or
    // GLOBAL (weights)
    if (h->strategy == BH_STRATEGY_AUTO && *strategy == BH_STRATEGY_CACHE && h->probe_state != 0 && h->probe_dev) {
        DeviceGuard dg(h->device);
        unsigned int flag = 0;
        if (cudaMemcpy(&flag, h->probe_dev + (weighted ? 3 : 2), sizeof flag, cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(BH_ECUDA, "reading the AUTO decision: %s", cudaGetErrorString(cudaGetLastError()));
        if (flag == 1) *strategy = weighted ? BH_STRATEGY_GLOBAL : BH_STRATEGY_SORT;
    }
    return BH_OK;
}

bh_status bh_set_chunk(bh_hist *h, int64_t events) {
    if (check_hist(h)) return BH_EINVAL;
    if (events < 1024) return fail(BH_EINVAL, "chunk must be >= 1024 events");
    h->chunk = events;
    return BH_OK;
}

bh_status bh_set_debug(bh_hist *h, int32_t flags) {
    if (check_hist(h)) return BH_EINVAL;
    h->debug = flags;
    return BH_OK;
}

bh_status bh_set_multi_mode(bh_hist *h, int32_t mode) {
    if (check_hist(h)) return BH_EINVAL;
    if (mode != BH_MULTI_PASSES && mode != BH_MULTI_ONE_PASS) return fail(BH_EINVAL, "unknown multi mode %d", mode);
    h->multi_mode = mode;
    return BH_OK;
}

bh_status bh_launch_count(const bh_hist *h, int64_t *count) {
    if (check_hist(h)) return BH_EINVAL;
    if (!count) return fail(BH_EINVAL, "NULL output");
    *count = h->launches;
    return BH_OK;
}

}  // extern "C"
