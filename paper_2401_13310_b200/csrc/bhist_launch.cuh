// bhist_launch.cuh — host-side launch dispatch for the templated fill kernels.
//
// The fill templates (k_fill, k_fill_f32, k_fill_expr, k_part_scatter) have a few
// hundred instantiations; each (DIM, weighted) pair is compiled in its own translation
// unit (bhist_fill_d<DIM><u|w>.cu, built in parallel) behind the plain functions
// declared at the bottom, which bhist.cu calls.
#pragma once
#include <cuda_runtime.h>

#include "../../include/bhist.h"
#include "bhist_kernels.cuh"
#include "bhist_sort.cuh"
#include "bhist_bulk.cuh"

#include <mutex>
#include <unordered_map>

namespace bh {

// cudaFuncSetAttribute is a driver call (~microseconds); small fills are launch-latency
// bound, so the dynamic shared-memory limit is raised once per (kernel, device).
inline cudaError_t ensure_smem(const void *kern, size_t bytes) {
    // the 48 KB default covers dynamic + static shared memory together, so anything above
    // ~40 KB of dynamic memory needs the opt-in (kernels carry a few KB of static smem)
    if (bytes <= 32 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::unordered_map<uint64_t, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t key = reinterpret_cast<uint64_t>(kern) * 64u + (uint64_t)dev;
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done[key] = bytes;
    return e;
}

struct LaunchCfg {
    int strategy;
    bool weighted, vec, vsm;
    int vm;                      // 0 fixed axes only, 1 variable tables in smem, 2 in global, 3 smem + all
                                 // variable axes compact (k_fill only; the other kernels take 1)
    int grid;
    size_t smem;
};

template <int DIM, bool W, int SINK, bool VEC, int VM>
cudaError_t launch_t(const FillP &p, const LaunchCfg &c, cudaStream_t s) {
    auto kern = k_fill<DIM, W, SINK, VEC, VM>;
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void *>(kern), c.smem)) return e;
    kern<<<c.grid, FillThreads<SINK, DIM, W>::v, c.smem, s>>>(p);
    return cudaGetLastError();
}

template <int DIM, bool W, int SINK, bool VEC>
cudaError_t launch_m(const FillP &p, const LaunchCfg &c, cudaStream_t s) {
    switch (c.vm) {
    case 0: return launch_t<DIM, W, SINK, VEC, 0>(p, c, s);
    case 1: return launch_t<DIM, W, SINK, VEC, 1>(p, c, s);
    case 3: return launch_t<DIM, W, SINK, VEC, 3>(p, c, s);
    default: return launch_t<DIM, W, SINK, VEC, 2>(p, c, s);
    }
}

template <int DIM, bool W, int SINK>
cudaError_t launch_v(const FillP &p, const LaunchCfg &c, cudaStream_t s) {
    return c.vec ? launch_m<DIM, W, SINK, true>(p, c, s) : launch_m<DIM, W, SINK, false>(p, c, s);
}

template <int DIM, bool W>
cudaError_t launch_s(const FillP &p, const LaunchCfg &c, cudaStream_t s) {
    switch (c.strategy) {
    case BH_STRATEGY_PRIV:
        if constexpr (W) {
            if (p.wc_off >= 0) return launch_v<DIM, W, SINK_PRIVA>(p, c, s);
        }
        return launch_v<DIM, W, SINK_PRIV>(p, c, s);
    case BH_STRATEGY_CACHE: return launch_v<DIM, W, SINK_CACHE>(p, c, s);
    default: return launch_v<DIM, W, SINK_GLOBAL>(p, c, s);
    }
}


template <int DIM, bool W, int VM, int RC>
cudaError_t launch_part1(const FillP &p, const PartP &q, int grid, size_t smem, cudaStream_t s) {
    auto kern = k_part_scatter<DIM, W, VM, RC>;
    if (cudaError_t e = ensure_smem(reinterpret_cast<const void *>(kern), smem)) return e;
    kern<<<grid, kPartThreads, smem, s>>>(p, q);
    return cudaGetLastError();
}

template <int DIM, bool W, int RC>
cudaError_t launch_part1_r(const FillP &p, const PartP &q, int vm, int grid, size_t smem, cudaStream_t s) {
    return vm == 0 ? launch_part1<DIM, W, 0, RC>(p, q, grid, smem, s)
                   : vm == 1 ? launch_part1<DIM, W, 1, RC>(p, q, grid, smem, s) : launch_part1<DIM, W, 2, RC>(p, q, grid, smem, s);
}

template <int DIM, bool W>
cudaError_t launch_part1_v(const FillP &p, const PartP &q, int vm, int rc, int grid, size_t smem, cudaStream_t s) {
    if (rc == 1) return launch_part1_r<DIM, W, 1>(p, q, vm, grid, smem, s);
    if constexpr (W) return launch_part1_r<DIM, W, 4>(p, q, vm, grid, smem, s);
    else return launch_part1_r<DIM, W, 8>(p, q, vm, grid, smem, s);
}

template <int DIM, bool W, int SINK, typename CT>
cudaError_t launch_f32_s(const FillP &p, const LaunchCfg &c, cudaStream_t s) {
    auto kern = c.vm == 0 ? k_fill_f32<DIM, W, SINK, 0, CT>
                          : (c.vm == 1 || c.vm == 3) ? k_fill_f32<DIM, W, SINK, 1, CT> : k_fill_f32<DIM, W, SINK, 2, CT>;
    if (cudaError_t r = ensure_smem(reinterpret_cast<const void *>(kern), c.smem)) return r;
    kern<<<c.grid, ThreadsOf<SINK>::v, c.smem, s>>>(p);
    return cudaGetLastError();
}

template <int DIM, bool W, typename CT>
cudaError_t launch_f32_w(const FillP &p, const LaunchCfg &c, cudaStream_t s) {
    switch (c.strategy) {
    case BH_STRATEGY_PRIV:
        if constexpr (W) {
            if (p.wc_off >= 0) return launch_f32_s<DIM, W, SINK_PRIVA, CT>(p, c, s);
        }
        return launch_f32_s<DIM, W, SINK_PRIV, CT>(p, c, s);
    case BH_STRATEGY_CACHE: return launch_f32_s<DIM, W, SINK_CACHE, CT>(p, c, s);
    default: return launch_f32_s<DIM, W, SINK_GLOBAL, CT>(p, c, s);
    }
}


template <int DIM, bool W, int SINK>
cudaError_t launch_expr_s(const FillP &p, const ExprP &e, const LaunchCfg &c, cudaStream_t s) {
    auto kern = c.vm == 0 ? k_fill_expr<DIM, W, SINK, 0>
                          : (c.vm == 1 || c.vm == 3) ? k_fill_expr<DIM, W, SINK, 1> : k_fill_expr<DIM, W, SINK, 2>;
    if (cudaError_t r = ensure_smem(reinterpret_cast<const void *>(kern), c.smem)) return r;
    kern<<<c.grid, ThreadsOf<SINK>::v, c.smem, s>>>(p, e);
    return cudaGetLastError();
}

template <int DIM, bool W>
cudaError_t launch_expr_w(const FillP &p, const ExprP &e, const LaunchCfg &c, cudaStream_t s) {
    switch (c.strategy) {
    case BH_STRATEGY_PRIV:
        if constexpr (W) {
            if (p.wc_off >= 0) return launch_expr_s<DIM, W, SINK_PRIVA>(p, e, c, s);
        }
        return launch_expr_s<DIM, W, SINK_PRIV>(p, e, c, s);
    case BH_STRATEGY_CACHE: return launch_expr_s<DIM, W, SINK_CACHE>(p, e, c, s);
    default: return launch_expr_s<DIM, W, SINK_GLOBAL>(p, e, c, s);
    }
}


template <int DIM, bool W, int SINK>
cudaError_t launch_bulk_s(const FillP &p, const LaunchCfg &c, BulkCtl *ctl, BulkDev *dev,
                          long long timeout_ns, int stage_off, int te, cudaStream_t s) {
    auto kern = c.vm == 0 ? k_bulk<DIM, W, SINK, 0>
                          : c.vm == 1 ? k_bulk<DIM, W, SINK, 1> : c.vm == 3 ? k_bulk<DIM, W, SINK, 3> : k_bulk<DIM, W, SINK, 2>;
    if (cudaError_t r = ensure_smem(reinterpret_cast<const void *>(kern), c.smem)) return r;
    // every CTA must be resident at once (each takes a share of every bulk): c.grid is the SM
    // count, times the CTAs per SM the kernel's shared memory and registers allow
    int per_sm = 0;
    if (cudaError_t r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ThreadsOf<SINK>::v, c.smem)) return r;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    kern<<<c.grid * per_sm, ThreadsOf<SINK>::v, c.smem, s>>>(p, ctl, dev, timeout_ns, stage_off, te);
    return cudaGetLastError();
}

template <int DIM, bool W>
cudaError_t launch_bulk_w(const FillP &p, const LaunchCfg &c, BulkCtl *ctl, BulkDev *dev,
                          long long timeout_ns, int stage_off, int te, cudaStream_t s) {
    switch (c.strategy) {
    case BH_STRATEGY_PRIV:
        if constexpr (W) {
            if (p.wc_off >= 0) return launch_bulk_s<DIM, W, SINK_PRIVA>(p, c, ctl, dev, timeout_ns, stage_off, te, s);
        }
        return launch_bulk_s<DIM, W, SINK_PRIV>(p, c, ctl, dev, timeout_ns, stage_off, te, s);
    case BH_STRATEGY_CACHE: return launch_bulk_s<DIM, W, SINK_CACHE>(p, c, ctl, dev, timeout_ns, stage_off, te, s);
    default: return launch_bulk_s<DIM, W, SINK_GLOBAL>(p, c, ctl, dev, timeout_ns, stage_off, te, s);
    }
}

// one definition per (DIM, W) in bhist_fill_d<DIM><u|w>.cu
template <int DIM, bool W> cudaError_t fill_launch(const FillP &p, const LaunchCfg &c, cudaStream_t s);
template <int DIM, bool W> cudaError_t fill_launch_f32(const FillP &p, const LaunchCfg &c, cudaStream_t s);
template <int DIM, bool W> cudaError_t fill_launch_i32(const FillP &p, const LaunchCfg &c, cudaStream_t s);
template <int DIM, bool W> cudaError_t fill_launch_expr(const FillP &p, const ExprP &e, const LaunchCfg &c, cudaStream_t s);
template <int DIM, bool W> cudaError_t fill_launch_part1(const FillP &p, const PartP &q, int vm, int rc, int grid, size_t smem, cudaStream_t s);
template <int DIM, bool W> cudaError_t fill_launch_bulk(const FillP &p, const LaunchCfg &c, BulkCtl *ctl,
                                                        BulkDev *dev, long long timeout_ns, int stage_off, int te,
                                                        cudaStream_t s);

#define BH_DEFINE_FILL_TU(DIM, W)                                                                          \
    template <> cudaError_t fill_launch<DIM, W>(const FillP &p, const LaunchCfg &c, cudaStream_t s) {      \
        return launch_s<DIM, W>(p, c, s);                                                                  \
    }                                                                                                      \
    template <> cudaError_t fill_launch_f32<DIM, W>(const FillP &p, const LaunchCfg &c, cudaStream_t s) {  \
        return launch_f32_w<DIM, W, float>(p, c, s);                                                       \
    }                                                                                                      \
    template <> cudaError_t fill_launch_i32<DIM, W>(const FillP &p, const LaunchCfg &c, cudaStream_t s) {  \
        return launch_f32_w<DIM, W, int32_t>(p, c, s);                                                     \
    }                                                                                                      \
    template <> cudaError_t fill_launch_expr<DIM, W>(const FillP &p, const ExprP &e, const LaunchCfg &c,   \
                                                     cudaStream_t s) {                                     \
        return launch_expr_w<DIM, W>(p, e, c, s);                                                          \
    }                                                                                                      \
    template <> cudaError_t fill_launch_part1<DIM, W>(const FillP &p, const PartP &q, int vm, int rc,      \
                                                      int grid, size_t smem, cudaStream_t s) {             \
        return launch_part1_v<DIM, W>(p, q, vm, rc, grid, smem, s);                                        \
    }                                                                                                      \
    template <> cudaError_t fill_launch_bulk<DIM, W>(const FillP &p, const LaunchCfg &c, BulkCtl *ctl,     \
                                                     BulkDev *dev, long long timeout_ns, int stage_off,    \
                                                     int te, cudaStream_t s) {                             \
        return launch_bulk_w<DIM, W>(p, c, ctl, dev, timeout_ns, stage_off, te, s);                                    \
    }

}  // namespace bh
