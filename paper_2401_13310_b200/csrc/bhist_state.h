// bhist_state.h — the opaque bh_hist of include/bhist.h (host-side; shared by the
// translation units of the library's host code: bhist.cu and bhist_jit.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/bhist.h"
#include "bhist_kernels.cuh"
#include "bhist_bulk.cuh"

constexpr int kStageSlots = 2;

struct bh_hist {
    int device = 0;
    int dim = 0;
    int nsm = 148;
    int K = 0;
    int64_t G = 0;
    bh::AxisP ax[bh::kMaxDim] = {};
    int32_t st1 = 1, st2 = 1;
    int strategy = BH_STRATEGY_AUTO;
    int debug = 0;
    int multi_mode = BH_MULTI_PASSES;   // bh_fill_multi plan when this histogram is hs[0]
    int64_t chunk = 1 << 22;
    int64_t launches = 0;
    size_t smem_optin = 0;
    int max_grid = 0;
    // device state
    unsigned long long *count = nullptr;
    double *sw = nullptr;             // interleaved (sum w, sum w^2) per bin [2G]
    double *stats = nullptr;
    unsigned long long *entries = nullptr;
    double *partials = nullptr;
    unsigned int *counter = nullptr;
    long long *limbs = nullptr;       // EXACT: per bin 2 x kLimbs int64 limbs (sumw, sumw2), zero between fills
    unsigned long long *maxbits = nullptr;   // EXACT: bit pattern of max|w| of the current launch
    double *pack_buf = nullptr;       // device buffer for bh_read
    double *pack_host = nullptr;      // pinned host buffer for bh_read
    void *narrow_buf = nullptr;       // bh_read_as: device [content | sumw2] as float32 / int32 [2G]
    unsigned char *narrow_host = nullptr;   // its pinned host twin
    // SORT strategy scratch (grown on demand): records, segment offsets, partition totals
    uint16_t *part_l = nullptr;
    double *part_w = nullptr;
    uint32_t *part_offs = nullptr;
    unsigned long long *part_cnt = nullptr, *part_cp = nullptr;
    int64_t part_cap_l = 0, part_cap_w = 0, part_cap_offs = 0;
    int part_P = 0;
    // AUTO's SORT decision for large unit-weight fills: 0 not probed since create/reset,
    // 1 probed (probe_dev[2] on the device: 1 SORT, 0 CACHE; both paths are launched gated)
    int probe_state = 0;
    // AUTO's lane-private hot-cell window for large weighted PRIVA fills (k_hot_probe):
    // 0 not probed since create/reset, 1 probed (hot_dev->flag on the device gates the kernels)
    bh::HotTab *hot_dev = nullptr;
    int hot_state = 0;
    // state 2 (after bh_reset): the decision stands for a fill over the SAME input buffers and
    // size (probe_key / hot_key), and is re-probed for any other
    uint64_t probe_key = 0, hot_key = 0;
    unsigned int *probe_dev = nullptr;
    std::vector<void *> axis_mem;     // edges and guide tables
    // host->device double buffer
    cudaStream_t copy_stream = nullptr;
    double *stage[kStageSlots] = {};  // each slot: (dim+1) columns of `chunk` doubles
    int64_t stage_chunk = 0;
    cudaEvent_t copied[kStageSlots] = {}, consumed[kStageSlots] = {};
    bool weighted_content = false;     // a weighted fill (or a full unpack) since create/reset
    bool slot_used[kStageSlots] = {};  // consumed[slot] recorded at least once (persists across calls)
    int next_slot = 0;                 // ring position (persists across calls)
    // persistent bulk consumer (bh_bulk_*; bhist_bulk.cuh)
    bh::BulkCtl *bulk_ctl = nullptr;                 // pinned, mapped host memory
    bh::BulkDev *bulk_dev = nullptr;                 // device: arrivals + the forwarded descriptors
    double *bulk_stage[bh::kBulkRing] = {};          // pinned copies of pageable bulks, per ring slot
    int64_t bulk_stage_cap = 0;                      // doubles per staging slot
    bool bulk_active = false, bulk_weighted = false;
    long long bulk_seq = 0;                          // bulks posted in this session
    long long bulk_timeout_ns = 0;
    cudaStream_t bulk_stream = nullptr;              // the caller's stream of the session
    cudaStream_t bulk_kstream = nullptr;             // the library's stream the resident kernel runs on
    cudaEvent_t bulk_ev[2] = {};                     // [0] caller's work before begin, [1] kernel done
};

namespace bh {
// The one-pass fused multi-histogram fill of bh_fill_multi (bhist_jit.cu): a kernel
// specialized to this histogram set, compiled at run time with NVRTC and cached.
// Returns BH_OK with *done = true when it filled every histogram in idx[0..m); *done =
// false (and BH_OK) when the set cannot take the fused path (NVRTC unavailable, ...).
bh_status fused_fill(bh_hist *const *hs, const int *idx, int m, const int32_t *col_of_axis,
                     const uint8_t *weighted, int64_t n, const double *const *cols, int32_t ncols,
                     const double *w, cudaStream_t s, bool *done);
bh_status set_error(bh_status st, const char *msg);
size_t axis_table_bytes_of(const AxisP &a);
}  // namespace bh
