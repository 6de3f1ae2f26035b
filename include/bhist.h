/* bhist.h — C ABI of libbhist: B200-native (sm_100a) bulk histogram filling.
 *
 * The operation (arXiv 2401.13310, §3.1): filling a histogram
 * with a bulk of events is three steps per event — (1) find the bin from the
 * coordinate(s), (2) increment that bin by one or by the event weight, (3) update
 * the statistics sums.  The paper's GPU version keeps the histogram in device
 * memory across bulks (RHnCUDA), "transfers bulk of events to the
 * GPU and launches kernels ... per bulk", and copies the result back "once all
 * bulks have been processed".  This header exposes exactly that
 * life cycle: create from axes, fill bulks on a stream, read back bins and stats.
 *
 * Conventions (DESIGN.md "Readings" R1–R17 give the paper passages):
 *  - Axis bins: 0 = underflow, 1..nbins in range, nbins+1 = overflow.
 *    Fixed axis: b = 1 + (int)((nbins*(x-xmin))/(xmax-xmin)) in IEEE binary64
 *    with that association (R2); x < xmin -> 0; !(x < xmax) -> nbins+1 (so
 *    x == xmax and NaN go to overflow, R5).  Variable axis: b = number of edges
 *    <= x (half-open [e_{i-1}, e_i), R1), with the same flow routing.
 *  - Global bin: g = b0 + (n0+2)*(b1 + (n1+2)*b2), axis 0 fastest (R9).
 *  - Per bin: content = sum of w, sumw2 = sum of w*w (w = 1 for unit fills).
 *  - Stats (ROOT GetStats order, R7/R8), over events whose bin is in range on
 *    every axis (R6):  1D [sumw, sumw2, sumwx, sumwx2]
 *                      2D + [sumwy, sumwy2, sumwxy]
 *                      3D + [sumwz, sumwz2, sumwxz, sumwyz]
 *  - entries += n for every fill (all events, flow included).
 *  - Fills accumulate into the existing state (include-initial).
 *
 * Ownership: the library owns all histogram storage (allocated on `device` at
 * bh_create, freed at bh_destroy).  Input buffers are borrowed: device pointers
 * must stay valid and unmodified until the stream has executed the fill.
 * Streams: `bh_stream` is a cudaStream_t passed as an opaque pointer (NULL = the
 * legacy default stream).  No call synchronizes the device; bh_read synchronizes
 * only its stream; bh_fill_host waits only for its own host->device copies; a fill
 * that needs more SORT scratch than the histogram holds (BH_STRATEGY_SORT below)
 * synchronizes its stream once to grow it.  A histogram is single-writer: issue
 * its fills on one stream at a time.
 * Errors: every call returns a bh_status; no exception crosses the ABI;
 * bh_last_error() gives a thread-local message for the last failure.  NaN/inf
 * coordinates and any weight value are not errors.  Asynchronous kernel faults
 * surface as BH_ECUDA at the next call that synchronizes (bh_read).
 */
#ifndef BHIST_H
#define BHIST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bh_hist bh_hist; /* opaque; owns its device storage on one device */
typedef void *bh_stream;        /* cudaStream_t */
typedef int32_t bh_status;

#define BH_OK 0
#define BH_EINVAL (-1)    /* invalid argument (axes, sizes, NULL pointers, ...) */
#define BH_ENOMEM (-2)    /* device or pinned-host allocation failed */
#define BH_ECUDA (-3)     /* CUDA runtime error (launch, copy, asynchronous fault) */
#define BH_EDEVICE (-4)   /* bad device ordinal / no device */
#define BH_EMISMATCH (-5) /* incompatible histograms (bh_fill_multi) */

/* One axis.  Fixed: edges == NULL, xmin < xmax finite, nbins*(xmax-xmin) finite.
 * Variable: edges = HOST pointer to nbins+1 strictly increasing finite doubles
 * (copied at bh_create; xmin/xmax ignored).  nbins >= 1.  The product of
 * (nbins_a + 2) over all axes must be < 2^31. */
typedef struct {
    int32_t nbins;
    double xmin;
    double xmax;
    const double *edges;
} bh_axis;

/* Fill strategies (bh_set_strategy).  AUTO picks by bin-space size and weights:
 * PRIV   block-private shared-memory bins, flushed once per CTA (PAPER.md:138,
 *        "each block fills a local copy ... in shared memory"); bh_set_strategy accepts it
 *        when the unit-weight bins (4 B each) fit; weighted fills whose 16-B cells do not
 *        fit then use CACHE;
 * GLOBAL device-wide atomics straight into the L2-resident histogram;
 * CACHE  per-CTA shared-memory cache of the hottest bins with global fallback
 *        (hot-bin contention, BASELINE.json config 4). */
#define BH_STRATEGY_AUTO 0
#define BH_STRATEGY_PRIV 1
#define BH_STRATEGY_GLOBAL 2
#define BH_STRATEGY_CACHE 3
/* EXACT  weighted fills of bh_fill / bh_fill_host / bh_fill_multi (solo passes) add
 *        each launch's per-bin sums of w and w*w as exact scaled-integer sums (int64
 *        limbs, order independent) rounded once: bitwise reproducible run to run, and
 *        the correctly rounded sum whenever the weights lie within 2^43 of the launch's
 *        max|w|.  Unit-weight fills are exact in every mode;
 *        bh_fill_expr uses AUTO.  Slower (six L2 integer atomics per event). */
#define BH_STRATEGY_EXACT 4
/* SORT   two-pass partitioned fill for bin spaces too large for PRIV (faster than CACHE
 *        on spread-out unit-weight data, slower on peaked or weighted data: AUTO uses it
 *        only for unit-weight fills of >= ~39M events once an asynchronous probe of a
 *        sample of an earlier such fill found no partition holding > 5% of the events;
 *        bh_get_strategy then reports SORT for unit weights): pass 1 bins each event, accumulates the stats and writes a record
 *        (bin mod 2^pb, w) into a partition-sorted scratch buffer (p = bin >> pb,
 *        pb = 15 unit / 13 weighted; at most 2048 partitions); pass 2 reduces each
 *        partition in shared memory and adds it to the bins once per CTA.  The
 *        "sort-then-segmented-reduce" path for large 2D/3D bin spaces.  Scratch of
 *        2 (unit) or 10 (weighted) bytes per event of a chunk (<= 2^28 / 2^26 events)
 *        is allocated by the histogram on first use.  bh_fill_f32 and bh_fill_expr
 *        use CACHE instead. */
#define BH_STRATEGY_SORT 5

/* Debug flags (bh_set_debug) — negative controls for tests only. */
#define BH_DEBUG_SKIP_COPY_WAIT 1 /* bh_fill_host: fill without waiting for the H2D copy (PAPER.md:223 race) */
#define BH_DEBUG_FIND_BINS_GLOBAL 2 /* bh_find_bins: search variable axes in global memory, not the fills' staged tables */
#define BH_DEBUG_REQUIRE_JIT 4      /* bh_fill_multi (flag on hs[0]): use the one-pass kernel and fail instead
                                       of falling back when the run-time compiled kernel is unavailable */

/* ABI version (major*10000 + minor*100 + patch). */
int32_t bh_version(void);

/* Thread-local, NUL-terminated message describing the last failing call ("" if none). */
const char *bh_last_error(void);

/* Create a dim-D histogram (dim in {1,2,3}) from `axes[dim]` on CUDA `device`.
 * State starts zeroed.  *out receives the handle.  Errors: BH_EINVAL, BH_EDEVICE,
 * BH_ENOMEM, BH_ECUDA.  Synchronous (allocations + table build). */
bh_status bh_create(int32_t dim, const bh_axis *axes, int32_t device, bh_hist **out);

/* Free all storage.  NULL is accepted.  Synchronizes the device the histogram lives on. */
bh_status bh_destroy(bh_hist *h);

/* Zero bins, sumw2, stats and entries (stream-ordered on s). */
bh_status bh_reset(bh_hist *h, bh_stream s);

/* Fill n events (PAPER.md:126 three steps).  coords: array of `dim` DEVICE
 * pointers, coords[a][i] = coordinate of event i on axis a (float64, SoA).
 * w: DEVICE pointer to n float64 weights, or NULL for unit weights.  Async on s.
 * n == 0 is a no-op.  Errors: BH_EINVAL (n < 0, NULL coords), BH_ECUDA. */
bh_status bh_fill(bh_hist *h, int64_t n, const double *const *coords, const double *w, bh_stream s);

/* bh_fill for float32 columns (DEVICE pointers): every value is
 * widened exactly to float64 first, so the result equals bh_fill on the widened columns,
 * at half the input bytes.  BH_STRATEGY_EXACT falls back to AUTO here. */
bh_status bh_fill_f32(bh_hist *h, int64_t n, const float *const *coords, const float *w, bh_stream s);

/* Same with int32 coordinate columns (e.g. multiplicities; RDataFrame fills histograms
 * from integer columns too, "different ... input data types") and
 * optional float32 weights: each coordinate widens exactly to float64, so the result
 * equals bh_fill on the widened columns.  DEVICE pointers, 4 B per value. */
bh_status bh_fill_i32(bh_hist *h, int64_t n, const int32_t *const *coords, const float *w, bh_stream s);

/* Same as bh_fill but coords/w are HOST pointers (pinned: DMA straight from them;
 * pageable: staged by the driver).  Events are copied in chunks into a device
 * double-buffer on an internal copy stream, overlapped with the fills on s.
 * Returns once every host byte has been consumed (the caller may overwrite its
 * buffers — the fix of PAPER.md:223); kernels may still be in flight on s. */
bh_status bh_fill_host(bh_hist *h, int64_t n, const double *const *coords, const double *w, bh_stream s);

/* bh_fill_host with float32 coordinate/weight columns (bh_fill_f32 semantics: exact
 * widening): HOST pointers, 4 B per value, so half the PCIe bytes of bh_fill_host.  Same
 * staging, overlap and return rule. */
bh_status bh_fill_host_f32(bh_hist *h, int64_t n, const float *const *coords, const float *w, bh_stream s);

/* bh_fill_host with int32 coordinate columns and optional float32 weights (bh_fill_i32
 * semantics), HOST pointers. */
bh_status bh_fill_host_i32(bh_hist *h, int64_t n, const int32_t *const *coords, const float *w, bh_stream s);

/* Persistent bulk consumer: the paper's per-bulk fill loop (RHnCUDA "transfers bulk of events
 * to the GPU and launches kernels ... per bulk"; bulks of 32768 events,
 * PAPER.md:241) without a kernel launch or a copy per bulk (at such sizes
 * launch and transfer overheads dominate).  bh_bulk_begin launches ONE kernel on stream s that
 * stays resident (one CTA per SM) until bh_bulk_end; each bh_bulk_submit posts a bulk to it
 * through a descriptor ring in mapped pinned host memory, and every CTA reads its share of the
 * bulk straight from the host columns over PCIe (zero-copy) into its private bins and register
 * statistics; the bins are flushed and the statistics reduced once, at bh_bulk_end.
 *  bh_bulk_begin(h, weighted, timeout_ms, s): weighted != 0 -> every bulk carries weights.
 *      timeout_ms (0 = 10000): the kernel leaves (dropping the session's fills, reported as
 *      BH_ECUDA by the next bulk call) if no bulk arrives for that long, so a host that dies
 *      mid-session cannot leave the GPU occupied.  Strategy as for a large bh_fill (PRIV, CACHE
 *      or GLOBAL; EXACT/SORT histograms get BH_EINVAL).  The kernel runs on a stream of the
 *      library's own, after the work queued on s before the call; bh_bulk_end orders s after
 *      the session, so other work on s or any other stream is never held back by it.
 *  bh_bulk_submit(h, n, coords, w, &ticket): HOST columns of n (<= 2^31) float64 events (w iff
 *      weighted).  Pinned (page-locked) columns are read in place: the caller must not modify
 *      them until bh_bulk_wait(ticket) returns; pageable columns are first copied into pinned
 *      staging (in pieces of <= 65536 events; the call returns with them reusable).  Up to 4
 *      bulks (pieces) are in flight; a further submit waits for the oldest.
 *  bh_bulk_wait(h, ticket): returns once the bulk's host bytes are consumed.
 *  bh_bulk_fill(h, n, coords, w) = submit + wait.
 *  bh_bulk_end(h): posts the end of the sequence and returns once every CTA has flushed its
 *      bins and statistics (the kernel then exits; bh_read(h, ..., s) sees the full result);
 *      BH_ECUDA if the consumer had timed out (the session's fills are lost).
 * While a session is active the histogram's other calls (fill, read, reset, pack, ...) return
 * BH_EINVAL.  The result equals bh_fill of the concatenated bulks (entries += n per bulk). */
bh_status bh_bulk_begin(bh_hist *h, int32_t weighted, int32_t timeout_ms, bh_stream s);
bh_status bh_bulk_submit(bh_hist *h, int64_t n, const double *const *coords, const double *w, int64_t *ticket);
bh_status bh_bulk_wait(bh_hist *h, int64_t ticket);
bh_status bh_bulk_fill(bh_hist *h, int64_t n, const double *const *coords, const double *w);
bh_status bh_bulk_end(bh_hist *h);

/* Fused multi-histogram fill (one pass over the columns; PAPER.md:470 future work,
 * BASELINE.json config 5).  hs[nh] (1 <= nh <= 8, distinct, same device);
 * col_of_axis[3*i + a] = index into cols[] of the column feeding axis a of
 * histogram i (unused entries ignored); weighted[i] != 0 -> histogram i adds w
 * (then w must be a DEVICE pointer to n weights), else unit weights.  cols:
 * ncols (1..8) DEVICE pointers to float64 columns of n events.  Each histogram
 * gets exactly the result of bh_fill with its own columns.  Async on s.  Errors:
 * BH_EINVAL, BH_EMISMATCH (different devices), BH_ECUDA. */
bh_status bh_fill_multi(bh_hist *const *hs, int32_t nh, const int32_t *col_of_axis, const uint8_t *weighted,
                        int64_t n, const double *const *cols, int32_t ncols, const double *w, bh_stream s);

/* Fused Filter + Define (the RDataFrame example of PAPER.md:95-98,
 * df.Filter(...).Define(...).Histo1D(...), without materializing the derived column).
 * Per event: registers r[0..16) start as r[c] = cols[c][i] for c < ncols (DEVICE float64
 * columns), 0 otherwise; the nops (<= 32) ops of prog run in order; the event is skipped
 * unless filter_reg < 0 or r[filter_reg] != 0; otherwise it is filled at coordinates
 * r[axis_reg[a]] (a < dim) with weight r[weight_reg] (unit weights if weight_reg < 0).
 * entries counts the events that pass.  Every op is IEEE correctly rounded, so derived
 * coordinates equal the same expression evaluated in binary64 anywhere.  Async on s.
 * Errors: BH_EINVAL (bad opcode / register / counts), BH_ECUDA. */
typedef struct {
    int32_t op;      /* BH_OP_* */
    int32_t dst;     /* destination register */
    int32_t a, b, c; /* operand registers (unused ones ignored, must still be in range) */
    int32_t pad;
    double imm;      /* BH_OP_CONST value */
} bh_op;
#define BH_OP_CONST 0  /* r[dst] = imm */
#define BH_OP_COPY 1   /* r[dst] = r[a] */
#define BH_OP_ADD 2    /* r[a] + r[b] */
#define BH_OP_SUB 3    /* r[a] - r[b] */
#define BH_OP_MUL 4    /* r[a] * r[b] */
#define BH_OP_DIV 5    /* r[a] / r[b] */
#define BH_OP_SQRT 6   /* sqrt(r[a]) */
#define BH_OP_ABS 7    /* |r[a]| */
#define BH_OP_NEG 8    /* -r[a] */
#define BH_OP_MIN 9    /* fmin(r[a], r[b]) (IEEE minNum: a NaN operand yields the other) */
#define BH_OP_MAX 10   /* fmax(r[a], r[b]) */
#define BH_OP_LT 11    /* 1.0 if r[a] < r[b] else 0.0 (likewise LE GT GE EQ NE) */
#define BH_OP_LE 12
#define BH_OP_GT 13
#define BH_OP_GE 14
#define BH_OP_EQ 15
#define BH_OP_NE 16
#define BH_OP_AND 17   /* (r[a] != 0) && (r[b] != 0) */
#define BH_OP_OR 18    /* (r[a] != 0) || (r[b] != 0) */
#define BH_OP_NOT 19   /* !(r[a] != 0) */
#define BH_OP_SELECT 20 /* r[a] != 0 ? r[b] : r[c] */
bh_status bh_fill_expr(bh_hist *h, int64_t n, const double *const *cols, int32_t ncols, const bh_op *prog,
                       int32_t nops, const int32_t *axis_reg, int32_t weight_reg, int32_t filter_reg, bh_stream s);

/* Step (1) of PAPER.md:126 alone, per event (parity/debug): out[i] = the global bin
 * b0 + (n0+2)*(b1 + (n1+2)*b2) of event i (FindBin per axis; DESIGN.md
 * readings R1, R2, R4, R5, R9), int32, DEVICE pointer of n elements, caller-owned.  Runs
 * the same FindBin code the fills run, variable-axis tables staged in shared memory as
 * the fills stage them (BH_DEBUG_FIND_BINS_GLOBAL: the float64 global-memory search).
 * Async on s; BH_EINVAL on NULL pointers or n < 0. */
bh_status bh_find_bins(const bh_hist *h, int64_t n, const double *const *coords, int32_t *out, bh_stream s);

/* Shape: dimension, number of bins including flow bins, number of stats (4/7/11). Any may be NULL. */
bh_status bh_info(const bh_hist *h, int32_t *dim, int64_t *nbins_total, int32_t *nstats);

/* Number of doubles in the packed state: 2*nbins_total + nstats + 1. */
bh_status bh_packed_size(const bh_hist *h, int64_t *n_doubles);

/* Write the state as float64 [content(G) | sumw2(G) | stats(K) | entries(1)] to
 * the DEVICE buffer dev_out (caller-owned, bh_packed_size doubles) for an all-reduce SUM
 * across ranks: the state is a sum over events (SPEC.md S:113-121 merge),
 * so partial histograms of disjoint event shards add elementwise.  Async on s.
 * Unit-weight counts are integers < 2^53, exact in any summation order.  BH_EINVAL on NULL. */
bh_status bh_pack(const bh_hist *h, double *dev_out, bh_stream s);

/* Replace the state with a packed buffer (DEVICE pointer, bh_packed_size doubles, layout of
 * bh_pack), e.g. after the all-reduce of SURVEY.md §8(e).  Async on s; BH_EINVAL on NULL. */
bh_status bh_unpack(bh_hist *h, const double *dev_in, bh_stream s);

/* The multi-GPU exchange of SURVEY.md §8(e) for several histograms in ONE collective:
 * hs[nh] (1 <= nh <= 8, same device) are packed one after the other into one DEVICE
 * buffer of bh_packed_size_multi doubles (caller-owned).  unit (may be NULL): unit[i] != 0
 * packs histogram i as [content(G) | stats(K) | entries] without its sum of w^2, which for
 * unit weights equals the content (reading R12), halving the payload; bh_pack_multi
 * refuses (BH_EINVAL) a unit entry for a histogram that received a weighted fill (or a
 * full unpack) since its create/reset.  bh_unpack_multi replaces the states from such a
 * buffer (sum of w^2 := content for unit entries).  Async on s.  The buffer is a sum over
 * events, so ranks holding disjoint shards reduce it elementwise (SUM). */
bh_status bh_packed_size_multi(bh_hist *const *hs, int32_t nh, const uint8_t *unit, int64_t *n_doubles);
bh_status bh_pack_multi(bh_hist *const *hs, int32_t nh, const uint8_t *unit, double *dev_out, bh_stream s);
bh_status bh_unpack_multi(bh_hist *const *hs, int32_t nh, const uint8_t *unit, const double *dev_in, bh_stream s);

/* Diagnostics (no GPU needed): compile the one-pass fused kernel of bh_fill_multi for the
 * histogram-set instantiation `kernel_expr` (e.g. "bh::k_fused<bh::Role<...>>", the form the
 * planner generates) with NVRTC for sm_100a, `threads` per CTA and `ept` events per thread
 * per tile.  Writes a NUL-terminated message (the NVRTC log on failure) to log[log_size].
 * BH_OK, BH_EINVAL, or BH_ECUDA when NVRTC is unavailable or the compile fails. */
bh_status bh_jit_compile_check(const char *kernel_expr, int32_t threads, int32_t ept, char *log, int64_t log_size);

/* Read back to HOST buffers (any may be NULL): contents[G], sumw2[G], stats[K] (ROOT
 * GetStats order, reading R8), entries — "only copy back ... once all bulks have been
 * processed".  Buffers are caller-owned.  Synchronizes stream s; reports
 * earlier asynchronous faults as BH_ECUDA. */
bh_status bh_read(const bh_hist *h, double *contents, double *sumw2, double *stats, int64_t *entries,
                  bh_stream s);

/* TH1F / TH1I-style contents (the paper's bin type T, PAPER.md:141 `T *histogram`, P:164
 * `(T) weight`; "different ... data types"), reading R18 of DESIGN.md: the device
 * state stays exact (u64 counts, float64 sums) and the narrow type is taken once, at read:
 *   BH_CONTENT_F32  contents[i] = RN_float32(content_i), sumw2[i] = RN_float32(sumw2_i), where
 *                   content_i / sumw2_i are the float64 values bh_read returns (one rounding,
 *                   independent of the order of the adds -- unlike float32 atomics);
 *   BH_CONTENT_I32  contents[i] = sumw2[i] = min(count_i, INT32_MAX) (ROOT's TH1I saturates
 *                   at INT32_MAX); only for histograms filled with unit weights (a TH1I
 *                   counts entries) -- BH_EINVAL if any weighted fill or unpack touched it.
 * contents / sumw2 are caller-owned HOST arrays of G float (F32) or int32_t (I32), either may
 * be NULL; stats[K] and entries as in bh_read.  The narrowing runs on the device and halves
 * the bytes copied back.  Synchronizes stream s. */
#define BH_CONTENT_F64 0
#define BH_CONTENT_F32 1
#define BH_CONTENT_I32 2
bh_status bh_read_as(const bh_hist *h, int32_t content_type, void *contents, void *sumw2, double *stats,
                     int64_t *entries, bh_stream s);

/* Force a fill strategy (BH_STRATEGY_*); BH_EINVAL if it cannot hold this histogram. */
bh_status bh_set_strategy(bh_hist *h, int32_t strategy);

/* Strategy the next fill will use (resolves AUTO). */
bh_status bh_get_strategy(const bh_hist *h, int32_t weighted, int32_t *strategy);

/* Events per chunk for bh_fill_host (default 1<<22); >= 1024. */
bh_status bh_set_chunk(bh_hist *h, int64_t events);

/* Plan of bh_fill_multi, set on the histogram passed as hs[0]:
 * BH_MULTI_PASSES (default)  histograms that read the same columns and have small private
 *     states share a pass (k_fill_multi), every other histogram gets its own bh_fill pass:
 *     each pass reads only its own columns, and each histogram gets the whole GPU and the
 *     single-histogram kernel's sinks.  The fill is bound by the shared-memory bin updates
 *     (SM time), not by HBM: C5 measured 5.5 ms this way vs 10.5 ms in one pass;
 * BH_MULTI_ONE_PASS  the one-pass kernel specialized at run time to the histogram set
 *     (NVRTC, cached per set): every column byte is read from DRAM once (PAPER.md:470
 *     "multiple histograms using data in different (parts of the) columns"; C5: 7.0 GB of
 *     DRAM reads per 1.25e8 events instead of 15 GB), histograms too large for one SM's shared
 *     memory together split over the CTAs of a thread-block cluster.  Falls back to the
 *     passes if NVRTC is unavailable (BH_DEBUG_REQUIRE_JIT: fail instead).
 * Results are the same either way (each histogram equals bh_fill on its own columns). */
#define BH_MULTI_PASSES 0
#define BH_MULTI_ONE_PASS 1
bh_status bh_set_multi_mode(bh_hist *h, int32_t mode);

/* Debug flags (BH_DEBUG_*), tests only. */
bh_status bh_set_debug(bh_hist *h, int32_t flags);

/* Number of kernels this histogram has launched so far (for bench/telemetry). */
bh_status bh_launch_count(const bh_hist *h, int64_t *count);

#ifdef __cplusplus
}
#endif

#endif /* BHIST_H */
