/*
 * hbk.h — C ABI of the B200-native HB-CSF / B-CSF sparse MTTKRP library
 * (libhbk.so, built for sm_100a).
 *
 * The reference (`tenkit`, /root/reference/pkg/src/tenkit) is pure Python/NumPy
 * and has no FFI, so this header is the boundary a maintainer would bind from
 * the reference's Python API with ctypes.  Each entry
 * point names the reference function it replaces (file:line, relative to
 * /root/reference/pkg/src/tenkit/).
 *
 * Conventions
 *  - Every call returns an int status: HBK_OK or one of the HBK_E* codes.  The
 *    message for the last failure on the calling thread is hbk_last_error().
 *    The Python shim maps HBK_EINVAL -> ValueError, HBK_ETYPE -> TypeError,
 *    HBK_ECUDA -> RuntimeError, HBK_ENOMEM -> MemoryError, mirroring the
 *    reference's exception types (kernels.py:62-88, balance.py:39-48,128-150).
 *  - Pointers marked [dev] are CUDA device pointers on the current device;
 *    [host] are host pointers.  `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).
 *  - Handles (hbk_coo, hbk_csl, hbk_csf, hbk_sched, hbk_plan) own their device
 *    arrays and are immutable after creation (reference: "treat instances as
 *    immutable", coo.py:58).  They are reference counted: *_retain adds a
 *    reference, *_release drops one and frees the arrays at zero.
 *  - Build calls (create/sort/canonicalize/build/split/schedule/plan) may
 *    synchronise `stream` to learn output sizes.  hbk_plan_execute is fully
 *    asynchronous on `stream`.
 *  - Index arrays are uint32 on the device; nnz must be < 2^32 - 1.
 */
#ifndef HBK_H
#define HBK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HBK_ABI_VERSION 1
#define HBK_MAX_ORDER 8

#define HBK_OK 0
#define HBK_EINVAL 1 /* ValueError   */
#define HBK_ETYPE 2  /* TypeError    */
#define HBK_ECUDA 3  /* RuntimeError */
#define HBK_ENOMEM 4 /* MemoryError  */

/* SliceKind values, formats.py:41-46 */
#define HBK_SLICE_COO 0
#define HBK_SLICE_CSL 1
#define HBK_SLICE_CSF 2

typedef struct hbk_coo hbk_coo;
typedef struct hbk_csl hbk_csl;
typedef struct hbk_csf hbk_csf;
typedef struct hbk_sched hbk_sched;
typedef struct hbk_plan hbk_plan;

const char* hbk_last_error(void);
int hbk_abi_version(void);
/* Number of SMs of the current device (0 and HBK_ECUDA when no device). */
int hbk_device_sms(int* sms);

/* ------------------------------------------------------------------ COO --
 * CooTensor, coo.py:42-114.  Stored as SoA uint32 columns + fp32 values for
 * the kernels + the caller's fp64 values (kept for exact export).            */
typedef struct {
  int order;
  int64_t dims[HBK_MAX_ORDER];
  int64_t nnz;
  int has_sorted;                      /* sorted_under is not None          */
  int sorted_under[HBK_MAX_ORDER];
  int unique_mode;                     /* >=0: every slice of that mode holds
                                          one nonzero (HB-CSF coo_part)      */
} hbk_coo_info;

/* CooTensor(dims, indices, values, sorted_under): idx [dev] nnz x order
 * row-major, vals [dev] fp64.  Range checking is the caller's (coo.py:80-84
 * is done by the Python shim).  sorted_under may be NULL (unknown).        */
int hbk_coo_create(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx,
                   const double* vals, const int* sorted_under, void* stream, hbk_coo** out);
/* Same, from fp32 values (no fp64 copy is kept; export widens fp32). */
int hbk_coo_create_f32(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx,
                       const float* vals, const int* sorted_under, void* stream, hbk_coo** out);
int hbk_coo_info_get(const hbk_coo* t, hbk_coo_info* info);
/* Copy back: idx [host] nnz x order uint32 row-major, vals [host] fp64. Either may be NULL. */
int hbk_coo_export(const hbk_coo* t, uint32_t* idx, double* vals, void* stream);
/* Device views of the SoA columns (col < order) and fp32 values. */
int hbk_coo_device_arrays(const hbk_coo* t, const uint32_t** cols, const float** vals32);
/* Device-to-device copy-out: idx [dev] nnz x order row-major, v64/v32 [dev];
 * any pointer may be NULL. */
int hbk_coo_export_device(const hbk_coo* t, uint32_t* idx, double* v64, float* v32, void* stream);
/* sort_by_mode_order, coo.py:208-224: stable lexicographic order, mode_order[0]
 * major.  Returns a new retained handle (or t itself, retained, when
 * t->sorted_under == mode_order, coo.py:221-222).                           */
int hbk_coo_sort(hbk_coo* t, const int* mode_order, void* stream, hbk_coo** out);
/* canonicalize, coo.py:227-247: identity sort, duplicates merged, exact zeros
 * dropped.  merge = 0: sum duplicates exactly as np.add.reduceat does
 * (first + pairwise(rest)), then drop 0.0; merge = 1: keep the first of each
 * duplicate run (set semantics; used by the synthetic generator).          */
int hbk_coo_canonicalize(const hbk_coo* t, int merge, void* stream, hbk_coo** out);
/* Slice view of a COO tensor for mttkrp_coo (kernels.py:109-151): entries
 * grouped by `mode` (sorted under (mode, *rest) unless already mode-major),
 * returned as a CSL-shaped handle over ALL slices.                         */
int hbk_coo_slices(hbk_coo* t, int mode, void* stream, hbk_csl** out);
void hbk_coo_retain(hbk_coo* t);
void hbk_coo_release(hbk_coo* t);

/* ------------------------------------------------------------------ CSL --
 * CslSlices, formats.py:207-233.                                           */
typedef struct {
  int order;
  int64_t dims[HBK_MAX_ORDER];
  int mode_order[HBK_MAX_ORDER];
  int64_t num_slices;
  int64_t nnz;
} hbk_csl_info;

#define HBK_CSL_SLICE_PTR 0 /* int64  [S+1]           */
#define HBK_CSL_SLICE_IDX 1 /* uint32 [S]             */
#define HBK_CSL_REST_IDX 2  /* uint32 [nnz x (N-1)]   */
#define HBK_CSL_VALUES 3    /* fp64   [nnz]           */
int hbk_csl_info_get(const hbk_csl* s, hbk_csl_info* info);
int hbk_csl_export(const hbk_csl* s, int which, void* host_dst, void* stream);
void hbk_csl_retain(hbk_csl* s);
void hbk_csl_release(hbk_csl* s);

/* ------------------------------------------------------------------ CSF --
 * CsfTensor, formats.py:49-117.                                            */
typedef struct {
  int order;
  int64_t dims[HBK_MAX_ORDER];
  int mode_order[HBK_MAX_ORDER];
  int64_t nnz;
  int64_t level_sizes[HBK_MAX_ORDER]; /* len(idxs[d]), d < order-1 */
  int split;
} hbk_csf_info;

#define HBK_CSF_PTR 0    /* int64  [level_sizes[level]+1] */
#define HBK_CSF_IDX 1    /* uint32 [level_sizes[level]]   */
#define HBK_CSF_LEAF 2   /* uint32 [nnz]                  */
#define HBK_CSF_VALUES 3 /* fp64   [nnz]                  */
int hbk_csf_info_get(const hbk_csf* c, hbk_csf_info* info);
int hbk_csf_export(const hbk_csf* c, int which, int level, void* host_dst, void* stream);

/* build_csf, formats.py:120-168. */
int hbk_build_csf(hbk_coo* t, const int* mode_order, void* stream, hbk_csf** out);
/* build_hbcsf, formats.py:260-299: three slice-disjoint parts.  coo_part keeps
 * unpermuted coordinates sorted under mode_order (formats.py:273-275).     */
int hbk_build_hbcsf(hbk_coo* t, const int* mode_order, void* stream, hbk_coo** coo_part,
                    hbk_csl** csl_part, hbk_csf** csf_part);
/* classify_slices, formats.py:194-204: labels [host] int8 [num_slices]. */
int hbk_classify_slices(const hbk_csf* c, int8_t* labels, void* stream);
/* Slice / fiber populations of a tree, reduced on the device (the inspect
 * statistics of coo.py:281-325 compute_stats, balance.py:210-227
 * imbalance_metrics and formats.py:315-328 slice_census, without exporting
 * the pointer arrays).  Slice sizes are nonzeros per slice, fiber sizes
 * nonzeros per leaf-parent node (per segment once split).  Sums of squares
 * are exact integers (sum <= nnz * max < 2^64), so the caller forms the
 * population variance exactly.  Slice classes follow classify_slices.      */
typedef struct {
  int64_t slices, fibers, nnz;
  int64_t max_slice, max_fiber;
  uint64_t sumsq_slice, sumsq_fiber;
  int64_t coo_slices, csl_slices, csf_slices;
} hbk_population;
int hbk_csf_population(const hbk_csf* c, hbk_population* out, void* stream);
/* split_fibers, balance.py:65-90.  *out = NULL (status OK) when no fiber
 * exceeds fiber_threshold (the reference returns the input object).        */
int hbk_split_fibers(const hbk_csf* c, int64_t fiber_threshold, void* stream, hbk_csf** out);
void hbk_csf_retain(hbk_csf* c);
void hbk_csf_release(hbk_csf* c);

/* ------------------------------------------------------------- schedule --
 * assign_slice_blocks / BlockSchedule, balance.py:100-189.                 */
typedef struct {
  int64_t num_units;
  int64_t num_slices;
  int64_t num_fibers;
  int64_t block_size;
} hbk_sched_info;
#define HBK_SCHED_UNITS 0 /* int64 [num_units x 4]: block_id, slice_pos, fiber_start, fiber_stop */
#define HBK_SCHED_MULT 1  /* int64 [num_slices] multiplicities */
int hbk_assign_slice_blocks(const hbk_csf* c, int64_t block_size, void* stream, hbk_sched** out);
/* A schedule from host units (BlockSchedule built by the caller):
 * units [host] int64 num_units x 4 as above, mult [host] int64 [num_slices]. */
int hbk_sched_from_units(const hbk_csf* c, const int64_t* units, int64_t num_units,
                         const int64_t* mult, void* stream, hbk_sched** out);
int hbk_sched_info_get(const hbk_sched* s, hbk_sched_info* info);
int hbk_sched_export(const hbk_sched* s, int which, int64_t* host_dst, void* stream);
/* BlockSchedule.validate_for, balance.py:128-150 (HBK_EINVAL on mismatch). */
int hbk_sched_validate(const hbk_sched* s, const hbk_csf* c, void* stream);
void hbk_sched_retain(hbk_sched* s);
void hbk_sched_release(hbk_sched* s);

/* --------------------------------------------------------------- MTTKRP --
 * mttkrp_hbcsf / mttkrp_csf / mttkrp_csl / mttkrp_coo / mttkrp_scheduled,
 * kernels.py:109-342.  A plan binds up to three slice-disjoint parts of one
 * tensor (any may be NULL) for one output mode and rank, precomputes the
 * work list (B-CSF units), and is then executed any number of times.
 *   coo  : an HB-CSF coo_part (unique_mode == mode), one nonzero per row
 *   csl  : a CslSlices (or hbk_coo_slices view) with mode_order[0] == mode
 *   csf  : a CsfTensor with mode_order[0] == mode (split or not)
 *   sched: optional BlockSchedule of csf; its units become the CSF work
 *          units (one 8-lane group per unit) exactly as mttkrp_scheduled.
 * The output (dims[mode] x rank fp32, row-major, caller-owned) is fully
 * written: rows owned by no part are zero-filled inside the same launch.
 * A plan owns its split-slice workspace, task counters and fork/join
 * streams; executions of ONE plan are therefore ordered by the library:
 * each execute/probe makes its stream wait for the previous execution of
 * the same plan (an event recorded on whatever stream issued it, under a
 * per-plan lock), so concurrent calls from several host threads or streams
 * are safe and serialise on the device; distinct plans run concurrently.
 * An execute is capturable into a CUDA graph (inside a capture the
 * capturing stream provides the order).                                    */
typedef struct {
  int mode;
  int rank;
  int64_t out_rows;
  int64_t tasks_csf, tasks_csl, tasks_coo, tasks_zero;
  int64_t split_rows;      /* rows accumulated by more than one task      */
  int64_t launches;        /* kernel launches per execute                 */
  int fast_path;           /* 1: order-3 float4 kernel; 0: generic kernel */
  int64_t op_muls, op_adds; /* OpCount of the reference kernel, R-weighted */
  int64_t nnz;
  int64_t stream_bytes;    /* index + value bytes read per execute        */
  int64_t tasks_heavy;     /* group tasks of the heavy-slice CSF layout   */
  int64_t hot_rows;        /* reserved (0) */
  int64_t csl_blocks;      /* B-row blocks of the fast CSL task order (0/1 = unblocked) */
  int64_t gather_rows;     /* factor rows one execute gathers (B-position plans) */
  int64_t leaf_blocks;     /* leaf-row blocks of the leaf-blocked heavy slices (0 = none) */
  int64_t leaf_blocked_nnz; /* nonzeros in the leaf-blocked heavy slices */
  int64_t leaf_head_share_ppm; /* share (ppm) of leaf accesses served by the rows a quarter of the L2 holds (leaf-blocking candidates) */
} hbk_plan_info;

int hbk_plan_create(hbk_coo* coo, hbk_csl* csl, hbk_csf* csf, hbk_sched* sched, int mode,
                    int rank, void* stream, hbk_plan** out);
int hbk_plan_info_get(const hbk_plan* p, hbk_plan_info* info);
/* factors: [host] array of `order` [dev] pointers, factor d row-major
 * dims[d] x rank fp32 (factors[mode] is not read, kernels.py:62-66).
 * out: [dev] dims[mode] x rank fp32.                                       */
int hbk_plan_execute(const hbk_plan* p, const float* const* factors, float* out, void* stream);
/* hbk_plan_execute with flags.  HBK_EXEC_SKIP_UNOWNED: rows no bucket owns
 * (see hbk_plan_rows) may be left unwritten instead of zero-filled — for
 * callers that only read the owned rows (the CP-ALS row update).           */
#define HBK_EXEC_SKIP_UNOWNED 1
int hbk_plan_execute_ex(const hbk_plan* p, const float* const* factors, float* out, int flags,
                        void* stream);
/* fp64 mode: factors/out fp64, the buckets' original fp64 values, fp64
 * accumulation (generic kernel).  For accuracy-sensitive callers, e.g. the
 * CP-ALS fit, whose algebraic form amplifies fp32 rounding near convergence. */
int hbk_plan_execute_f64(const hbk_plan* p, const double* const* factors, double* out,
                         void* stream);
void hbk_plan_release(hbk_plan* p);
/* Roofline calibration: walk the plan's task lists and streams exactly as
 * hbk_plan_execute does but only gather the factor rows (no arithmetic, no
 * output).  Its time is the row-gather ceiling of this plan on this GPU;
 * info.gather_rows / time = rows per second.  B-position plans only. */
int hbk_plan_probe(const hbk_plan* p, const float* const* factors, void* stream);
/* Hardware roofline anchor: one launch gathering ~`gathers` 128-byte rows at
 * pseudo-random indices of a zeroed `rows`-row scratch matrix (`rows` a power
 * of two; the library keeps the scratch), ctas_per_sm x 256-thread CTAs per
 * SM, 8-lane groups as in the MTTKRP kernels, no index streams or arithmetic.
 * The caller times it on `stream`; rows per launch = ctas_per_sm x SMs x 32
 * groups x ceil8(gathers / groups).  Scratch within the L2: the L2 -> SM
 * random-row rate; beyond it: the HBM random-row rate.  rows = 0 frees the
 * scratch (the other arguments are then ignored). */
int hbk_row_ceiling(int64_t rows, int ctas_per_sm, int64_t gathers, void* stream);
/* The same matrix (hbk_row_ceiling with the same rows must have run first),
 * gathered through an index stream read like the MTTKRP kernels read theirs:
 * each 8-lane group walks a contiguous span of idx[n] (device u32, taken
 * modulo rows), one coalesced load per lane per 8 positions, SHFL
 * broadcasts, L1-allocating row loads.  Rows per launch = groups x
 * floor8(n / groups).  The caller picks the row distribution. */
int hbk_row_ceiling_stream(const uint32_t* idx, int64_t n, int64_t rows, int ctas_per_sm, void* stream);
/* cudaStreamSynchronize on the caller's stream (the host calling convention
 * waits for its result copy without a Python-level stream object).        */
int hbk_stream_synchronize(void* stream);
/* The output rows a plan's buckets own (rows the MTTKRP can make nonzero),
 * ascending.  *count = their number; rows [dev] u32 (capacity >= *count) or
 * NULL to only count.  Synchronises the stream (the count comes back).      */
int hbk_plan_rows(const hbk_plan* p, uint32_t* rows, int64_t* count, void* stream);
/* Finiteness scan for the host calling convention (replaces the per-call
 * np.isfinite of kernels.py:82-86 on factors already uploaded): async, one
 * launch; flags[i] (device int32) = 1 if bufs[i][0..counts[i]) holds a NaN or
 * Inf, else 0.  n <= 8. */
int hbk_nonfinite_f32(const float* const* bufs, const int64_t* counts, int n, int32_t* flags,
                      void* stream);
/* Host staging of the host-array calling convention (kernels.py:62-88,
 * the factors' np.asarray + float conversion): narrows n float64 host
 * arrays srcs[i][0..counts[i]) into page-locked float32 buffers stage[i]
 * on a pool of host threads and issues the host-to-device copies into
 * dst[i] (device) on `stream` chunk by chunk as the narrowing proceeds.
 * Returns once every copy is enqueued (stage[i] must stay untouched until
 * the stream passes them).  flags[i] (host) = 1 if the fp32 copy of factor
 * i holds a NaN or Inf (kernels.py:82-86).  n <= 8. */
int hbk_stage_f64_to_f32(const double* const* srcs, const int64_t* counts, int n,
                         float* const* stage, float* const* dst, int32_t* flags, void* stream);
/* The same for the fp64 kernels (precision="fp64"): a page-locked float64
 * copy (streaming stores) sent chunk by chunk; flags[i] = 1 on a NaN/Inf. */
int hbk_stage_f64_to_f64(const double* const* srcs, const int64_t* counts, int n,
                         double* const* stage, double* const* dst, int32_t* flags, void* stream);

/* ------------------------------------------------------- FROSTT text --
 * parse_frostt / load_frostt / write_frostt, coo.py:117-205, on the host
 * (multi-threaded; no device needed).  Parsing rules are the reference's:
 * '#' starts a comment, blank lines are skipped, 1-based indices, order from
 * the first data line (or `order` + `dims` when dims != NULL).  On a
 * malformed line the call fails with HBK_EINVAL and, when the failure has a
 * line, *out is still set so hbk_tns_info can report err_line (release it).
 * threads: 0 = all cores (>= 1 MiB per chunk), > 0 = at most that many,
 * < 0 = exactly -threads chunks.                                             */
typedef struct hbk_tns hbk_tns;
int hbk_tns_parse(const char* text, int64_t len, int order, const int64_t* dims, int threads,
                  hbk_tns** out);
int hbk_tns_load(const char* path, int order, const int64_t* dims, int threads, hbk_tns** out);
/* order, nnz, dims [HBK_MAX_ORDER] (max index + 1 per mode, or the given
 * dims), err_line (0 = none); any pointer may be NULL. */
int hbk_tns_info(const hbk_tns* t, int* order, int64_t* nnz, int64_t* dims, int64_t* err_line);
/* idx [host] nnz x order uint32 0-based row-major, vals [host] fp64. */
int hbk_tns_export(const hbk_tns* t, uint32_t* idx, double* vals);
void hbk_tns_release(hbk_tns* t);
/* write_frostt text of nnz entries (1-based, "%.17g" values); *text is
 * malloc'ed, free with hbk_tns_free_text. */
int hbk_tns_format(const uint32_t* idx, const double* vals, int64_t nnz, int order, int threads,
                   char** text, int64_t* len);
void hbk_tns_free_text(char* text);

/* ------------------------------------------------------------- CP-ALS --
 * Row update of one ALS mode on a row shard (cpd.py:157-195), fused:
 *   F = Y * M                 (cpd.py:172; M = pinv(V), 32x32 row-major fp32)
 *   gram  = F^T F             (cpd.py:39-42; fp64, overwritten)
 *   inner = sum_r w_r sum_i Y[i,r] F[i,r]   (cpd.py:176-184 fit term; NULL
 *                               to skip; colw = w [dev] fp32 [32] or NULL = 1)
 * Y, F [dev] rows x rank fp32 row-major (may not alias); rank must be 32.   */
int hbk_als_update(const float* Y, int64_t rows, int rank, const float* M, const float* colw,
                   float* F, double* gram, double* inner, void* stream);
/* The same update restricted to the listed rows (ascending u32 row ids [dev],
 * nlist of them): only those rows of Y are read and of F written — for modes
 * whose other rows are known to be zero in Y (and already zero in F), e.g.
 * rows no bucket owns (hbk_plan_rows).  Gram and fit term as above.         */
int hbk_als_update_rows(const float* Y, const uint32_t* list, int64_t nlist, int rank,
                        const float* M, const float* colw, float* F, double* gram, double* inner,
                        void* stream);

/* ------------------------------------------------------------ sharding --
 * Multi-GPU partitioner: slice nnz histogram of `mode`.
 * hist [dev] int64 [dims[mode]] is overwritten.                            */
int hbk_coo_slice_histogram(const hbk_coo* t, int mode, int64_t* hist, void* stream);
/* Fibers per slice: the number of distinct (mode, mid_mode) coordinate
 * pairs of every mode-`mode` slice, i.e. the leaf-parent count of each slice
 * of the CSF tree ordered (mode, mid_mode, ...) (formats.py:143-162) — the
 * partitioner's cost model charges a slice its nonzeros plus its fibers (one
 * gathered factor row each).  hist [dev] int64 [dims[mode]] is overwritten. */
int hbk_coo_fiber_histogram(const hbk_coo* t, int mode, int mid_mode, int64_t* hist, void* stream);
/* Keep only entries whose `mode` coordinate lies in [row_begin, row_end)
 * (coordinates and dims unchanged). */
int hbk_coo_select_rows(const hbk_coo* t, int mode, int64_t row_begin, int64_t row_end,
                        void* stream, hbk_coo** out);
/* The same selection, rebased: the shard's `mode` coordinates are shifted by
 * -row_begin and dims[mode] = row_end - row_begin (> 0), so an MTTKRP of the
 * shard writes exactly the rank's own output rows (no zero-fill of the other
 * ranks' rows).  Used by the row-sharded multi-GPU CP-ALS.                 */
int hbk_coo_shard_rows(const hbk_coo* t, int mode, int64_t row_begin, int64_t row_end,
                       void* stream, hbk_coo** out);

#ifdef __cplusplus
}
#endif
#endif /* HBK_H */
