/*
 * runq_b200.h — C ABI of the B200-native compressed-execution path.
 *
 * Drop-in boundary for the reference engine's hot path (arXiv 2506.10092,
 * `runq`, /root/reference/proj). Each entry point names the reference
 * interface it replaces (file:line under proj/core). The reference API is C++
 * (value-semantics columns, exceptions); this ABI keeps the same operator
 * set, argument meaning and output encodings, but
 *   - columns/masks/arrays live in device memory behind opaque handles,
 *   - errors are int status codes with a thread-local message
 *     (rq_last_error) instead of exceptions (error.hpp:11-32),
 *   - no C++ or torch types cross the boundary.
 *
 * Ownership: every handle returned through an out-parameter is owned by the
 * caller and released with the matching *_free. Handles are immutable and
 * share device buffers internally (reference-counted), so an operator that
 * keeps its input's positions (arith_scalar, filter with a full-cover mask)
 * does not copy them. All work is enqueued on the context's CUDA stream;
 * calls that must know an output size (materialising intersections,
 * compactions) synchronise that stream once.
 *
 * Threading: one context per host thread. Handles may be read from any
 * context on the same device.
 */
#ifndef RUNQ_B200_H
#define RUNQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (runq::Error / OverflowError / ResourceError, error.hpp:11-26) ---- */
enum rq_status {
  RQ_OK = 0,
  RQ_INVALID = 1,  /* runq::Error: precondition / size mismatch / int div by zero */
  RQ_OVERFLOW = 2, /* runq::OverflowError (kernels.cpp:21-31) */
  RQ_RESOURCE = 3, /* runq::ResourceError (primitives.cpp:172-178) or device OOM */
  RQ_CUDA = 4,     /* CUDA runtime failure */
  RQ_NCCL = 5      /* NCCL failure */
};

/* ---- dtypes: runq::DType order (dtype.hpp:11) ---- */
enum rq_dtype { RQ_I8 = 0, RQ_I16 = 1, RQ_I32 = 2, RQ_I64 = 3, RQ_F32 = 4, RQ_F64 = 5 };

/* ---- encodings: runq::Encoding / runq::MaskEncoding (column.hpp:13-14) ---- */
enum rq_encoding {
  RQ_ENC_PLAIN = 0,
  RQ_ENC_RLE = 1,
  RQ_ENC_INDEX = 2,
  RQ_ENC_PLAIN_INDEX = 3,
  RQ_ENC_RLE_INDEX = 4
};
enum rq_mask_encoding {
  RQ_MASK_PLAIN = 0,
  RQ_MASK_RLE = 1,
  RQ_MASK_INDEX = 2,
  RQ_MASK_COMPOSITE = 3
};

/* ---- operators: runq::compute::BinOp (align.hpp:70) ---- */
enum rq_binop {
  RQ_ADD = 0, RQ_SUB = 1, RQ_MUL = 2, RQ_DIV = 3,
  RQ_LT = 4, RQ_LE = 5, RQ_EQ = 6, RQ_NE = 7, RQ_GE = 8, RQ_GT = 9
};

/* ---- aggregate functions: runq::agg::AggFn (groupby.hpp:7) ---- */
enum rq_aggfn {
  RQ_SUM = 0, RQ_COUNT = 1, RQ_MIN = 2, RQ_MAX = 3, RQ_AVG = 4, RQ_STD = 5, RQ_VAR = 6
};

typedef struct rq_ctx_s* rq_ctx_t;   /* device + stream + allocator + pinned scratch */
typedef struct rq_arr_s* rq_arr_t;   /* typed device array (runq::Array, array.hpp:16) */
typedef struct rq_col_s* rq_col_t;   /* runq::Column (column.hpp:78) */
typedef struct rq_mask_s* rq_mask_t; /* runq::MaskColumn (column.hpp:133) */

/* Scalar literal: runq::compute::Scalar = variant<int64_t,double> (align.hpp:76). */
typedef struct rq_scalar {
  int32_t is_float;
  int32_t _pad;
  int64_t i;
  double f;
} rq_scalar;

/*
 * Host-side column image used by rq_col_upload / rq_col_download.
 * Field use per encoding (column.hpp:22-76):
 *   PLAIN       : dtype = storage dtype, logical, has_center/center, n rows, v
 *   RLE         : dtype of v, n runs, v, s, e, total_size
 *   INDEX       : dtype of v, n points, v, p, total_size
 *   PLAIN_INDEX : base as PLAIN (dtype/logical/center/n/v); outliers in
 *                 dtype2 (== logical), n2, v2, p2
 *   RLE_INDEX   : runs as RLE (dtype/n/v/s/e); points in dtype2, n2, v2, p2
 * For download, call rq_col_describe first (fills everything but the
 * pointers), allocate, then rq_col_download copies into the pointers.
 * Upload of a gapless RLE column (runs tile [0, total_size), as ingest
 * produces them) may pass s = NULL: starts are implied (s_0 = 0,
 * s_i = e_{i-1} + 1) and derived on the device, so only v and e cross PCIe.
 */
typedef struct rq_host_column {
  int32_t encoding;
  int32_t dtype;
  int32_t logical;
  int32_t has_center;
  int64_t center;
  int64_t total_size;
  int64_t n;
  void* v;
  int64_t* s;
  int64_t* e;
  int64_t* p;
  int32_t dtype2;
  int32_t _pad;
  int64_t n2;
  void* v2;
  int64_t* p2;
} rq_host_column;

/*
 * Host-side mask image (column.hpp:111-131):
 *   PLAIN     : n bytes in bits (total_size == n)
 *   RLE       : n runs in s, e
 *   INDEX     : n positions in p
 *   COMPOSITE : runs n in s, e; points n2 in p2
 */
typedef struct rq_host_mask {
  int32_t encoding;
  int32_t _pad;
  int64_t total_size;
  int64_t n;
  uint8_t* bits;
  int64_t* s;
  int64_t* e;
  int64_t* p;
  int64_t n2;
  int64_t* p2;
} rq_host_mask;

/* ---------------------------------------------------------------------- */
/* errors / context                                                         */
/* ---------------------------------------------------------------------- */

/* Message of the last failing call on this host thread ("" if none). */
const char* rq_last_error(void);
/* Build/version string: compile target, git-independent. */
const char* rq_version(void);

int rq_ctx_create(int device, rq_ctx_t* out);
int rq_ctx_destroy(rq_ctx_t ctx);
int rq_ctx_synchronize(rq_ctx_t ctx);
/* The context's CUDA stream (cudaStream_t) for interop. */
void* rq_ctx_stream(rq_ctx_t ctx);
/* Kernel launches issued by this context so far (evidence counter). */
int64_t rq_ctx_launches(rq_ctx_t ctx);
/* Per-kernel CUDA-event timing: when enabled, each tagged kernel launch is
 * bracketed by events on the context stream (SURVEY.md §5 tracing). */
int rq_ctx_set_profiling(rq_ctx_t ctx, int32_t enable);
/* Limit the profile to the comma-separated tags (NULL or "": every tag). */
int rq_ctx_profile_only(rq_ctx_t ctx, const char* tags);
/* JSON {"tag": {"ms": total, "count": launches}, ...} into buf (syncs). */
int rq_ctx_profile_report(rq_ctx_t ctx, int32_t reset, char* buf, int64_t cap);

/* ---------------------------------------------------------------------- */
/* arrays (runq::Array, array.hpp:16-99; positions are RQ_I64 arrays)       */
/* ---------------------------------------------------------------------- */

int rq_arr_upload(rq_ctx_t ctx, int32_t dtype, const void* host, int64_t n, rq_arr_t* out);
/* Uninitialised device array of n elements, filled by rq_arr_write: a column
 * larger than host RAM streams into HBM in row chunks (the reference builds
 * columns in host memory only, array.hpp:16-99). */
int rq_arr_alloc(rq_ctx_t ctx, int32_t dtype, int64_t n, rq_arr_t* out);
/* Copies host[0, count) into elements [offset, offset + count) (stream-ordered;
 * the host buffer must stay valid until the context synchronises). */
int rq_arr_write(rq_ctx_t ctx, rq_arr_t a, int64_t offset, const void* host, int64_t count);
/* Wraps caller-owned device memory without copying; caller keeps it alive. */
int rq_arr_wrap_device(rq_ctx_t ctx, int32_t dtype, void* dev, int64_t n, rq_arr_t* out);
int rq_arr_info(rq_arr_t a, int32_t* dtype, int64_t* n);
void* rq_arr_device_ptr(rq_arr_t a);
int rq_arr_download(rq_ctx_t ctx, rq_arr_t a, void* host);
/* downloads n arrays (hosts[i] sized like arrs[i]) with one synchronisation */
int rq_arr_download_many(rq_ctx_t ctx, int32_t n, const rq_arr_t* arrs, void* const* hosts);
int rq_arr_free(rq_arr_t a);

/* ---------------------------------------------------------------------- */
/* columns and masks                                                        */
/* ---------------------------------------------------------------------- */

int rq_col_upload(rq_ctx_t ctx, const rq_host_column* h, rq_col_t* out);
int rq_col_describe(rq_col_t c, rq_host_column* h);
int rq_col_download(rq_ctx_t ctx, rq_col_t c, rq_host_column* h);

/* Column images — the reference's dump_column format (column.cpp:513-563:
 * one JSON header line, then the arrays back to back) as the shard on-disk /
 * wire format. rq_col_dump_image returns a malloc'd image (free with
 * rq_image_free); rq_col_load_image uploads an image's sections straight to
 * the device. Errors: RQ_INVALID for a malformed or truncated image. */
int rq_col_dump_image(rq_ctx_t ctx, rq_col_t c, void** image, int64_t* nbytes);
int rq_col_load_image(rq_ctx_t ctx, const void* image, int64_t nbytes, rq_col_t* out);
void rq_image_free(void* image);
int rq_col_free(rq_col_t c);
int rq_col_encoding(rq_col_t c);
int64_t rq_col_total_size(rq_col_t c);
/* runq::Column::value_type (column.cpp:88-97) */
int rq_col_value_type(rq_col_t c);
/* Builds columns from device arrays (shared, not copied). */
int rq_col_make_rle(rq_ctx_t ctx, rq_arr_t v, rq_arr_t s, rq_arr_t e, int64_t total_size,
                    rq_col_t* out);
int rq_col_make_index(rq_ctx_t ctx, rq_arr_t v, rq_arr_t p, int64_t total_size, rq_col_t* out);
int rq_col_make_plain(rq_ctx_t ctx, rq_arr_t values, int32_t logical, int32_t has_center,
                      int64_t center, rq_col_t* out);
/* Part arrays of a column: which = 0:v 1:s 2:e 3:p 4:v2 5:p2 (new handles). */
int rq_col_part(rq_col_t c, int which, rq_arr_t* out);

int rq_mask_upload(rq_ctx_t ctx, const rq_host_mask* h, rq_mask_t* out);
int rq_mask_describe(rq_mask_t m, rq_host_mask* h);
int rq_mask_download(rq_ctx_t ctx, rq_mask_t m, rq_host_mask* h);
int rq_mask_free(rq_mask_t m);
/* runq::MaskColumn::true_count (column.cpp:112-128); device reduction. */
int rq_mask_true_count(rq_ctx_t ctx, rq_mask_t m, int64_t* out);

/* ---------------------------------------------------------------------- */
/* encoding primitives: runq::enc (primitives.hpp:28-92)                    */
/* ---------------------------------------------------------------------- */

/* enc::range_intersect (primitives.cpp:15-46): fragments s,e + idx1,idx2. */
int rq_range_intersect(rq_ctx_t ctx, rq_arr_t s1, rq_arr_t e1, rq_arr_t s2, rq_arr_t e2,
                       rq_arr_t* s, rq_arr_t* e, rq_arr_t* idx1, rq_arr_t* idx2);
/* enc::idx_in_rle (primitives.cpp:48-61). */
int rq_idx_in_rle(rq_ctx_t ctx, rq_arr_t p, rq_arr_t s, rq_arr_t e, rq_arr_t* p_out,
                  rq_arr_t* run_of, rq_arr_t* idx_of);
/* enc::rle_contain_idx (primitives.cpp:63-86); identical results. */
int rq_rle_contain_idx(rq_ctx_t ctx, rq_arr_t p, rq_arr_t s, rq_arr_t e, rq_arr_t* p_out,
                       rq_arr_t* run_of, rq_arr_t* idx_of);
/* enc::idx_in_idx (primitives.cpp:88-100). */
int rq_idx_in_idx(rq_ctx_t ctx, rq_arr_t p1, rq_arr_t p2, rq_arr_t* p_out, rq_arr_t* idx1,
                  rq_arr_t* idx2);
/* enc::plain_mask_to_rle / plain_mask_to_index (primitives.cpp:349-368). */
int rq_plain_mask_to_rle(rq_ctx_t ctx, rq_mask_t plain, rq_mask_t* out);
int rq_plain_mask_to_index(rq_ctx_t ctx, rq_mask_t plain, rq_mask_t* out);
/* enc::compact_rle (primitives.cpp:370-379). */
int rq_compact_rle(rq_ctx_t ctx, rq_col_t rle, rq_col_t* out);
/* enc::plain_to_rle (primitives.cpp:223-250): runs start where the STORED
 * value changes; run values are decoded (logical dtype, +center). */
int rq_plain_to_rle(rq_ctx_t ctx, rq_col_t plain, rq_col_t* out);
/* enc::plain_to_rle_index (primitives.cpp:252-279): runs of length >= min_run
 * stay runs, shorter runs become points. min_run < 2 -> RQ_INVALID. */
int rq_plain_to_rle_index(rq_ctx_t ctx, rq_col_t plain, int64_t min_run, rq_col_t* out);
/* enc::plain_to_plain_index (primitives.cpp:293-347): trimmed mid-range centre,
 * narrowest base type, values outside it become int64 outliers.
 * trim_fraction outside [0, 0.5) -> RQ_INVALID. */
int rq_plain_to_plain_index(rq_ctx_t ctx, rq_col_t plain, double trim_fraction, rq_col_t* out);

/* ---------------------------------------------------------------------- */
/* ingest: encoding selection and table sort (runq::io, ingest.hpp:29-66)  */
/* ---------------------------------------------------------------------- */

/* runq::io::Scheme (ingest.hpp:29). */
enum { RQ_SCHEME_PLAIN = 0, RQ_SCHEME_PLAIN_CENTERED = 1, RQ_SCHEME_RLE = 2, RQ_SCHEME_RLE_INDEX = 3,
       RQ_SCHEME_PLAIN_INDEX = 4 };

/* runq::io::HeuristicConfig (ingest.hpp:41-48); rq_heuristic_default fills
 * the reference defaults (1e6 rows, ratio 20, trim 0.05, min_run 2, 0.5). */
typedef struct rq_heuristic {
  int64_t row_threshold;
  double ratio_threshold;
  double trim;
  int64_t min_run;
  double unit_run_share;
} rq_heuristic;

/* runq::io::EncodingChoice (ingest.hpp:33-39). */
typedef struct rq_encoding_choice {
  int32_t scheme;
  int32_t width;      /* storage dtype of the (narrowed) plain base */
  int64_t min_run;
  double trim_fraction;
  int32_t has_center;
  int32_t _pad;
  int64_t center;
} rq_encoding_choice;

void rq_heuristic_default(rq_heuristic* cfg);
/* io::choose_encoding (ingest.cpp:217-271): run profile, trimmed split and
 * centred width all computed on the device; cfg NULL = defaults. */
int rq_choose_encoding(rq_ctx_t ctx, rq_col_t plain, const rq_heuristic* cfg, rq_encoding_choice* out);
/* io::encode (ingest.cpp:273-290). */
int rq_encode(rq_ctx_t ctx, rq_col_t plain, const rq_encoding_choice* choice, rq_col_t* out);
/* io::sort_table (ingest.cpp:292-344): stable lexicographic sort of every
 * column by the key columns cols[by[0..nby)]; inputs must be plain, outputs
 * are decoded plain columns (logical dtype). out holds ncols handles. */
int rq_sort_table(rq_ctx_t ctx, const rq_col_t* cols, int32_t ncols, const int32_t* by, int32_t nby,
                  rq_col_t* out);

/* kernels::bucketize (kernels.cpp:10-19): searchsorted of x in boundaries. */
int rq_bucketize(rq_ctx_t ctx, rq_arr_t x, rq_arr_t boundaries, int32_t right, rq_arr_t* out);

/* ---------------------------------------------------------------------- */
/* column model helpers (column.hpp:178-189, align.hpp:43-48)               */
/* ---------------------------------------------------------------------- */

/* decode_values (column.cpp:283-309): bit-width-reduced unpack to logical
 * dtype (+center), Plain+Index overlay. Plain and Plain+Index only. */
int rq_decode_values(rq_ctx_t ctx, rq_col_t c, rq_arr_t* out);
/* compute::normalize_basic (align.cpp:102-115). */
int rq_normalize_basic(rq_ctx_t ctx, rq_col_t c, rq_col_t* out);

/* ---------------------------------------------------------------------- */
/* align-compute: runq::compute (align.hpp:59-95)                           */
/* ---------------------------------------------------------------------- */

/* compute::align (align.cpp:219-231). shape_kind: 0 dense, 1 run, 2 point.
 * Run shapes return s,e; point shapes return p; dense returns neither. */
int rq_align(rq_ctx_t ctx, rq_col_t a, rq_col_t b, int32_t* shape_kind, rq_arr_t* s,
             rq_arr_t* e, rq_arr_t* p, rq_arr_t* v1, rq_arr_t* v2);
/* compute::arith (align.cpp:495-508). */
int rq_arith(rq_ctx_t ctx, rq_col_t a, rq_col_t b, int32_t op, rq_col_t* out);
/* compute::compare (align.cpp:510-523). */
int rq_compare(rq_ctx_t ctx, rq_col_t a, rq_col_t b, int32_t op, rq_mask_t* out);
/* compute::arith_scalar (align.cpp:571-596). */
int rq_arith_scalar(rq_ctx_t ctx, rq_col_t a, rq_scalar k, int32_t op, int32_t reversed,
                    rq_col_t* out);
/* compute::compare_scalar (align.cpp:598-652): predicate -> RLE/Index/Plain/Composite mask. */
int rq_compare_scalar(rq_ctx_t ctx, rq_col_t a, rq_scalar k, int32_t op, int32_t reversed,
                      rq_mask_t* out);
/* compute::filter (align.cpp:755-771). */
int rq_filter(rq_ctx_t ctx, rq_col_t a, rq_mask_t m, rq_col_t* out);

/* masks::and_mask (mask_ops.cpp:183-209). */
int rq_mask_and(rq_ctx_t ctx, rq_mask_t a, rq_mask_t b, rq_mask_t* out);
/* masks::or_mask (mask_ops.cpp:211-237). */
int rq_mask_or(rq_ctx_t ctx, rq_mask_t a, rq_mask_t b, rq_mask_t* out);
/* masks::not_mask (mask_ops.cpp:239-265). */
int rq_mask_not(rq_ctx_t ctx, rq_mask_t a, rq_mask_t* out);

/* ---------------------------------------------------------------------- */
/* joins: runq::joins (join.hpp:58-59)                                      */
/* ---------------------------------------------------------------------- */

/* joins::semi_join_mask (join.cpp:368-406): probe-side mask of the entries
 * (runs / points / rows) whose key occurs on the build side; keys compared
 * as f64 (−0 == +0) if either side is float, else int64. RLE probe → RLE
 * mask of the hit runs; Plain probe → Plain mask; otherwise Index mask. */
int rq_semi_join_mask(rq_ctx_t ctx, rq_col_t probe, rq_col_t build, rq_mask_t* out);

/* joins::hash_build_probe (join.cpp:167-181): the matching (build, probe)
 * position pairs of two value arrays, probe-major, each probe's matches in
 * build-entry order. */
int rq_hash_build_probe(rq_ctx_t ctx, rq_arr_t build_values, rq_arr_t probe_values, rq_arr_t* build_pos,
                        rq_arr_t* probe_pos);

/* joins::JoinIndex (join.hpp:7-31): `rows` (UnsortedIndexJoin) when is_rle
 * = 0, else the reference ranges (v = source run, s, e) of UnsortedRleJoin. */
typedef struct rq_join_side {
  int32_t is_rle;
  int32_t _pad;
  rq_arr_t rows;
  rq_arr_t v, s, e;
} rq_join_side;

/* joins::get_join_index (join.cpp:183-238): equi-join index of two columns in
 * the reference's pairing order (probe-major, matches in build-entry order;
 * the side with fewer entries builds, ties: the left side probes). Runs join
 * as single entries; each side's index is RLE-shaped iff its column is RLE.
 * Output arrays are new handles owned by the caller. */
int rq_get_join_index(rq_ctx_t ctx, rq_col_t left, rq_col_t right, rq_join_side* left_out,
                      rq_join_side* right_out, int64_t* cardinality);

/* joins::apply_join_index (join.cpp:245-366): the column's values in the
 * join index's row order (Plain for row references; RLE / Index ranges keep
 * their encoding). References outside the covered rows raise RQ_INVALID. */
int rq_apply_join_index(rq_ctx_t ctx, rq_col_t col, const rq_join_side* j, rq_col_t* out);

/* ---------------------------------------------------------------------- */
/* aggregation: runq::agg (groupby.hpp:22-50)                               */
/* ---------------------------------------------------------------------- */

/* agg::aggregate_all (groupby.cpp:164-172). Result is one element of dtype
 * *out_dtype (RQ_I64 or RQ_F64) written to *out_i64 or *out_f64. */
int rq_aggregate_all(rq_ctx_t ctx, rq_col_t data, int32_t fn, int32_t* out_dtype,
                     int64_t* out_i64, double* out_f64);

/* agg::group_aggregate (groupby.cpp:144-162). keys[n_keys], data[n_data] with
 * fns[n_data]. Outputs: n_groups, key arrays (device, ascending lexicographic)
 * out_keys[n_keys] and aggregate arrays out_vals[n_data]. */
int rq_group_aggregate(rq_ctx_t ctx, const rq_col_t* keys, int32_t n_keys, const rq_col_t* data,
                       const int32_t* fns, int32_t n_data, int64_t* n_groups, rq_arr_t* out_keys,
                       rq_arr_t* out_vals);

/* The query runner's GroupAgg (runner.cpp:302-336): group_aggregate over
 * normalize_basic(keys) / normalize_basic(data). Same outputs as calling
 * rq_normalize_basic on every input first, but composite inputs are folded
 * part by part instead of being expanded to rows. */
int rq_group_aggregate_normalized(rq_ctx_t ctx, const rq_col_t* keys, int32_t n_keys,
                                  const rq_col_t* data, const int32_t* fns, int32_t n_data,
                                  int64_t* n_groups, rq_arr_t* out_keys, rq_arr_t* out_vals);

/* ---------------------------------------------------------------------- */
/* fused entry points (no reference counterpart: one kernel for an operator
 * chain whose intermediate the reference materialises)                     */
/* ---------------------------------------------------------------------- */

/* aggregate_all(arith(a, b, op), fn) without materialising arith's output
 * (align.cpp:495-508 + groupby.cpp:164-172). fn in {SUM, COUNT, AVG}. */
int rq_aggregate_binop(rq_ctx_t ctx, rq_col_t a, rq_col_t b, int32_t op, int32_t fn,
                       int32_t* out_dtype, int64_t* out_i64, double* out_f64);

/* aggregate_all(arith(filter(a,m), filter(b,m), op), fn) with
 * m = compare_scalar(c, k, cmp) — the filtered-aggregate query shape of
 * runner.cpp:243-336 — in one pass over the compressed inputs. */
int rq_filtered_aggregate_binop(rq_ctx_t ctx, rq_col_t c, rq_scalar k, int32_t cmp,
                                rq_col_t a, rq_col_t b, int32_t op, int32_t fn,
                                int32_t* out_dtype, int64_t* out_i64, double* out_f64);

/* One aggregate expression of the query runner's GroupAgg
 * (runner.cpp:302-336 over the plan's arith / arith_scalar nodes,
 * align.cpp:495-508, :571-596): a left-deep chain
 * ((t0 ops[0] t1) ops[1] t2) of up to 3 terms; a term is `col` (op = -1) or
 * `col op k` (`k op col` when reversed). n_terms = 0 is COUNT(*). */
typedef struct rq_term {
  rq_col_t col;
  int32_t op;       /* RQ_ADD..RQ_DIV, or -1 for the bare column */
  int32_t reversed; /* scalar on the left */
  rq_scalar k;
} rq_term;
typedef struct rq_expr {
  int32_t n_terms;
  int32_t ops[2];
  rq_term terms[3];
} rq_expr;

/* The runner's Filter → expressions → GroupAgg sequence (runner.cpp:243-336):
 * every operand filtered by `mask` (NULL: no WHERE), each expression
 * evaluated, then group_aggregate(normalize_basic(...)) over `keys`
 * (n_keys = 0: aggregate_all per expression, returned as one group). fns[i]
 * is the aggregate of exprs[i]. Same outputs as rq_group_aggregate_normalized.
 * Runs as one pass over the compressed columns (K12) when the shape allows
 * (RLE mask, RLE integer keys, plain / RLE / Plain+Index operands,
 * SUM / AVG / COUNT); otherwise through the operator chain. *fused (may be
 * NULL) reports which. */
int rq_group_aggregate_exprs(rq_ctx_t ctx, rq_mask_t mask, const rq_col_t* keys, int32_t n_keys,
                             const rq_expr* exprs, const int32_t* fns, int32_t n_exprs, int64_t* n_groups,
                             rq_arr_t* out_keys, rq_arr_t* out_vals, int32_t* fused);

/* One WHERE conjunct of the runner's predicate tree (runner.cpp:114-193):
 * `col op k` (compare_scalar, align.cpp:598-652) or, with n_in > 0,
 * `col IN (in_list[0..n_in))` = OR of equalities (mask_ops.cpp:211-237). */
typedef struct rq_pred {
  rq_col_t col;
  int32_t op;   /* RQ_LT..RQ_GT (ignored when n_in > 0) */
  int32_t n_in;
  rq_scalar k;
  const rq_scalar* in_list;
} rq_pred;

/* rq_group_aggregate_exprs with the WHERE clause given as conjuncts instead
 * of a materialised mask (`mask` may still be given: it is AND-ed in). With
 * RLE predicate columns the predicates are evaluated once per segment of the
 * joint run alignment (no mask is built); otherwise the mask is built with
 * compare_scalar / mask_or / mask_and exactly as the runner does. */
int rq_group_aggregate_where(rq_ctx_t ctx, const rq_pred* where, int32_t n_where, rq_mask_t mask,
                             const rq_col_t* keys, int32_t n_keys, const rq_expr* exprs, const int32_t* fns,
                             int32_t n_exprs, int64_t* n_groups, rq_arr_t* out_keys, rq_arr_t* out_vals,
                             int32_t* fused);

/* ---------------------------------------------------------------------- */
/* query runner: runq::query (plan.hpp:13-80, runner.hpp:14-95)             */
/* ---------------------------------------------------------------------- */

typedef struct rq_catalog_s* rq_catalog_t; /* runq::query::Catalog (runner.hpp:14-28) */
typedef struct rq_result_s* rq_result_t;   /* runq::query::ResultTable (runner.hpp:42-48) */

int rq_catalog_create(rq_catalog_t* out);
int rq_catalog_destroy(rq_catalog_t cat);
/* Adds a column (TableColumn, table.hpp:14-19) to `table` (created on first
 * use). dict: the dictionary's strings in code order (dictionary.hpp:16-43),
 * or dict_n = 0 for non-string columns; columns naming the same dict_name
 * share one dictionary (no recoding across them in joins). is_date: the
 * column holds days since 1970-01-01 and takes 'YYYY-MM-DD' literals. */
int rq_catalog_add_column(rq_catalog_t cat, const char* table, const char* column, rq_col_t col,
                          const char* const* dict, int64_t dict_n, const char* dict_name, int32_t is_date);
/* runq::query::run in Compressed mode (runner.cpp:86-373): parses the JSON
 * plan (plan.cpp:13-105) and executes it on the device, materialising the
 * result rows. */
int rq_run_plan(rq_ctx_t ctx, rq_catalog_t cat, const char* plan_json, rq_result_t* out);
/* fused_nodes: GroupAgg nodes that ran as one fused call */
int rq_result_info(rq_result_t r, int32_t* n_cols, int64_t* rows, int32_t* fused_nodes);
/* name stays valid until rq_result_free; values is a new array handle */
int rq_result_column(rq_result_t r, int32_t i, const char** name, rq_arr_t* values);
int rq_result_free(rq_result_t r);

/* ---------------------------------------------------------------------- */
/* boundary completions: the rest of the reference operator surface the    */
/* reference's own tests and the C++ drop-in adapter call                   */
/* (paper_2506_10092_b200/adapter/). Shapes (compute::Shape, align.hpp:12-25)*/
/* cross the ABI as (kind, n, s, e, p): kind 0 dense with n slots, 1 runs   */
/* s/e (n runs), 2 points p (n points); unused handles are NULL.            */
/* ---------------------------------------------------------------------- */

/* compute::decompose (align.cpp:86-100); RLE+Index raises RQ_INVALID. */
int rq_decompose(rq_ctx_t ctx, rq_col_t c, int32_t* kind, int64_t* n, rq_arr_t* s, rq_arr_t* e, rq_arr_t* p,
                 rq_arr_t* values);
/* compute::align_many (align.cpp:233-254): the left-fold alignment; values[ncols]. */
int rq_align_many(rq_ctx_t ctx, const rq_col_t* cols, int32_t ncols, int32_t* kind, int64_t* n, rq_arr_t* s,
                  rq_arr_t* e, rq_arr_t* p, rq_arr_t* values);
/* compute::shape_weights (align.cpp:57-70): run lengths or ones. */
int rq_shape_weights(rq_ctx_t ctx, int32_t kind, int64_t n, rq_arr_t s, rq_arr_t e, rq_arr_t p, rq_arr_t* out);
/* agg::group (groupby.cpp:46-50) = align_many + unique_with_inverse: the
 * aligned shape, inverse (group id per slot), keys_out[n_keys], n_groups. */
int rq_group(rq_ctx_t ctx, const rq_col_t* keys, int32_t n_keys, int32_t* kind, int64_t* n, rq_arr_t* s,
             rq_arr_t* e, rq_arr_t* p, rq_arr_t* inverse, rq_arr_t* keys_out, int64_t* n_groups);
/* agg::group_on_arrays (groupby.cpp:33-44) over aligned key arrays (the shape stays with the caller). */
int rq_group_on_arrays(rq_ctx_t ctx, const rq_arr_t* key_values, int32_t n_keys, rq_arr_t* inverse,
                       rq_arr_t* keys_out, int64_t* n_groups);
/* agg::aggregate_array (groupby.cpp:67-135): run-length-weighted SUM /
 * COUNT / AVG / STD / VAR, MIN / MAX with empty-group sentinels; f64 sums
 * fold each group in slot order (bit-identical to the reference). */
int rq_aggregate_array(rq_ctx_t ctx, int32_t kind, int64_t n, rq_arr_t s, rq_arr_t e, rq_arr_t p, rq_arr_t values,
                       rq_arr_t inverse, int64_t n_groups, int32_t fn, rq_arr_t* out);

/* kernels::Reduce (kernels.hpp:44) */
enum { RQ_REDUCE_SUM = 0, RQ_REDUCE_MIN = 1, RQ_REDUCE_MAX = 2, RQ_REDUCE_COUNT = 3 };
/* kernels::scatter_reduce (kernels.cpp:97-125): values fold in input order
 * per group; out-of-range group index raises RQ_INVALID. */
int rq_scatter_reduce(rq_ctx_t ctx, rq_arr_t values, rq_arr_t index, int64_t n_groups, int32_t reduce,
                      rq_arr_t* out);
/* kernels::unique_with_inverse (kernels.cpp:127-187): keys ascending lexicographic. */
int rq_unique_with_inverse(rq_ctx_t ctx, const rq_arr_t* cols, int32_t n, rq_arr_t* keys_out, rq_arr_t* inverse,
                           int64_t* n_groups);
/* kernels::cumsum / checked_sum (kernels.cpp:21-38): int64 overflow raises RQ_OVERFLOW. */
int rq_cumsum(rq_ctx_t ctx, rq_arr_t x, int32_t exclusive, rq_arr_t* out);
int rq_checked_sum(rq_ctx_t ctx, rq_arr_t x, int64_t* out);
/* kernels::repeat_interleave / range_arange (kernels.cpp:40-60). */
int rq_repeat_interleave(rq_ctx_t ctx, rq_arr_t values, rq_arr_t counts, rq_arr_t* out);
int rq_range_arange(rq_ctx_t ctx, rq_arr_t start, rq_arr_t length, rq_arr_t* out);
/* kernels::gather (kernels.cpp:195-219): out-of-range index raises RQ_INVALID. */
int rq_gather(rq_ctx_t ctx, rq_arr_t values, rq_arr_t idx, rq_arr_t* out);
/* kernels::sort_with_perm / adjacent_ne (kernels.cpp:221-245); adjacent_ne is RQ_I8 0/1. */
int rq_sort_with_perm(rq_ctx_t ctx, rq_arr_t values, rq_arr_t* sorted, rq_arr_t* perm);
int rq_adjacent_ne(rq_ctx_t ctx, rq_arr_t x, rq_arr_t* out);
/* enc::range_union / merge_sorted_idx / concat_sort_idx / complement_rle /
 * complement_index (primitives.cpp:102-167). */
int rq_range_union(rq_ctx_t ctx, rq_arr_t s1, rq_arr_t e1, rq_arr_t s2, rq_arr_t e2, rq_arr_t* s, rq_arr_t* e);
int rq_merge_sorted_idx(rq_ctx_t ctx, rq_arr_t p1, rq_arr_t p2, rq_arr_t* out);
int rq_concat_sort_idx(rq_ctx_t ctx, rq_arr_t p1, rq_arr_t p2, rq_arr_t* out);
int rq_complement_rle(rq_ctx_t ctx, rq_arr_t s, rq_arr_t e, int64_t total, rq_arr_t* s_out, rq_arr_t* e_out);
int rq_complement_index(rq_ctx_t ctx, rq_arr_t p, int64_t total, rq_arr_t* s_out, rq_arr_t* e_out);
/* enc::rle_to_index / rle_to_plain for columns and masks (primitives.cpp:172-220);
 * an expansion above `budget` elements raises RQ_RESOURCE. */
int rq_rle_to_index(rq_ctx_t ctx, rq_col_t c, int64_t budget, rq_col_t* out);
int rq_rle_to_plain(rq_ctx_t ctx, rq_col_t c, double fill, int64_t budget, rq_col_t* out);
int rq_mask_rle_to_index(rq_ctx_t ctx, rq_mask_t m, int64_t budget, rq_mask_t* out);
int rq_mask_rle_to_plain(rq_ctx_t ctx, rq_mask_t m, int64_t budget, rq_mask_t* out);
/* enc::compact_rle_index (primitives.cpp:381-420). */
int rq_compact_rle_index(rq_ctx_t ctx, rq_col_t c, rq_col_t* out);
/* decode_full (column.cpp:311-329; gaps raise RQ_INVALID) and to_rows (column.cpp:331-376). */
int rq_decode_full(rq_ctx_t ctx, rq_col_t c, rq_arr_t* out);
int rq_to_rows(rq_ctx_t ctx, rq_col_t c, rq_arr_t* positions, rq_arr_t* values);
/* runq::ColumnStats / stats (column.hpp:162-173, column.cpp:244-279): the
 * reference's byte accounting (positions at 8 B, RLE run = w + 16 B). */
typedef struct rq_column_stats {
  int64_t n_runs;
  double avg_run_length;
  int64_t encoded_bytes;
  int64_t plain_bytes;
  double compression_ratio;
} rq_column_stats;
int rq_col_stats(rq_ctx_t ctx, rq_col_t c, rq_column_stats* out);

/* ---------------------------------------------------------------------- */
/* row-range sharding (multi-GPU; no reference counterpart)                 */
/* ---------------------------------------------------------------------- */

/* Slices a host column image to rows [lo, hi) as a standalone shard: runs
 * crossing a cut are split with their value duplicated, positions are
 * rebased to the shard (p - lo) and total_size = hi - lo. Pure host function
 * (no device work); output arrays are allocated with malloc and released
 * with rq_host_column_free. */
int rq_shard_host_column(const rq_host_column* in, int64_t lo, int64_t hi, rq_host_column* out);
void rq_host_column_free(rq_host_column* h);

/* Communicators. Every rank runs the single-GPU path on its
 * row-range shard; the partial aggregates are combined with ONE collective
 * on the context stream: a grouped ncclAllReduce of 8-byte partials for
 * global aggregates, an ncclAllGather of fixed-capacity (key, partial)
 * packets + a device regroup (keys ascending) for group tables. Integer
 * SUM / COUNT combine by wrapping addition (bit-exact); f64 sums reassociate
 * (1e-9 relative); AVG is recomputed from the merged SUM and COUNT;
 * STD / VAR are rejected (RQ_INVALID: not exact under a merge). The result
 * is identical on every rank. NCCL errors (incl. ncclCommGetAsyncError,
 * polled after each merge) return RQ_NCCL. */
typedef struct rq_comm_s* rq_comm_t;
enum { RQ_COMM_NCCL = 0, RQ_COMM_HOST = 1 };
/* host transport: gathers every rank's `bytes` from `send` into
 * recv[rank * bytes ...] (same `bytes` on every rank); returns 0 on success */
typedef int (*rq_host_allgather_fn)(const void* send, int64_t bytes, void* recv, void* user);

/* ncclGetUniqueId into id[0..128) (rank 0 creates it, the launcher
 * broadcasts it); NCCL is loaded on first use (libnccl.so.2). */
int rq_comm_unique_id(void* id, int64_t cap);
/* ncclCommInitRank on the context's device (one rank per GPU). */
int rq_comm_init_nccl(rq_ctx_t ctx, const void* id, int32_t nranks, int32_t rank, rq_comm_t* out);
/* Host transport (several ranks on one device, e.g. tests over gloo). */
int rq_comm_init_host(rq_ctx_t ctx, int32_t nranks, int32_t rank, rq_host_allgather_fn fn, void* user,
                      rq_comm_t* out);
int rq_comm_info(rq_comm_t comm, int32_t* nranks, int32_t* rank, int32_t* transport);
int rq_comm_destroy(rq_comm_t comm);

/* Low level: merges per-rank partial tables (n_groups rows of n_keys key
 * arrays + n_parts 8-byte partial arrays, part_fns in SUM/COUNT/MIN/MAX)
 * into the global table: keys ascending, COUNT / SUM partials summed, MIN /
 * MAX re-reduced. n_keys = 0: one row per rank, all-reduced. */
int rq_merge_group_tables(rq_ctx_t ctx, rq_comm_t comm, const rq_arr_t* keys, int32_t n_keys,
                          const rq_arr_t* parts, const int32_t* part_fns, int32_t n_parts, int64_t n_groups,
                          int64_t* out_groups, rq_arr_t* out_keys, rq_arr_t* out_parts);

/* The sharded forms of the entry points above: same arguments plus the
 * communicator, called by every rank on its shard; outputs are the merged
 * global result (on every rank). */
int rq_aggregate_all_sharded(rq_ctx_t ctx, rq_comm_t comm, rq_col_t data, int32_t fn, int32_t* out_dtype,
                             int64_t* out_i64, double* out_f64);
int rq_aggregate_binop_sharded(rq_ctx_t ctx, rq_comm_t comm, rq_col_t a, rq_col_t b, int32_t op, int32_t fn,
                               int32_t* out_dtype, int64_t* out_i64, double* out_f64);
int rq_filtered_aggregate_binop_sharded(rq_ctx_t ctx, rq_comm_t comm, rq_col_t c, rq_scalar k, int32_t cmp,
                                        rq_col_t a, rq_col_t b, int32_t op, int32_t fn, int32_t* out_dtype,
                                        int64_t* out_i64, double* out_f64);
/* normalized != 0: rq_group_aggregate_normalized semantics */
int rq_group_aggregate_sharded(rq_ctx_t ctx, rq_comm_t comm, const rq_col_t* keys, int32_t n_keys,
                               const rq_col_t* data, const int32_t* fns, int32_t n_data, int32_t normalized,
                               int64_t* n_groups, rq_arr_t* out_keys, rq_arr_t* out_vals);
int rq_group_aggregate_where_sharded(rq_ctx_t ctx, rq_comm_t comm, const rq_pred* where, int32_t n_where,
                                     rq_mask_t mask, const rq_col_t* keys, int32_t n_keys, const rq_expr* exprs,
                                     const int32_t* fns, int32_t n_exprs, int64_t* n_groups, rq_arr_t* out_keys,
                                     rq_arr_t* out_vals, int32_t* fused);

#ifdef __cplusplus
}
#endif

#endif /* RUNQ_B200_H */
