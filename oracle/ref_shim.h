/*
 * ref_shim.h — TEST INFRASTRUCTURE ONLY (checker, never shipped or measured
 * as the product). extern "C" face of the UNMODIFIED reference library
 * (/root/reference/proj/core, compiled in place by oracle/Makefile into
 * oracle/_ref/librunq_ref.so) so the Python tests and bench.py's
 * cpu_baseline / --impl reference legs can call the reference operator API
 * on the same host column images the product's C ABI takes.
 *
 * Every output array is malloc'ed by the shim and released with
 * ref_free_column / ref_free_mask / ref_free_array.
 */
#ifndef RUNQ_REF_SHIM_H
#define RUNQ_REF_SHIM_H

#include "../include/runq_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ref_host_array {
  int32_t dtype;
  int32_t _pad;
  int64_t n;
  void* data;
} ref_host_array;

const char* ref_last_error(void);
void ref_free_column(rq_host_column* c);
void ref_free_mask(rq_host_mask* m);
void ref_free_array(ref_host_array* a);

/* round trip through runq::Column (validation of the image conversion) */
int ref_dump_column(const rq_host_column* a, ref_host_array* out);
int ref_roundtrip(const rq_host_column* a, rq_host_column* out);
/* runq::validate (column.cpp:178-216): number of violations */
int ref_validate(const rq_host_column* a);

int ref_range_intersect(const int64_t* s1, const int64_t* e1, int64_t n1, const int64_t* s2,
                        const int64_t* e2, int64_t n2, ref_host_array* s, ref_host_array* e,
                        ref_host_array* idx1, ref_host_array* idx2);
int ref_idx_in_rle(const int64_t* p, int64_t np, const int64_t* s, const int64_t* e, int64_t nr,
                   ref_host_array* p_out, ref_host_array* run_of, ref_host_array* idx_of);
int ref_rle_contain_idx(const int64_t* p, int64_t np, const int64_t* s, const int64_t* e,
                        int64_t nr, ref_host_array* p_out, ref_host_array* run_of,
                        ref_host_array* idx_of);
int ref_idx_in_idx(const int64_t* p1, int64_t n1, const int64_t* p2, int64_t n2,
                   ref_host_array* p_out, ref_host_array* idx1, ref_host_array* idx2);
int ref_bucketize(const int64_t* x, int64_t nx, const int64_t* b, int64_t nb, int32_t right,
                  ref_host_array* out);
int ref_plain_mask_to_rle(const rq_host_mask* m, rq_host_mask* out);
int ref_plain_mask_to_index(const rq_host_mask* m, rq_host_mask* out);
int ref_compact_rle(const rq_host_column* a, rq_host_column* out);
int ref_plain_to_rle(const rq_host_column* a, rq_host_column* out);
int ref_plain_to_rle_index(const rq_host_column* a, int64_t min_run, rq_host_column* out);
int ref_plain_to_plain_index(const rq_host_column* a, double trim, rq_host_column* out);
/* runq::io (ingest.hpp:56-62): encoding selection, encode, table sort */
int ref_choose_encoding(const rq_host_column* a, const rq_heuristic* cfg, rq_encoding_choice* out);
int ref_encode(const rq_host_column* a, const rq_encoding_choice* ch, rq_host_column* out);
int ref_sort_table(const rq_host_column* cols, int32_t ncols, const int32_t* by, int32_t nby,
                   rq_host_column* out);

int ref_decode_values(const rq_host_column* a, ref_host_array* out);
int ref_normalize_basic(const rq_host_column* a, rq_host_column* out);
int ref_align(const rq_host_column* a, const rq_host_column* b, int32_t* shape_kind,
              ref_host_array* s, ref_host_array* e, ref_host_array* p, ref_host_array* v1,
              ref_host_array* v2);
int ref_arith(const rq_host_column* a, const rq_host_column* b, int32_t op, rq_host_column* out);
int ref_compare(const rq_host_column* a, const rq_host_column* b, int32_t op, rq_host_mask* out);
int ref_arith_scalar(const rq_host_column* a, rq_scalar k, int32_t op, int32_t reversed,
                     rq_host_column* out);
int ref_compare_scalar(const rq_host_column* a, rq_scalar k, int32_t op, int32_t reversed,
                       rq_host_mask* out);
int ref_filter(const rq_host_column* a, const rq_host_mask* m, rq_host_column* out);
typedef struct ref_join_side {
  int32_t is_rle;
  int64_t n;
  int64_t* rows;
  int64_t *v, *s, *e;
} ref_join_side;
int ref_get_join_index(const rq_host_column* left, const rq_host_column* right, ref_join_side* lo,
                       ref_join_side* ro, int64_t* cardinality);
int ref_apply_join_index(const rq_host_column* col, const ref_join_side* j, rq_host_column* out);
void ref_free(void* p);
int ref_catalog_create(void** out);
void ref_catalog_free(void* c);
int ref_catalog_add_column(void* c, const char* table, const char* column, const rq_host_column* col,
                           const char* const* dict, int64_t dict_n, const char* dict_name, int32_t is_date);
int ref_run_plan(void* c, const char* json, void** out);
int ref_result_info(void* r, int32_t* ncols, int64_t* rows);
int ref_result_column(void* r, int32_t i, const char** name, int32_t* dtype, const void** data, int64_t* n);
void ref_result_free(void* r);
int ref_hash_build_probe(const void* bv, int32_t bdt, int64_t nb, const void* pv, int32_t pdt, int64_t np,
                         int64_t** bpos, int64_t** ppos, int64_t* n);
int ref_semi_join_mask(const rq_host_column* probe, const rq_host_column* build, rq_host_mask* out);
int ref_and_mask(const rq_host_mask* a, const rq_host_mask* b, rq_host_mask* out);
int ref_or_mask(const rq_host_mask* a, const rq_host_mask* b, rq_host_mask* out);
int ref_not_mask(const rq_host_mask* a, rq_host_mask* out);
int ref_mask_true_count(const rq_host_mask* a, int64_t* out);

int ref_aggregate_all(const rq_host_column* a, int32_t fn, int32_t* out_dtype, int64_t* out_i64,
                      double* out_f64);
/* keys[nk], data[nd], fns[nd]; out_keys[nk], out_vals[nd] */
int ref_group_aggregate(const rq_host_column* keys, int32_t nk, const rq_host_column* data,
                        const int32_t* fns, int32_t nd, int64_t* n_groups,
                        ref_host_array* out_keys, ref_host_array* out_vals);

/*
 * Query-shaped chains timed by bench.py (cpu_baseline / --impl reference).
 * Each runs the reference operator API exactly as runner.cpp would chain it,
 * over `nshards` row-range shards of the same inputs on `nthreads` host
 * threads (the reference is single-threaded and its operators are pure,
 * README.md:30-31, so shards are independent), and returns the combined
 * aggregate plus the wall time in *seconds.
 */
/* C1: aggregate_all(arith(a, b, op), SUM) */
int ref_chain_sum_binop(const rq_host_column* a_shards, const rq_host_column* b_shards,
                        int32_t nshards, int32_t nthreads, int32_t op, int32_t* out_dtype,
                        int64_t* out_i64, double* out_f64, double* seconds);
/* C2: aggregate_all(arith(filter(a,m), filter(b,m), op), SUM), m = compare_scalar(c,k,cmp) */
int ref_chain_filtered_sum(const rq_host_column* c_shards, const rq_host_column* a_shards,
                           const rq_host_column* b_shards, int32_t nshards, int32_t nthreads,
                           rq_scalar k, int32_t cmp, int32_t op, int32_t* out_dtype,
                           int64_t* out_i64, double* out_f64, double* seconds);

#ifdef __cplusplus
}
#endif

#endif
