// capi_ops.cpp — operator half of the C ABI (include/runq_b200.h).
#include <cstdlib>
#include <cstring>

#include "rq_internal.hpp"

using namespace rqb;

namespace {

CtxPtr ctx_of(rq_ctx_t c) {
  if (!c || !c->ctx) fail("null context");
  RQ_CUDA_CHECK(cudaSetDevice(c->ctx->device));
  return c->ctx;
}
const DArr& arr_of(rq_arr_t a) {
  if (!a) fail("null array handle");
  return a->a;
}
const DCol& col_of(rq_col_t c) {
  if (!c) fail("null column handle");
  return c->c;
}
const DMask& mask_of(rq_mask_t m) {
  if (!m) fail("null mask handle");
  return m->m;
}
Scalar scal(rq_scalar k) {
  Scalar s;
  s.is_float = k.is_float != 0;
  s.i = k.i;
  s.f = k.f;
  return s;
}
void put(rq_arr_t* out, const DArr& a) {
  if (out) *out = wrap_arr(a);
}
void put_agg(const AggOut& r, int32_t* out_dtype, int64_t* out_i64, double* out_f64) {
  if (out_dtype) *out_dtype = r.dtype;
  if (out_i64) *out_i64 = r.i;
  if (out_f64) *out_f64 = r.f;
}
void require_pos(const DArr& a, const char* what) {
  if (a.dt != RQ_I64) fail(std::string(what) + ": positions must be i64");
}

}  // namespace

extern "C" {

int rq_range_intersect(rq_ctx_t c, rq_arr_t s1, rq_arr_t e1, rq_arr_t s2, rq_arr_t e2,
                       rq_arr_t* s, rq_arr_t* e, rq_arr_t* idx1, rq_arr_t* idx2) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    Intersection r = range_intersect(ctx, arr_of(s1), arr_of(e1), arr_of(s2), arr_of(e2),
                                     idx1 != nullptr, idx2 != nullptr);
    put(s, r.s);
    put(e, r.e);
    put(idx1, r.idx1);
    put(idx2, r.idx2);
  });
}

int rq_idx_in_rle(rq_ctx_t c, rq_arr_t p, rq_arr_t s, rq_arr_t e, rq_arr_t* p_out,
                  rq_arr_t* run_of, rq_arr_t* idx_of) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require_pos(arr_of(p), "idx_in_rle");
    PointsInRuns r = points_in_runs(ctx, arr_of(p), arr_of(s), arr_of(e), run_of != nullptr,
                                    idx_of != nullptr);
    put(p_out, r.p_out);
    put(run_of, r.run_of);
    put(idx_of, r.idx_of);
  });
}

int rq_rle_contain_idx(rq_ctx_t c, rq_arr_t p, rq_arr_t s, rq_arr_t e, rq_arr_t* p_out,
                       rq_arr_t* run_of, rq_arr_t* idx_of) {
  // primitives.hpp:43-46: same result set as idx_in_rle; one device kernel
  return rq_idx_in_rle(c, p, s, e, p_out, run_of, idx_of);
}

int rq_idx_in_idx(rq_ctx_t c, rq_arr_t p1, rq_arr_t p2, rq_arr_t* p_out, rq_arr_t* idx1,
                  rq_arr_t* idx2) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require_pos(arr_of(p1), "idx_in_idx");
    require_pos(arr_of(p2), "idx_in_idx");
    PointsIntersect r = points_intersect(ctx, arr_of(p1), arr_of(p2), idx1 != nullptr,
                                         idx2 != nullptr);
    put(p_out, r.p_out);
    put(idx1, r.idx1);
    put(idx2, r.idx2);
  });
}

int rq_plain_mask_to_rle(rq_ctx_t c, rq_mask_t plain, rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DMask& m = mask_of(plain);
    require(m.enc == RQ_MASK_PLAIN, "plain_mask_to_rle: plain mask required");
    DMask r;
    r.enc = RQ_MASK_RLE;
    r.total = m.bits.n;
    plain_mask_to_rle(ctx, m.bits, r.s, r.e);
    *out = wrap_mask(std::move(r));
  });
}

int rq_plain_mask_to_index(rq_ctx_t c, rq_mask_t plain, rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DMask& m = mask_of(plain);
    require(m.enc == RQ_MASK_PLAIN, "plain_mask_to_index: plain mask required");
    DMask r;
    r.enc = RQ_MASK_INDEX;
    r.total = m.bits.n;
    r.p = plain_mask_to_index(ctx, m.bits);
    *out = wrap_mask(std::move(r));
  });
}

int rq_compact_rle(rq_ctx_t c, rq_col_t rle, rq_col_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DCol& in = col_of(rle);
    require(in.enc == RQ_ENC_RLE, "compact_rle: rle column required");
    DCol r;
    r.enc = RQ_ENC_RLE;
    r.v = in.v;
    r.logical = in.v.dt;
    int64_t covered = 0;
    r.s = compact_positions(ctx, in.s, in.e, r.e, &covered);
    r.total = covered;
    *out = wrap_col(std::move(r));
  });
}

int rq_bucketize(rq_ctx_t c, rq_arr_t x, rq_arr_t boundaries, int32_t right, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    put(out, bucketize(ctx, arr_of(x), arr_of(boundaries), right != 0));
  });
}

int rq_decode_values(rq_ctx_t c, rq_col_t col, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DCol& in = col_of(col);
    if (in.enc == RQ_ENC_PLAIN) put(out, decode_plain(ctx, in));
    else if (in.enc == RQ_ENC_PLAIN_INDEX) put(out, decode_plain_index(ctx, in));
    else fail("decode_values: plain or plain+index only");
  });
}

int rq_plain_to_rle(rq_ctx_t c, rq_col_t plain, rq_col_t* out) {
  return api_guard([&] { *out = wrap_col(plain_to_rle(ctx_of(c), col_of(plain))); });
}

int rq_plain_to_rle_index(rq_ctx_t c, rq_col_t plain, int64_t min_run, rq_col_t* out) {
  return api_guard([&] { *out = wrap_col(plain_to_rle_index(ctx_of(c), col_of(plain), min_run)); });
}

int rq_plain_to_plain_index(rq_ctx_t c, rq_col_t plain, double trim, rq_col_t* out) {
  return api_guard([&] { *out = wrap_col(plain_to_plain_index(ctx_of(c), col_of(plain), trim)); });
}

void rq_heuristic_default(rq_heuristic* cfg) {
  if (!cfg) return;
  const HeuristicD d;
  cfg->row_threshold = d.row_threshold;
  cfg->ratio_threshold = d.ratio_threshold;
  cfg->trim = d.trim;
  cfg->min_run = d.min_run;
  cfg->unit_run_share = d.unit_run_share;
}

int rq_choose_encoding(rq_ctx_t c, rq_col_t plain, const rq_heuristic* cfg, rq_encoding_choice* out) {
  return api_guard([&] {
    require(out != nullptr, "choose_encoding: null output");
    HeuristicD h;
    if (cfg) {
      h.row_threshold = cfg->row_threshold;
      h.ratio_threshold = cfg->ratio_threshold;
      h.trim = cfg->trim;
      h.min_run = cfg->min_run;
      h.unit_run_share = cfg->unit_run_share;
    }
    const EncodingChoiceD ch = choose_encoding(ctx_of(c), col_of(plain), h);
    out->scheme = ch.scheme;
    out->width = ch.width;
    out->min_run = ch.min_run;
    out->trim_fraction = ch.trim;
    out->has_center = ch.has_center ? 1 : 0;
    out->_pad = 0;
    out->center = ch.center;
  });
}

int rq_encode(rq_ctx_t c, rq_col_t plain, const rq_encoding_choice* choice, rq_col_t* out) {
  return api_guard([&] {
    require(choice != nullptr, "encode: null choice");
    EncodingChoiceD ch;
    ch.scheme = choice->scheme;
    ch.width = choice->width;
    ch.min_run = choice->min_run;
    ch.trim = choice->trim_fraction;
    ch.has_center = choice->has_center != 0;
    ch.center = choice->center;
    *out = wrap_col(encode_column(ctx_of(c), col_of(plain), ch));
  });
}

int rq_sort_table(rq_ctx_t c, const rq_col_t* cols, int32_t ncols, const int32_t* by, int32_t nby,
                  rq_col_t* out) {
  return api_guard([&] {
    require(ncols > 0 && cols && out, "sort_table: no columns");
    require(nby > 0 && by, "sort_table: no sort columns");
    std::vector<const DCol*> in;
    for (int32_t i = 0; i < ncols; ++i) in.push_back(&col_of(cols[i]));
    std::vector<DCol> res = sort_table(ctx_of(c), in, std::vector<int>(by, by + nby));
    for (int32_t i = 0; i < ncols; ++i) out[i] = wrap_col(std::move(res[i]));
  });
}

int rq_normalize_basic(rq_ctx_t c, rq_col_t col, rq_col_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_col(normalize_basic(ctx, col_of(col)));
  });
}

int rq_align(rq_ctx_t c, rq_col_t a, rq_col_t b, int32_t* shape_kind, rq_arr_t* s, rq_arr_t* e,
             rq_arr_t* p, rq_arr_t* v1, rq_arr_t* v2) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    Aligned r = align(ctx, col_of(a), col_of(b));
    if (shape_kind) *shape_kind = r.kind;
    if (r.kind == 1) {
      put(s, r.s);
      put(e, r.e);
    } else if (r.kind == 2) {
      put(p, r.p);
    }
    put(v1, r.v1);
    put(v2, r.v2);
  });
}

int rq_arith(rq_ctx_t c, rq_col_t a, rq_col_t b, int32_t op, rq_col_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_col(arith(ctx, col_of(a), col_of(b), op));
  });
}

int rq_compare(rq_ctx_t c, rq_col_t a, rq_col_t b, int32_t op, rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_mask(compare(ctx, col_of(a), col_of(b), op));
  });
}

int rq_arith_scalar(rq_ctx_t c, rq_col_t a, rq_scalar k, int32_t op, int32_t reversed,
                    rq_col_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_col(arith_scalar(ctx, col_of(a), scal(k), op, reversed != 0));
  });
}

int rq_compare_scalar(rq_ctx_t c, rq_col_t a, rq_scalar k, int32_t op, int32_t reversed,
                      rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_mask(compare_scalar(ctx, col_of(a), scal(k), op, reversed != 0));
  });
}

int rq_filter(rq_ctx_t c, rq_col_t a, rq_mask_t m, rq_col_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_col(filter(ctx, col_of(a), mask_of(m)));
  });
}

int rq_semi_join_mask(rq_ctx_t c, rq_col_t probe, rq_col_t build, rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(out != nullptr, "null out");
    *out = wrap_mask(semi_join_mask(ctx, col_of(probe), col_of(build)));
  });
}

namespace {
void side_to_abi(const JoinSideD& j, rq_join_side* o) {
  o->is_rle = j.is_rle ? 1 : 0;
  o->_pad = 0;
  o->rows = j.is_rle ? nullptr : wrap_arr(j.rows);
  o->v = j.is_rle ? wrap_arr(j.v) : nullptr;
  o->s = j.is_rle ? wrap_arr(j.s) : nullptr;
  o->e = j.is_rle ? wrap_arr(j.e) : nullptr;
}
}  // namespace

int rq_hash_build_probe(rq_ctx_t c, rq_arr_t build_values, rq_arr_t probe_values, rq_arr_t* build_pos,
                        rq_arr_t* probe_pos) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(build_pos && probe_pos, "null out");
    DArr b, p;
    hash_build_probe(ctx, arr_of(build_values), arr_of(probe_values), b, p);
    *build_pos = wrap_arr(b);
    *probe_pos = wrap_arr(p);
  });
}

int rq_get_join_index(rq_ctx_t c, rq_col_t left, rq_col_t right, rq_join_side* left_out, rq_join_side* right_out,
                      int64_t* cardinality) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(left_out && right_out, "null out");
    JoinResultD r = get_join_index(ctx, col_of(left), col_of(right));
    side_to_abi(r.left, left_out);
    side_to_abi(r.right, right_out);
    if (cardinality) *cardinality = r.cardinality;
  });
}

int rq_apply_join_index(rq_ctx_t c, rq_col_t col, const rq_join_side* j, rq_col_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(j != nullptr && out != nullptr, "null argument");
    JoinSideD s;
    s.is_rle = j->is_rle != 0;
    if (s.is_rle) {
      require(j->v && j->s && j->e, "apply_join_index: ranges required");
      s.v = arr_of(j->v);
      s.s = arr_of(j->s);
      s.e = arr_of(j->e);
      require(s.s.n == s.e.n && s.v.n == s.s.n, "apply_join_index: range arrays differ in length");
    } else {
      require(j->rows != nullptr, "apply_join_index: rows required");
      s.rows = arr_of(j->rows);
    }
    *out = wrap_col(apply_join_index(ctx, col_of(col), s));
  });
}

int rq_mask_and(rq_ctx_t c, rq_mask_t a, rq_mask_t b, rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_mask(mask_and(ctx, mask_of(a), mask_of(b)));
  });
}

int rq_mask_or(rq_ctx_t c, rq_mask_t a, rq_mask_t b, rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_mask(mask_or(ctx, mask_of(a), mask_of(b)));
  });
}

int rq_mask_not(rq_ctx_t c, rq_mask_t a, rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    *out = wrap_mask(mask_not(ctx, mask_of(a)));
  });
}

int rq_aggregate_all(rq_ctx_t c, rq_col_t data, int32_t fn, int32_t* out_dtype, int64_t* out_i64,
                     double* out_f64) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    put_agg(aggregate_column(ctx, col_of(data), fn), out_dtype, out_i64, out_f64);
  });
}

static int group_aggregate_api(rq_ctx_t c, const rq_col_t* keys, int32_t n_keys, const rq_col_t* data,
                               const int32_t* fns, int32_t n_data, int64_t* n_groups, rq_arr_t* out_keys,
                               rq_arr_t* out_vals, bool normalize) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(n_keys > 0, "group: empty key list");
    std::vector<const DCol*> k, d;
    std::vector<int> f;
    for (int i = 0; i < n_keys; ++i) k.push_back(&col_of(keys[i]));
    for (int i = 0; i < n_data; ++i) {
      d.push_back(&col_of(data[i]));
      f.push_back(fns[i]);
    }
    GroupAggOut r = group_aggregate(ctx, k, d, f, normalize);
    if (n_groups) *n_groups = r.n_groups;
    for (int i = 0; i < n_keys; ++i) out_keys[i] = wrap_arr(r.keys[static_cast<size_t>(i)]);
    for (int i = 0; i < n_data; ++i) out_vals[i] = wrap_arr(r.vals[static_cast<size_t>(i)]);
  });
}

int rq_group_aggregate_sharded(rq_ctx_t c, rq_comm_t comm, const rq_col_t* keys, int32_t n_keys,
                               const rq_col_t* data, const int32_t* fns, int32_t n_data, int32_t normalized,
                               int64_t* n_groups, rq_arr_t* out_keys, rq_arr_t* out_vals) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(n_keys > 0, "group: empty key list");
    std::vector<const DCol*> k, d;
    std::vector<int> f;
    for (int i = 0; i < n_keys; ++i) k.push_back(&col_of(keys[i]));
    for (int i = 0; i < n_data; ++i) {
      d.push_back(&col_of(data[i]));
      f.push_back(fns[i]);
    }
    GroupAggOut r = sharded(
        ctx, comm_of(comm), f,
        [&](const PartialPlan& p) {
          std::vector<const DCol*> ld;
          for (int i : p.src) ld.push_back(d[static_cast<size_t>(i)]);
          return group_aggregate(ctx, k, ld, p.local_fns, normalized != 0);
        },
        [&](int a, int b) { return d[static_cast<size_t>(a)] == d[static_cast<size_t>(b)]; });
    if (n_groups) *n_groups = r.n_groups;
    for (int i = 0; i < n_keys; ++i) out_keys[i] = wrap_arr(r.keys[static_cast<size_t>(i)]);
    for (int i = 0; i < n_data; ++i) out_vals[i] = wrap_arr(r.vals[static_cast<size_t>(i)]);
  });
}

int rq_aggregate_all_sharded(rq_ctx_t c, rq_comm_t comm, rq_col_t data, int32_t fn, int32_t* out_dtype,
                             int64_t* out_i64, double* out_f64) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DCol& d = col_of(data);
    put_agg(sharded_scalar(ctx, comm_of(comm), fn, [&](int f) { return aggregate_column(ctx, d, f); }), out_dtype,
            out_i64, out_f64);
  });
}

int rq_aggregate_binop_sharded(rq_ctx_t c, rq_comm_t comm, rq_col_t a, rq_col_t b, int32_t op, int32_t fn,
                               int32_t* out_dtype, int64_t* out_i64, double* out_f64) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DCol &x = col_of(a), &y = col_of(b);
    put_agg(sharded_scalar(ctx, comm_of(comm), fn, [&](int f) { return aggregate_binop(ctx, x, y, op, f); }),
            out_dtype, out_i64, out_f64);
  });
}

int rq_filtered_aggregate_binop_sharded(rq_ctx_t c, rq_comm_t comm, rq_col_t pred, rq_scalar k, int32_t cmp,
                                        rq_col_t a, rq_col_t b, int32_t op, int32_t fn, int32_t* out_dtype,
                                        int64_t* out_i64, double* out_f64) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DCol &p = col_of(pred), &x = col_of(a), &y = col_of(b);
    const Scalar ks = scal(k);
    put_agg(sharded_scalar(ctx, comm_of(comm), fn,
                           [&](int f) { return filtered_aggregate_binop(ctx, p, ks, cmp, x, y, op, f); }),
            out_dtype, out_i64, out_f64);
  });
}

int rq_group_aggregate(rq_ctx_t c, const rq_col_t* keys, int32_t n_keys, const rq_col_t* data,
                       const int32_t* fns, int32_t n_data, int64_t* n_groups, rq_arr_t* out_keys,
                       rq_arr_t* out_vals) {
  return group_aggregate_api(c, keys, n_keys, data, fns, n_data, n_groups, out_keys, out_vals, false);
}

int rq_group_aggregate_normalized(rq_ctx_t c, const rq_col_t* keys, int32_t n_keys, const rq_col_t* data,
                                  const int32_t* fns, int32_t n_data, int64_t* n_groups,
                                  rq_arr_t* out_keys, rq_arr_t* out_vals) {
  return group_aggregate_api(c, keys, n_keys, data, fns, n_data, n_groups, out_keys, out_vals, true);
}

int rq_aggregate_binop(rq_ctx_t c, rq_col_t a, rq_col_t b, int32_t op, int32_t fn,
                       int32_t* out_dtype, int64_t* out_i64, double* out_f64) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    put_agg(aggregate_binop(ctx, col_of(a), col_of(b), op, fn), out_dtype, out_i64, out_f64);
  });
}

int rq_filtered_aggregate_binop(rq_ctx_t c, rq_col_t pred, rq_scalar k, int32_t cmp, rq_col_t a,
                                rq_col_t b, int32_t op, int32_t fn, int32_t* out_dtype,
                                int64_t* out_i64, double* out_f64) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    put_agg(filtered_aggregate_binop(ctx, col_of(pred), scal(k), cmp, col_of(a), col_of(b), op, fn),
            out_dtype, out_i64, out_f64);
  });
}

static int group_aggregate_exprs_api(rq_ctx_t c, const rq_pred* where, int32_t n_where, rq_mask_t mask,
                                     const rq_col_t* keys, int32_t n_keys, const rq_expr* exprs,
                                     const int32_t* fns, int32_t n_exprs, int64_t* n_groups, rq_arr_t* out_keys,
                                     rq_arr_t* out_vals, int32_t* fused, rq_comm_t comm = nullptr) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(n_exprs > 0 && exprs != nullptr && fns != nullptr, "group_aggregate_exprs: no expressions");
    std::vector<const DCol*> k;
    for (int i = 0; i < n_keys; ++i) k.push_back(&col_of(keys[i]));
    std::vector<XExpr> xs(static_cast<size_t>(n_exprs));
    std::vector<int> f;
    for (int i = 0; i < n_exprs; ++i) {
      const rq_expr& e = exprs[i];
      require(e.n_terms >= 0 && e.n_terms <= 3, "group_aggregate_exprs: 0..3 terms per expression");
      for (int t = 0; t < e.n_terms; ++t) {
        XTerm tm;
        tm.col = &col_of(e.terms[t].col);
        tm.sop = e.terms[t].op;
        tm.rev = e.terms[t].reversed != 0;
        tm.k = scal(e.terms[t].k);
        require(tm.sop == -1 || (tm.sop >= RQ_ADD && tm.sop <= RQ_DIV), "arith: arithmetic operator required");
        xs[static_cast<size_t>(i)].terms.push_back(tm);
        if (t > 0) {
          require(e.ops[t - 1] >= RQ_ADD && e.ops[t - 1] <= RQ_DIV, "arith: arithmetic operator required");
          xs[static_cast<size_t>(i)].ops.push_back(e.ops[t - 1]);
        }
      }
      f.push_back(fns[i]);
    }
    std::vector<XPred> preds;
    for (int i = 0; i < n_where; ++i) {
      XPred q;
      q.col = &col_of(where[i].col);
      q.op = where[i].op;
      q.k = scal(where[i].k);
      require(where[i].n_in >= 0, "where: negative IN-list length");
      if (where[i].n_in == 0) require(q.op >= RQ_LT && q.op <= RQ_GT, "compare_scalar: comparison operator required");
      for (int j = 0; j < where[i].n_in; ++j) q.in.push_back(scal(where[i].in_list[j]));
      preds.push_back(q);
    }
    bool was_fused = false;
    const DMask* m = mask ? &mask_of(mask) : nullptr;
    const std::vector<XPred>* pp = preds.empty() ? nullptr : &preds;
    GroupAggOut r;
    if (comm) {  // this rank's partials (AVG → SUM, COUNT of the same expression), merged
      auto same_expr = [&](int a, int b) {
        const XExpr &x = xs[static_cast<size_t>(a)], &y = xs[static_cast<size_t>(b)];
        if (x.terms.size() != y.terms.size() || x.ops != y.ops) return false;
        for (size_t t = 0; t < x.terms.size(); ++t) {
          const XTerm &u = x.terms[t], &v = y.terms[t];
          if (u.col != v.col || u.sop != v.sop || u.rev != v.rev || u.k.is_float != v.k.is_float ||
              u.k.i != v.k.i || std::memcmp(&u.k.f, &v.k.f, 8) != 0)
            return false;
        }
        return true;
      };
      r = sharded(
          ctx, comm_of(comm), f,
          [&](const PartialPlan& p) {
            // COUNT partials run as COUNT(*): every aggregate of the GroupAgg
            // is aligned jointly (runner.cpp:306-336), so they count the same rows
            std::vector<XExpr> lx;
            for (size_t j = 0; j < p.src.size(); ++j)
              lx.push_back(p.local_fns[j] == RQ_COUNT ? XExpr{} : xs[static_cast<size_t>(p.src[j])]);
            return group_aggregate_exprs(ctx, m, k, lx, p.local_fns, &was_fused, pp);
          },
          same_expr);
    } else {
      // the plan's CUDA-graph key: handle ids, operators, literal bits, functions
      std::string key = "gae";
      auto add = [&](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
      auto add_s = [&](const rq_scalar& x) {
        add(&x.is_float, sizeof x.is_float);
        add(&x.i, sizeof x.i);
        add(&x.f, sizeof x.f);
      };
      const uint64_t mu = mask ? mask->uid : 0;
      add(&mu, 8);
      for (int i = 0; i < n_keys; ++i) add(&keys[i]->uid, 8);
      key += '|';
      for (int i = 0; i < n_exprs; ++i) {
        const rq_expr& x = exprs[i];
        add(&x.n_terms, sizeof x.n_terms);
        for (int t = 0; t < x.n_terms; ++t) {
          add(&x.terms[t].col->uid, 8);
          add(&x.terms[t].op, sizeof x.terms[t].op);
          add(&x.terms[t].reversed, sizeof x.terms[t].reversed);
          add_s(x.terms[t].k);
          if (t > 0) add(&x.ops[t - 1], sizeof x.ops[t - 1]);
        }
        add(&fns[i], sizeof fns[i]);
      }
      key += '|';
      for (int i = 0; i < n_where; ++i) {
        add(&where[i].col->uid, 8);
        add(&where[i].op, sizeof where[i].op);
        add(&where[i].n_in, sizeof where[i].n_in);
        add_s(where[i].k);
        for (int j = 0; j < where[i].n_in; ++j) add_s(where[i].in_list[j]);
      }
      ctx->graph_key = std::move(key);
      try {
        r = group_aggregate_exprs(ctx, m, k, xs, f, &was_fused, pp);
      } catch (...) {
        ctx->graph_key.clear();
        throw;
      }
      ctx->graph_key.clear();
    }
    if (fused) *fused = was_fused ? 1 : 0;
    if (n_groups) *n_groups = r.n_groups;
    for (int i = 0; i < n_keys; ++i) out_keys[i] = wrap_arr(r.keys[static_cast<size_t>(i)]);
    for (int i = 0; i < n_exprs; ++i) out_vals[i] = wrap_arr(r.vals[static_cast<size_t>(i)]);
  });
}

int rq_group_aggregate_exprs(rq_ctx_t c, rq_mask_t mask, const rq_col_t* keys, int32_t n_keys,
                             const rq_expr* exprs, const int32_t* fns, int32_t n_exprs, int64_t* n_groups,
                             rq_arr_t* out_keys, rq_arr_t* out_vals, int32_t* fused) {
  return group_aggregate_exprs_api(c, nullptr, 0, mask, keys, n_keys, exprs, fns, n_exprs, n_groups, out_keys,
                                   out_vals, fused);
}

int rq_group_aggregate_where_sharded(rq_ctx_t c, rq_comm_t comm, const rq_pred* where, int32_t n_where,
                                     rq_mask_t mask, const rq_col_t* keys, int32_t n_keys, const rq_expr* exprs,
                                     const int32_t* fns, int32_t n_exprs, int64_t* n_groups, rq_arr_t* out_keys,
                                     rq_arr_t* out_vals, int32_t* fused) {
  if (!comm) return api_guard([] { fail("null communicator"); });
  return group_aggregate_exprs_api(c, where, n_where, mask, keys, n_keys, exprs, fns, n_exprs, n_groups, out_keys,
                                   out_vals, fused, comm);
}

int rq_group_aggregate_where(rq_ctx_t c, const rq_pred* where, int32_t n_where, rq_mask_t mask,
                             const rq_col_t* keys, int32_t n_keys, const rq_expr* exprs, const int32_t* fns,
                             int32_t n_exprs, int64_t* n_groups, rq_arr_t* out_keys, rq_arr_t* out_vals,
                             int32_t* fused) {
  return group_aggregate_exprs_api(c, where, n_where, mask, keys, n_keys, exprs, fns, n_exprs, n_groups, out_keys,
                                   out_vals, fused);
}

// ---- host-side row-range sharding -------------------------------------------------

namespace {

void* dup_slice(const void* src, int64_t first, int64_t count, int width) {
  const size_t bytes = static_cast<size_t>(count > 0 ? count : 0) * width;
  void* p = std::malloc(bytes ? bytes : 1);
  if (bytes) std::memcpy(p, static_cast<const char*>(src) + first * width, bytes);
  return p;
}

int64_t lower_bound_h(const int64_t* a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// RLE runs clipped to [lo, hi): first run with e >= lo .. last run with s < hi
void slice_runs(const void* v, int width, const int64_t* s, const int64_t* e, int64_t n, int64_t lo,
                int64_t hi, void** v_out, int64_t** s_out, int64_t** e_out, int64_t* n_out) {
  const int64_t r0 = lower_bound_h(e, n, lo);
  const int64_t r1 = lower_bound_h(s, n, hi);  // first run starting at/after hi
  const int64_t cnt = r1 > r0 ? r1 - r0 : 0;
  *v_out = dup_slice(v, r0, cnt, width);
  *s_out = static_cast<int64_t*>(dup_slice(s, r0, cnt, 8));
  *e_out = static_cast<int64_t*>(dup_slice(e, r0, cnt, 8));
  if (cnt > 0) {
    if ((*s_out)[0] < lo) (*s_out)[0] = lo;            // split run crossing the low cut
    if ((*e_out)[cnt - 1] > hi - 1) (*e_out)[cnt - 1] = hi - 1;  // and the high cut
  }
  *n_out = cnt;
}

void slice_points(const void* v, int width, const int64_t* p, int64_t n, int64_t lo, int64_t hi,
                  void** v_out, int64_t** p_out, int64_t* n_out) {
  const int64_t a = lower_bound_h(p, n, lo);
  const int64_t b = lower_bound_h(p, n, hi);
  const int64_t cnt = b > a ? b - a : 0;
  *v_out = dup_slice(v, a, cnt, width);
  *p_out = static_cast<int64_t*>(dup_slice(p, a, cnt, 8));
  *n_out = cnt;
}

}  // namespace

// Row-range shard of a host column image: rows [lo, hi) of
// the table become a standalone table of hi - lo rows. Runs crossing a cut
// are split with their value duplicated; every position is rebased to the
// shard (p - lo) and total_size = hi - lo, so all columns of a shard align
// with each other, shard aggregates combine into the global aggregate, and
// materialised shard outputs concatenate (after adding lo) into the global
// result in shard order.
int rq_shard_host_column(const rq_host_column* in, int64_t lo, int64_t hi, rq_host_column* out) {
  return api_guard([&] {
    require(in && out, "null argument");
    require(0 <= lo && lo <= hi, "shard: bad row range");
    std::memset(out, 0, sizeof(*out));
    *out = *in;
    out->v = out->v2 = nullptr;
    out->s = out->e = out->p = out->p2 = nullptr;
    out->total_size = hi - lo;
    const int w = dt_width(in->dtype);
    auto rebase = [&](int64_t* a, int64_t n) {
      for (int64_t i = 0; i < n; ++i) a[i] -= lo;
    };
    switch (in->encoding) {
      case RQ_ENC_PLAIN:
      case RQ_ENC_PLAIN_INDEX: {
        require(hi <= in->n, "shard: range beyond plain column");
        out->n = hi - lo;
        out->v = dup_slice(in->v, lo, hi - lo, w);
        if (in->encoding == RQ_ENC_PLAIN_INDEX) {
          slice_points(in->v2, dt_width(in->dtype2), in->p2, in->n2, lo, hi, &out->v2, &out->p2,
                       &out->n2);
          rebase(out->p2, out->n2);
        }
        break;
      }
      case RQ_ENC_RLE:
        require(hi <= in->total_size, "shard: range beyond column");
        slice_runs(in->v, w, in->s, in->e, in->n, lo, hi, &out->v, &out->s, &out->e, &out->n);
        rebase(out->s, out->n);
        rebase(out->e, out->n);
        break;
      case RQ_ENC_INDEX:
        require(hi <= in->total_size, "shard: range beyond column");
        slice_points(in->v, w, in->p, in->n, lo, hi, &out->v, &out->p, &out->n);
        rebase(out->p, out->n);
        break;
      case RQ_ENC_RLE_INDEX:
        require(hi <= in->total_size, "shard: range beyond column");
        slice_runs(in->v, w, in->s, in->e, in->n, lo, hi, &out->v, &out->s, &out->e, &out->n);
        rebase(out->s, out->n);
        rebase(out->e, out->n);
        slice_points(in->v2, dt_width(in->dtype2), in->p2, in->n2, lo, hi, &out->v2, &out->p2,
                     &out->n2);
        rebase(out->p2, out->n2);
        break;
      default:
        fail("shard: unknown encoding");
    }
  });
}

void rq_host_column_free(rq_host_column* h) {
  if (!h) return;
  std::free(h->v);
  std::free(h->s);
  std::free(h->e);
  std::free(h->p);
  std::free(h->v2);
  std::free(h->p2);
  h->v = h->v2 = nullptr;
  h->s = h->e = h->p = h->p2 = nullptr;
}

}  // extern "C"
