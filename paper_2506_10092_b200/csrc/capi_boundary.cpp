// capi_boundary.cpp — C ABI for the rest of the reference operator surface
// (include/runq_b200.h, "boundary completions"): decompose / align_many /
// shape weights (align.hpp:25-68), the grouping API (groupby.hpp:12-50), the
// kernels helpers (kernels.hpp:13-72), the remaining enc conversions
// (primitives.hpp:54-92), decode_full / to_rows / stats (column.hpp:162-189).
// Every data-touching step is a device kernel (k_boundary.cu and the
// existing primitives); host code only moves handles and sizes.
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
void put(rq_arr_t* out, const DArr& a) {
  if (out) *out = wrap_arr(a);
}
void put_shape(const Decomp& d, int32_t* kind, int64_t* n, rq_arr_t* s, rq_arr_t* e, rq_arr_t* p) {
  if (kind) *kind = d.kind;
  if (n) *n = d.kind == 0 ? d.n : d.kind == 1 ? d.s.n : d.p.n;
  if (d.kind == 1) {
    put(s, d.s);
    put(e, d.e);
  } else if (s || e) {
    if (s) *s = nullptr;
    if (e) *e = nullptr;
  }
  if (d.kind == 2) put(p, d.p);
  else if (p) *p = nullptr;
}
Decomp shape_in(int32_t kind, int64_t n, rq_arr_t s, rq_arr_t e, rq_arr_t p) {
  Decomp d;
  require(kind >= 0 && kind <= 2, "shape: kind must be 0 (dense), 1 (run) or 2 (point)");
  d.kind = kind;
  if (kind == 0) d.n = n;
  if (kind == 1) {
    d.s = arr_of(s);
    d.e = arr_of(e);
    require(d.s.n == d.e.n, "shape: run starts / ends length mismatch");
  }
  if (kind == 2) d.p = arr_of(p);
  return d;
}
std::vector<const DCol*> cols_of(const rq_col_t* cols, int32_t n) {
  std::vector<const DCol*> v;
  for (int i = 0; i < n; ++i) v.push_back(&col_of(cols[i]));
  return v;
}

}  // namespace

extern "C" {

int rq_decompose(rq_ctx_t c, rq_col_t col, int32_t* kind, int64_t* n, rq_arr_t* s, rq_arr_t* e, rq_arr_t* p,
                 rq_arr_t* values) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    Decomp d = decompose_for_group(ctx, col_of(col));
    put_shape(d, kind, n, s, e, p);
    put(values, d.values);
  });
}

int rq_align_many(rq_ctx_t c, const rq_col_t* cols, int32_t ncols, int32_t* kind, int64_t* n, rq_arr_t* s,
                  rq_arr_t* e, rq_arr_t* p, rq_arr_t* values) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(ncols > 0, "align_many: no columns");
    MultiAligned ma = align_many(ctx, cols_of(cols, ncols));
    put_shape(ma.shape, kind, n, s, e, p);
    for (int i = 0; i < ncols; ++i) values[i] = wrap_arr(ma.values[static_cast<size_t>(i)]);
  });
}

int rq_shape_weights(rq_ctx_t c, int32_t kind, int64_t n, rq_arr_t s, rq_arr_t e, rq_arr_t p, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    put(out, shape_weights(ctx, shape_in(kind, n, s, e, p)));
  });
}

int rq_group_on_arrays(rq_ctx_t c, const rq_arr_t* key_values, int32_t n_keys, rq_arr_t* inverse,
                       rq_arr_t* keys_out, int64_t* n_groups) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(n_keys > 0, "group: empty key list");
    std::vector<DArr> kv;
    for (int i = 0; i < n_keys; ++i) kv.push_back(arr_of(key_values[i]));
    Unique u = unique_with_inverse(ctx, kv);
    put(inverse, u.inverse);
    for (int i = 0; i < n_keys; ++i) keys_out[i] = wrap_arr(u.keys[static_cast<size_t>(i)]);
    if (n_groups) *n_groups = u.n_groups;
  });
}

int rq_group(rq_ctx_t c, const rq_col_t* keys, int32_t n_keys, int32_t* kind, int64_t* n, rq_arr_t* s,
             rq_arr_t* e, rq_arr_t* p, rq_arr_t* inverse, rq_arr_t* keys_out, int64_t* n_groups) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(n_keys > 0, "group: empty key list");
    MultiAligned ma = align_many(ctx, cols_of(keys, n_keys));
    Unique u = unique_with_inverse(ctx, ma.values);
    put_shape(ma.shape, kind, n, s, e, p);
    put(inverse, u.inverse);
    for (int i = 0; i < n_keys; ++i) keys_out[i] = wrap_arr(u.keys[static_cast<size_t>(i)]);
    if (n_groups) *n_groups = u.n_groups;
  });
}

int rq_aggregate_array(rq_ctx_t c, int32_t kind, int64_t n, rq_arr_t s, rq_arr_t e, rq_arr_t p, rq_arr_t values,
                       rq_arr_t inverse, int64_t n_groups, int32_t fn, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    put(out, aggregate_array(ctx, shape_in(kind, n, s, e, p), arr_of(values), arr_of(inverse), n_groups, fn));
  });
}

int rq_scatter_reduce(rq_ctx_t c, rq_arr_t values, rq_arr_t index, int64_t n_groups, int32_t reduce,
                      rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(reduce >= RQ_REDUCE_SUM && reduce <= RQ_REDUCE_COUNT, "scatter_reduce: unknown reduction");
    put(out, scatter_reduce(ctx, arr_of(values), arr_of(index), n_groups, reduce));
  });
}

int rq_unique_with_inverse(rq_ctx_t c, const rq_arr_t* cols, int32_t n, rq_arr_t* keys_out, rq_arr_t* inverse,
                           int64_t* n_groups) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    std::vector<DArr> kv;
    for (int i = 0; i < n; ++i) kv.push_back(arr_of(cols[i]));
    Unique u = unique_with_inverse(ctx, kv);
    for (int i = 0; i < n; ++i) keys_out[i] = wrap_arr(u.keys[static_cast<size_t>(i)]);
    put(inverse, n > 0 ? u.inverse : alloc_arr(ctx, RQ_I64, 0));
    if (n_groups) *n_groups = u.n_groups;
  });
}

int rq_cumsum(rq_ctx_t c, rq_arr_t x, int32_t exclusive, rq_arr_t* out) {
  return api_guard([&] { put(out, checked_cumsum(ctx_of(c), arr_of(x), exclusive != 0)); });
}

int rq_checked_sum(rq_ctx_t c, rq_arr_t x, int64_t* out) {
  return api_guard([&] {
    const int64_t v = checked_sum(ctx_of(c), arr_of(x));
    if (out) *out = v;
  });
}

int rq_repeat_interleave(rq_ctx_t c, rq_arr_t values, rq_arr_t counts, rq_arr_t* out) {
  return api_guard([&] { put(out, repeat_interleave(ctx_of(c), arr_of(values), arr_of(counts))); });
}

int rq_range_arange(rq_ctx_t c, rq_arr_t start, rq_arr_t length, rq_arr_t* out) {
  return api_guard([&] { put(out, range_arange(ctx_of(c), arr_of(start), arr_of(length))); });
}

int rq_gather(rq_ctx_t c, rq_arr_t values, rq_arr_t idx, rq_arr_t* out) {
  return api_guard([&] { put(out, gather_checked(ctx_of(c), arr_of(values), arr_of(idx))); });
}

int rq_sort_with_perm(rq_ctx_t c, rq_arr_t values, rq_arr_t* sorted, rq_arr_t* perm) {
  return api_guard([&] {
    DArr so, pe;
    sort_with_perm(ctx_of(c), arr_of(values), so, pe);
    put(sorted, so);
    put(perm, pe);
  });
}

int rq_adjacent_ne(rq_ctx_t c, rq_arr_t x, rq_arr_t* out) {
  return api_guard([&] { put(out, adjacent_ne(ctx_of(c), arr_of(x))); });
}

int rq_range_union(rq_ctx_t c, rq_arr_t s1, rq_arr_t e1, rq_arr_t s2, rq_arr_t e2, rq_arr_t* s, rq_arr_t* e) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    require(arr_of(s1).n == arr_of(e1).n && arr_of(s2).n == arr_of(e2).n, "range_union: run list length mismatch");
    DArr S = merge_keys(ctx, arr_of(s1), arr_of(s2)), E = merge_keys(ctx, arr_of(e1), arr_of(e2));
    DArr so, eo;
    union_from_merged(ctx, S, E, so, eo);
    put(s, so);
    put(e, eo);
  });
}

namespace {
// sorted list with duplicates removed (std::unique after a merge / sort)
DArr dedup_sorted(const CtxPtr& ctx, const DArr& sorted) {
  DArr out;
  if (sorted.n == 0) return sorted;
  select_points(ctx, adjacent_ne(ctx, sorted), sorted, out, nullptr);
  return out;
}
}  // namespace

int rq_merge_sorted_idx(rq_ctx_t c, rq_arr_t p1, rq_arr_t p2, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    put(out, dedup_sorted(ctx, merge_keys(ctx, arr_of(p1), arr_of(p2))));
  });
}

int rq_concat_sort_idx(rq_ctx_t c, rq_arr_t p1, rq_arr_t p2, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DArr &a = arr_of(p1), &b = arr_of(p2);
    require(a.dt == RQ_I64 && b.dt == RQ_I64, "concat_sort_idx: int64 positions required");
    DArr cat = alloc_arr(ctx, RQ_I64, a.n + b.n);
    if (a.n) RQ_CUDA_CHECK(cudaMemcpyAsync(cat.raw_mut(), a.raw(), a.bytes(), cudaMemcpyDeviceToDevice, ctx->stream));
    if (b.n)
      RQ_CUDA_CHECK(cudaMemcpyAsync(cat.as<int64_t>() + a.n, b.raw(), b.bytes(), cudaMemcpyDeviceToDevice,
                                    ctx->stream));
    DArr sorted, perm;
    sort_with_perm(ctx, cat, sorted, perm);
    put(out, dedup_sorted(ctx, sorted));
  });
}

int rq_complement_rle(rq_ctx_t c, rq_arr_t s, rq_arr_t e, int64_t total, rq_arr_t* s_out, rq_arr_t* e_out) {
  return api_guard([&] {
    DArr so, eo;
    complement_runs(ctx_of(c), arr_of(s), arr_of(e), total, so, eo);
    put(s_out, so);
    put(e_out, eo);
  });
}

int rq_complement_index(rq_ctx_t c, rq_arr_t p, int64_t total, rq_arr_t* s_out, rq_arr_t* e_out) {
  return api_guard([&] {
    DArr so, eo;
    complement_runs(ctx_of(c), arr_of(p), arr_of(p), total, so, eo);  // points are one-row runs
    put(s_out, so);
    put(e_out, eo);
  });
}

int rq_rle_to_index(rq_ctx_t c, rq_col_t col, int64_t budget, rq_col_t* out) {
  return api_guard([&] { *out = wrap_col(rle_to_index(ctx_of(c), col_of(col), budget)); });
}

int rq_rle_to_plain(rq_ctx_t c, rq_col_t col, double fill, int64_t budget, rq_col_t* out) {
  return api_guard([&] { *out = wrap_col(rle_to_plain(ctx_of(c), col_of(col), fill, budget)); });
}

int rq_mask_rle_to_index(rq_ctx_t c, rq_mask_t m, int64_t budget, rq_mask_t* out) {
  return api_guard([&] { *out = wrap_mask(rle_mask_to_index(ctx_of(c), mask_of(m), budget)); });
}

int rq_mask_rle_to_plain(rq_ctx_t c, rq_mask_t m, int64_t budget, rq_mask_t* out) {
  return api_guard([&] { *out = wrap_mask(rle_mask_to_plain(ctx_of(c), mask_of(m), budget)); });
}

int rq_compact_rle_index(rq_ctx_t c, rq_col_t col, rq_col_t* out) {
  return api_guard([&] { *out = wrap_col(compact_rle_index(ctx_of(c), col_of(col))); });
}

int rq_decode_full(rq_ctx_t c, rq_col_t col, rq_arr_t* out) {
  return api_guard([&] { put(out, decode_full(ctx_of(c), col_of(col))); });
}

int rq_to_rows(rq_ctx_t c, rq_col_t col, rq_arr_t* positions, rq_arr_t* values) {
  return api_guard([&] {
    DArr p, v;
    col_to_rows(ctx_of(c), col_of(col), p, v);
    put(positions, p);
    put(values, v);
  });
}

int rq_col_stats(rq_ctx_t c, rq_col_t col, rq_column_stats* out) {
  return api_guard([&] {
    auto ctx = ctx_of(c);
    const DCol& x = col_of(col);
    require(out != nullptr, "null out");
    rq_column_stats st{};
    st.plain_bytes = x.total * dt_width(x.value_type());
    auto runs_bytes = [&](const DArr& v, int64_t nr) { return nr * (dt_width(v.dt) + 16); };
    switch (x.enc) {
      case RQ_ENC_PLAIN: st.encoded_bytes = static_cast<int64_t>(x.v.bytes()); break;
      case RQ_ENC_RLE:
        st.n_runs = x.s.n;
        st.encoded_bytes = runs_bytes(x.v, x.s.n);
        if (st.n_runs > 0) st.avg_run_length = static_cast<double>(covered_rows(ctx, x.s, x.e)) / st.n_runs;
        break;
      case RQ_ENC_INDEX:
        st.n_runs = x.p.n;
        st.encoded_bytes = x.p.n * (dt_width(x.v.dt) + 8);
        if (st.n_runs > 0) st.avg_run_length = 1.0;
        break;
      case RQ_ENC_PLAIN_INDEX:
        st.encoded_bytes = static_cast<int64_t>(x.v.bytes()) + x.p2.n * (dt_width(x.v2.dt) + 8);
        break;
      default:
        st.n_runs = x.s.n;
        st.encoded_bytes = runs_bytes(x.v, x.s.n) + x.p2.n * (dt_width(x.v2.dt) + 8);
        if (st.n_runs > 0) st.avg_run_length = static_cast<double>(covered_rows(ctx, x.s, x.e)) / st.n_runs;
        break;
    }
    if (st.encoded_bytes > 0)
      st.compression_ratio = static_cast<double>(st.plain_bytes) / static_cast<double>(st.encoded_bytes);
    *out = st;
  });
}

}  // extern "C"
