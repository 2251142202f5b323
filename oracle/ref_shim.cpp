// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. extern "C" adapter over the
// UNMODIFIED reference library (compiled from /root/reference/proj/core/src
// in place by oracle/Makefile). Converts host column images to runq::Column,
// calls the reference operator API, converts results back. Nothing here is
// on the product path; see ref_shim.h.
#include <sstream>
#include "ref_shim.h"

#include <chrono>
#include <map>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "runq/align.hpp"
#include "runq/column.hpp"
#include "runq/groupby.hpp"
#include "runq/join.hpp"
#include "runq/runner.hpp"
#include "runq/ingest.hpp"
#include "runq/table.hpp"
#include "runq/kernels.hpp"
#include "runq/mask_ops.hpp"
#include "runq/primitives.hpp"

using namespace runq;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return RQ_OK;
  } catch (const OverflowError& ex) {
    g_err = ex.what();
    return RQ_OVERFLOW;
  } catch (const ResourceError& ex) {
    g_err = ex.what();
    return RQ_RESOURCE;
  } catch (const Error& ex) {
    g_err = ex.what();
    return RQ_INVALID;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return RQ_INVALID;
  }
}

DType dt(int32_t d) { return static_cast<DType>(d); }

Array make_array(int32_t dtype, int64_t n, const void* data) {
  return dtype_dispatch(dt(dtype), [&](auto tag) {
    using T = decltype(tag);
    if (n == 0 || data == nullptr) return Array::empty(dtype_of_v<T>);
    return Array::from(std::span<const T>(static_cast<const T*>(data), static_cast<size_t>(n)));
  });
}

PosVec make_pos(int64_t n, const int64_t* p) {
  PosVec v(static_cast<size_t>(n));
  if (n) std::memcpy(v.data(), p, static_cast<size_t>(n) * 8);
  return v;
}

Column to_column(const rq_host_column* h) {
  switch (h->encoding) {
    case RQ_ENC_PLAIN: {
      std::optional<int64_t> c;
      if (h->has_center) c = h->center;
      return PlainColumn(make_array(h->dtype, h->n, h->v), dt(h->logical), c);
    }
    case RQ_ENC_RLE:
      return RleColumn{make_array(h->dtype, h->n, h->v), make_pos(h->n, h->s),
                       make_pos(h->n, h->e), h->total_size};
    case RQ_ENC_INDEX:
      return IndexColumn{make_array(h->dtype, h->n, h->v), make_pos(h->n, h->p), h->total_size};
    case RQ_ENC_PLAIN_INDEX: {
      std::optional<int64_t> c;
      if (h->has_center) c = h->center;
      PlainPlusIndexColumn pc;
      pc.base = PlainColumn(make_array(h->dtype, h->n, h->v), dt(h->logical), c);
      pc.outliers = IndexColumn{make_array(h->dtype2, h->n2, h->v2), make_pos(h->n2, h->p2), h->n};
      return pc;
    }
    case RQ_ENC_RLE_INDEX: {
      RlePlusIndexColumn rc;
      rc.runs = RleColumn{make_array(h->dtype, h->n, h->v), make_pos(h->n, h->s),
                          make_pos(h->n, h->e), h->total_size};
      rc.points = IndexColumn{make_array(h->dtype2, h->n2, h->v2), make_pos(h->n2, h->p2),
                              h->total_size};
      return rc;
    }
  }
  fail("ref_shim: unknown encoding");
}

MaskColumn to_mask(const rq_host_mask* h) {
  switch (h->encoding) {
    case RQ_MASK_PLAIN: {
      PlainMask m;
      m.bits.assign(h->bits, h->bits + h->n);
      return m;
    }
    case RQ_MASK_RLE:
      return RleMask{make_pos(h->n, h->s), make_pos(h->n, h->e), h->total_size};
    case RQ_MASK_INDEX:
      return IndexMask{make_pos(h->n, h->p), h->total_size};
    case RQ_MASK_COMPOSITE:
      return CompositeMask{RleMask{make_pos(h->n, h->s), make_pos(h->n, h->e), h->total_size},
                           IndexMask{make_pos(h->n2, h->p2), h->total_size}};
  }
  fail("ref_shim: unknown mask encoding");
}

void* dup_bytes(const void* src, size_t bytes) {
  void* p = std::malloc(bytes ? bytes : 1);
  if (bytes) std::memcpy(p, src, bytes);
  return p;
}

void* dup_array(const Array& a) { return dup_bytes(a.data(), static_cast<size_t>(a.byte_size())); }
int64_t* dup_pos(const PosVec& v) {
  return static_cast<int64_t*>(dup_bytes(v.data(), v.size() * 8));
}

void fill_array(ref_host_array* out, const Array& a) {
  out->dtype = static_cast<int32_t>(a.dtype());
  out->n = a.size();
  out->data = dup_array(a);
}
void fill_pos(ref_host_array* out, const PosVec& v) {
  out->dtype = RQ_I64;
  out->n = static_cast<int64_t>(v.size());
  out->data = dup_pos(v);
}

void from_column(const Column& c, rq_host_column* h) {
  std::memset(h, 0, sizeof(*h));
  h->encoding = static_cast<int32_t>(c.encoding());
  h->total_size = c.total_size();
  c.visit([&](const auto& x) {
    using T = std::decay_t<decltype(x)>;
    if constexpr (std::is_same_v<T, PlainColumn>) {
      h->dtype = static_cast<int32_t>(x.values.dtype());
      h->logical = static_cast<int32_t>(x.logical);
      h->has_center = x.center.has_value();
      h->center = x.center.value_or(0);
      h->n = x.size();
      h->v = dup_array(x.values);
    } else if constexpr (std::is_same_v<T, RleColumn>) {
      h->dtype = h->logical = static_cast<int32_t>(x.v.dtype());
      h->n = x.run_count();
      h->v = dup_array(x.v);
      h->s = dup_pos(x.s);
      h->e = dup_pos(x.e);
    } else if constexpr (std::is_same_v<T, IndexColumn>) {
      h->dtype = h->logical = static_cast<int32_t>(x.v.dtype());
      h->n = x.point_count();
      h->v = dup_array(x.v);
      h->p = dup_pos(x.p);
    } else if constexpr (std::is_same_v<T, PlainPlusIndexColumn>) {
      h->dtype = static_cast<int32_t>(x.base.values.dtype());
      h->logical = static_cast<int32_t>(x.base.logical);
      h->has_center = x.base.center.has_value();
      h->center = x.base.center.value_or(0);
      h->n = x.base.size();
      h->v = dup_array(x.base.values);
      h->dtype2 = static_cast<int32_t>(x.outliers.v.dtype());
      h->n2 = x.outliers.point_count();
      h->v2 = dup_array(x.outliers.v);
      h->p2 = dup_pos(x.outliers.p);
    } else {
      h->dtype = h->logical = static_cast<int32_t>(x.runs.v.dtype());
      h->n = x.runs.run_count();
      h->v = dup_array(x.runs.v);
      h->s = dup_pos(x.runs.s);
      h->e = dup_pos(x.runs.e);
      h->dtype2 = static_cast<int32_t>(x.points.v.dtype());
      h->n2 = x.points.point_count();
      h->v2 = dup_array(x.points.v);
      h->p2 = dup_pos(x.points.p);
    }
  });
}

void from_mask(const MaskColumn& m, rq_host_mask* h) {
  std::memset(h, 0, sizeof(*h));
  h->encoding = static_cast<int32_t>(m.encoding());
  h->total_size = m.total_size();
  m.visit([&](const auto& x) {
    using T = std::decay_t<decltype(x)>;
    if constexpr (std::is_same_v<T, PlainMask>) {
      h->n = x.size();
      h->bits = static_cast<uint8_t*>(dup_bytes(x.bits.data(), x.bits.size()));
    } else if constexpr (std::is_same_v<T, RleMask>) {
      h->n = x.run_count();
      h->s = dup_pos(x.s);
      h->e = dup_pos(x.e);
    } else if constexpr (std::is_same_v<T, IndexMask>) {
      h->n = static_cast<int64_t>(x.p.size());
      h->p = dup_pos(x.p);
    } else {
      h->n = x.runs.run_count();
      h->s = dup_pos(x.runs.s);
      h->e = dup_pos(x.runs.e);
      h->n2 = static_cast<int64_t>(x.points.p.size());
      h->p2 = dup_pos(x.points.p);
    }
  });
}

std::span<const int64_t> sp(const int64_t* p, int64_t n) {
  return {p, static_cast<size_t>(n)};
}

compute::BinOp bop(int32_t op) { return static_cast<compute::BinOp>(op); }
compute::Scalar scal(rq_scalar k) {
  if (k.is_float) return compute::Scalar(k.f);
  return compute::Scalar(k.i);
}

void put_scalar(const Array& a, int32_t* out_dtype, int64_t* out_i64, double* out_f64) {
  *out_dtype = static_cast<int32_t>(a.dtype());
  if (dtype_is_float(a.dtype())) *out_f64 = a.f64_at(0);
  else *out_i64 = a.i64_at(0);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_free_column(rq_host_column* c) {
  std::free(c->v);
  std::free(c->s);
  std::free(c->e);
  std::free(c->p);
  std::free(c->v2);
  std::free(c->p2);
  std::memset(c, 0, sizeof(*c));
}
void ref_free_mask(rq_host_mask* m) {
  std::free(m->bits);
  std::free(m->s);
  std::free(m->e);
  std::free(m->p);
  std::free(m->p2);
  std::memset(m, 0, sizeof(*m));
}
void ref_free_array(ref_host_array* a) {
  std::free(a->data);
  std::memset(a, 0, sizeof(*a));
}

// runq::dump_column (column.cpp:513-563): the column image as bytes
int ref_dump_column(const rq_host_column* a, ref_host_array* out) {
  return guarded([&] {
    std::ostringstream os;
    dump_column(to_column(a), os);
    const std::string b = os.str();
    out->dtype = 0;
    out->n = static_cast<int64_t>(b.size());
    out->data = dup_bytes(b.data(), b.size());
  });
}

int ref_roundtrip(const rq_host_column* a, rq_host_column* out) {
  return guarded([&] { from_column(to_column(a), out); });
}

int ref_validate(const rq_host_column* a) {
  int n = -1;
  guarded([&] { n = static_cast<int>(validate(to_column(a)).size()); });
  return n;
}

int ref_range_intersect(const int64_t* s1, const int64_t* e1, int64_t n1, const int64_t* s2,
                        const int64_t* e2, int64_t n2, ref_host_array* s, ref_host_array* e,
                        ref_host_array* idx1, ref_host_array* idx2) {
  return guarded([&] {
    auto r = enc::range_intersect(sp(s1, n1), sp(e1, n1), sp(s2, n2), sp(e2, n2));
    fill_pos(s, r.s);
    fill_pos(e, r.e);
    fill_pos(idx1, r.idx1);
    fill_pos(idx2, r.idx2);
  });
}

int ref_idx_in_rle(const int64_t* p, int64_t np, const int64_t* s, const int64_t* e, int64_t nr,
                   ref_host_array* p_out, ref_host_array* run_of, ref_host_array* idx_of) {
  return guarded([&] {
    auto r = enc::idx_in_rle(sp(p, np), sp(s, nr), sp(e, nr));
    fill_pos(p_out, r.p_out);
    fill_pos(run_of, r.run_of);
    fill_pos(idx_of, r.idx_of);
  });
}

int ref_rle_contain_idx(const int64_t* p, int64_t np, const int64_t* s, const int64_t* e,
                        int64_t nr, ref_host_array* p_out, ref_host_array* run_of,
                        ref_host_array* idx_of) {
  return guarded([&] {
    auto r = enc::rle_contain_idx(sp(p, np), sp(s, nr), sp(e, nr));
    fill_pos(p_out, r.p_out);
    fill_pos(run_of, r.run_of);
    fill_pos(idx_of, r.idx_of);
  });
}

int ref_idx_in_idx(const int64_t* p1, int64_t n1, const int64_t* p2, int64_t n2,
                   ref_host_array* p_out, ref_host_array* idx1, ref_host_array* idx2) {
  return guarded([&] {
    auto r = enc::idx_in_idx(sp(p1, n1), sp(p2, n2));
    fill_pos(p_out, r.p_out);
    fill_pos(idx1, r.idx1);
    fill_pos(idx2, r.idx2);
  });
}

int ref_bucketize(const int64_t* x, int64_t nx, const int64_t* b, int64_t nb, int32_t right,
                  ref_host_array* out) {
  return guarded([&] { fill_pos(out, kernels::bucketize(sp(x, nx), sp(b, nb), right != 0)); });
}

int ref_plain_mask_to_rle(const rq_host_mask* m, rq_host_mask* out) {
  return guarded([&] { from_mask(enc::plain_mask_to_rle(to_mask(m).plain()), out); });
}
int ref_plain_mask_to_index(const rq_host_mask* m, rq_host_mask* out) {
  return guarded([&] { from_mask(enc::plain_mask_to_index(to_mask(m).plain()), out); });
}
int ref_compact_rle(const rq_host_column* a, rq_host_column* out) {
  return guarded([&] { from_column(enc::compact_rle(to_column(a).rle()), out); });
}
int ref_plain_to_rle(const rq_host_column* a, rq_host_column* out) {
  return guarded([&] { from_column(enc::plain_to_rle(to_column(a).plain()), out); });
}
int ref_plain_to_rle_index(const rq_host_column* a, int64_t min_run, rq_host_column* out) {
  return guarded([&] { from_column(enc::plain_to_rle_index(to_column(a).plain(), min_run), out); });
}
int ref_plain_to_plain_index(const rq_host_column* a, double trim, rq_host_column* out) {
  return guarded([&] { from_column(enc::plain_to_plain_index(to_column(a).plain(), trim), out); });
}

int ref_choose_encoding(const rq_host_column* a, const rq_heuristic* cfg, rq_encoding_choice* out) {
  return guarded([&] {
    io::HeuristicConfig h;
    if (cfg) {
      h.row_threshold = cfg->row_threshold;
      h.ratio_threshold = cfg->ratio_threshold;
      h.trim = cfg->trim;
      h.min_run = cfg->min_run;
      h.unit_run_share = cfg->unit_run_share;
    }
    io::EncodingChoice ch = io::choose_encoding(to_column(a).plain(), h);
    out->scheme = static_cast<int32_t>(ch.scheme);
    out->width = static_cast<int32_t>(ch.width);
    out->min_run = ch.min_run;
    out->trim_fraction = ch.trim_fraction;
    out->has_center = ch.center.has_value() ? 1 : 0;
    out->_pad = 0;
    out->center = ch.center.value_or(0);
  });
}

int ref_encode(const rq_host_column* a, const rq_encoding_choice* c, rq_host_column* out) {
  return guarded([&] {
    io::EncodingChoice ch;
    ch.scheme = static_cast<io::Scheme>(c->scheme);
    ch.width = static_cast<DType>(c->width);
    ch.min_run = c->min_run;
    ch.trim_fraction = c->trim_fraction;
    if (c->has_center) ch.center = c->center;
    from_column(io::encode(to_column(a).plain(), ch), out);
  });
}

int ref_sort_table(const rq_host_column* cols, int32_t ncols, const int32_t* by, int32_t nby,
                   rq_host_column* out) {
  return guarded([&] {
    Table t;
    t.name = "t";
    for (int32_t i = 0; i < ncols; ++i) {
      TableColumn tc;
      tc.name = "c" + std::to_string(i);
      tc.column = std::make_shared<Column>(to_column(&cols[i]));
      t.columns.push_back(tc);
    }
    t.rows = ncols > 0 ? t.columns[0].column->total_size() : 0;
    std::vector<std::string> keys;
    for (int32_t i = 0; i < nby; ++i) keys.push_back("c" + std::to_string(by[i]));
    Table s = io::sort_table(t, keys);
    for (int32_t i = 0; i < ncols; ++i) from_column(*s.columns[static_cast<size_t>(i)].column, &out[i]);
  });
}

int ref_decode_values(const rq_host_column* a, ref_host_array* out) {
  return guarded([&] {
    Column c = to_column(a);
    if (c.encoding() == Encoding::Plain) fill_array(out, decode_values(c.plain()));
    else if (c.encoding() == Encoding::PlainPlusIndex)
      fill_array(out, decode_values(c.plain_index()));
    else fail("decode_values: plain or plain+index only");
  });
}

int ref_normalize_basic(const rq_host_column* a, rq_host_column* out) {
  return guarded([&] { from_column(compute::normalize_basic(to_column(a)), out); });
}

int ref_align(const rq_host_column* a, const rq_host_column* b, int32_t* shape_kind,
              ref_host_array* s, ref_host_array* e, ref_host_array* p, ref_host_array* v1,
              ref_host_array* v2) {
  return guarded([&] {
    auto ap = compute::align(to_column(a), to_column(b));
    *shape_kind = static_cast<int32_t>(ap.shape.index());
    if (auto* r = std::get_if<compute::RunShape>(&ap.shape)) {
      fill_pos(s, r->s);
      fill_pos(e, r->e);
    } else if (auto* q = std::get_if<compute::PointShape>(&ap.shape)) {
      fill_pos(p, q->p);
    }
    fill_array(v1, ap.v1);
    fill_array(v2, ap.v2);
  });
}

int ref_arith(const rq_host_column* a, const rq_host_column* b, int32_t op, rq_host_column* out) {
  return guarded([&] { from_column(compute::arith(to_column(a), to_column(b), bop(op)), out); });
}
int ref_compare(const rq_host_column* a, const rq_host_column* b, int32_t op, rq_host_mask* out) {
  return guarded([&] { from_mask(compute::compare(to_column(a), to_column(b), bop(op)), out); });
}
int ref_arith_scalar(const rq_host_column* a, rq_scalar k, int32_t op, int32_t reversed,
                     rq_host_column* out) {
  return guarded([&] {
    from_column(compute::arith_scalar(to_column(a), scal(k), bop(op), reversed != 0), out);
  });
}
int ref_compare_scalar(const rq_host_column* a, rq_scalar k, int32_t op, int32_t reversed,
                       rq_host_mask* out) {
  return guarded([&] {
    from_mask(compute::compare_scalar(to_column(a), scal(k), bop(op), reversed != 0), out);
  });
}
int ref_filter(const rq_host_column* a, const rq_host_mask* m, rq_host_column* out) {
  return guarded([&] { from_column(compute::filter(to_column(a), to_mask(m)), out); });
}
int ref_and_mask(const rq_host_mask* a, const rq_host_mask* b, rq_host_mask* out) {
  return guarded([&] { from_mask(masks::and_mask(to_mask(a), to_mask(b)), out); });
}
int ref_or_mask(const rq_host_mask* a, const rq_host_mask* b, rq_host_mask* out) {
  return guarded([&] { from_mask(masks::or_mask(to_mask(a), to_mask(b)), out); });
}
int ref_not_mask(const rq_host_mask* a, rq_host_mask* out) {
  return guarded([&] { from_mask(masks::not_mask(to_mask(a)), out); });
}
namespace {
void side_out(const joins::JoinIndex& j, ref_join_side* o) {
  o->is_rle = j.is_rle() ? 1 : 0;
  auto dupv = [](const PosVec& v) {
    return static_cast<int64_t*>(dup_bytes(v.data(), v.size() * sizeof(int64_t)));
  };
  if (j.is_rle()) {
    o->n = static_cast<int64_t>(j.rle().s.size());
    o->rows = nullptr;
    o->v = dupv(j.rle().v);
    o->s = dupv(j.rle().s);
    o->e = dupv(j.rle().e);
  } else {
    o->n = static_cast<int64_t>(j.index().rows.size());
    o->rows = dupv(j.index().rows);
    o->v = o->s = o->e = nullptr;
  }
}
joins::JoinIndex side_in(const ref_join_side* j) {
  auto vec = [&](const int64_t* p) { return PosVec(p, p + j->n); };
  if (j->is_rle) return joins::JoinIndex(joins::UnsortedRleJoin{vec(j->v), vec(j->s), vec(j->e)});
  return joins::JoinIndex(joins::UnsortedIndexJoin{vec(j->rows)});
}
}  // namespace

int ref_get_join_index(const rq_host_column* left, const rq_host_column* right, ref_join_side* lo,
                       ref_join_side* ro, int64_t* cardinality) {
  return guarded([&] {
    joins::JoinResult r = joins::get_join_index(to_column(left), to_column(right));
    side_out(r.left, lo);
    side_out(r.right, ro);
    *cardinality = r.cardinality;
  });
}
int ref_apply_join_index(const rq_host_column* col, const ref_join_side* j, rq_host_column* out) {
  return guarded([&] { from_column(joins::apply_join_index(to_column(col), side_in(j)), out); });
}
void ref_free(void* p) { std::free(p); }

// ---- query runner (runner.cpp:457-520) over a catalog built from column images ----
struct RefCatalog {
  query::Catalog cat;
  std::map<std::string, DictionaryPtr> dicts;
};
struct RefResult {
  query::ResultTable t;
};
int ref_catalog_create(void** out) {
  return guarded([&] { *out = new RefCatalog{}; });
}
void ref_catalog_free(void* c) { delete static_cast<RefCatalog*>(c); }
int ref_catalog_add_column(void* cp, const char* table, const char* column, const rq_host_column* col,
                           const char* const* dict, int64_t dict_n, const char* dict_name, int32_t is_date) {
  return guarded([&] {
    auto* c = static_cast<RefCatalog*>(cp);
    Table* t = nullptr;
    for (auto& x : c->cat.tables)
      if (x.name == table) t = &x;
    if (!t) {
      c->cat.tables.push_back(Table{});
      t = &c->cat.tables.back();
      t->name = table;
    }
    Column colv = to_column(col);
    t->rows = colv.total_size();
    DictionaryPtr dp;
    if (dict_n > 0 || dict_name) {
      const std::string key = dict_name ? dict_name : std::string(table) + "." + column;
      auto it = c->dicts.find(key);
      if (it != c->dicts.end() && dict_n == 0) {
        dp = it->second;
      } else {
        auto nd = std::make_shared<Dictionary>();
        for (int64_t i = 0; i < dict_n; ++i) nd->intern(dict[i]);
        dp = nd;
        c->dicts[key] = dp;
      }
    }
    t->columns.push_back(TableColumn{column, std::make_shared<const Column>(std::move(colv)), dp, is_date != 0});
  });
}
int ref_run_plan(void* cp, const char* json, void** out) {
  return guarded([&] {
    auto* c = static_cast<RefCatalog*>(cp);
    query::PlanPtr plan = query::parse_plan_json(json);
    query::RunReport r = query::run(c->cat, *plan, query::RunMode::Compressed);
    *out = new RefResult{std::move(r.result)};
  });
}
int ref_result_info(void* rp, int32_t* ncols, int64_t* rows) {
  return guarded([&] {
    auto* r = static_cast<RefResult*>(rp);
    *ncols = static_cast<int32_t>(r->t.columns.size());
    *rows = r->t.rows;
  });
}
int ref_result_column(void* rp, int32_t i, const char** name, int32_t* dtype, const void** data, int64_t* n) {
  return guarded([&] {
    auto* r = static_cast<RefResult*>(rp);
    const Array& a = r->t.columns[static_cast<size_t>(i)];
    *name = r->t.names[static_cast<size_t>(i)].c_str();
    *dtype = static_cast<int32_t>(a.dtype());
    *data = a.data();
    *n = a.size();
  });
}
void ref_result_free(void* r) { delete static_cast<RefResult*>(r); }
int ref_hash_build_probe(const void* bv, int32_t bdt, int64_t nb, const void* pv, int32_t pdt, int64_t np,
                         int64_t** bpos, int64_t** ppos, int64_t* n) {
  return guarded([&] {
    joins::ProbeHits h = joins::hash_build_probe(make_array(bdt, nb, bv), make_array(pdt, np, pv));
    *n = static_cast<int64_t>(h.build_pos.size());
    *bpos = static_cast<int64_t*>(dup_bytes(h.build_pos.data(), h.build_pos.size() * 8));
    *ppos = static_cast<int64_t*>(dup_bytes(h.probe_pos.data(), h.probe_pos.size() * 8));
  });
}

int ref_semi_join_mask(const rq_host_column* probe, const rq_host_column* build, rq_host_mask* out) {
  return guarded([&] { from_mask(joins::semi_join_mask(to_column(probe), to_column(build)), out); });
}
int ref_mask_true_count(const rq_host_mask* a, int64_t* out) {
  return guarded([&] { *out = to_mask(a).true_count(); });
}

int ref_aggregate_all(const rq_host_column* a, int32_t fn, int32_t* out_dtype, int64_t* out_i64,
                      double* out_f64) {
  return guarded([&] {
    Array r = agg::aggregate_all(to_column(a), static_cast<agg::AggFn>(fn));
    put_scalar(r, out_dtype, out_i64, out_f64);
  });
}

int ref_group_aggregate(const rq_host_column* keys, int32_t nk, const rq_host_column* data,
                        const int32_t* fns, int32_t nd, int64_t* n_groups,
                        ref_host_array* out_keys, ref_host_array* out_vals) {
  return guarded([&] {
    std::vector<Column> k, d;
    std::vector<agg::AggFn> f;
    for (int i = 0; i < nk; ++i) k.push_back(to_column(&keys[i]));
    for (int i = 0; i < nd; ++i) {
      d.push_back(to_column(&data[i]));
      f.push_back(static_cast<agg::AggFn>(fns[i]));
    }
    auto r = agg::group_aggregate(k, d, f);
    *n_groups = r.n_groups;
    for (int i = 0; i < nk; ++i) fill_array(&out_keys[i], r.keys[static_cast<size_t>(i)]);
    for (int i = 0; i < nd; ++i) fill_array(&out_vals[i], r.values[static_cast<size_t>(i)]);
  });
}

}  // extern "C"

// --- timed query chains ----------------------------------------------------------

namespace {

struct Partial {
  bool is_float = false;
  uint64_t i = 0;
  double f = 0.0;
  std::string err;
};

template <class Body>
int run_sharded(int32_t nshards, int32_t nthreads, Body&& body, int32_t* out_dtype,
                int64_t* out_i64, double* out_f64, double* seconds) {
  std::vector<Partial> parts(static_cast<size_t>(nshards));
  if (nthreads < 1) nthreads = 1;
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t) {
    pool.emplace_back([&, t] {
      for (int s = t; s < nshards; s += nthreads) {
        try {
          Array r = body(s);
          auto& p = parts[static_cast<size_t>(s)];
          p.is_float = dtype_is_float(r.dtype());
          if (p.is_float) p.f = r.f64_at(0);
          else p.i = static_cast<uint64_t>(r.i64_at(0));
        } catch (const std::exception& ex) {
          parts[static_cast<size_t>(s)].err = ex.what();
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t isum = 0;
  double fsum = 0.0;
  bool flt = false;
  for (auto& p : parts) {
    if (!p.err.empty()) {
      g_err = p.err;
      return RQ_INVALID;
    }
    flt = p.is_float;
    isum += p.i;  // int64 SUM wraps like the reference's int64 accumulator
    fsum += p.f;
  }
  *out_dtype = flt ? RQ_F64 : RQ_I64;
  *out_i64 = static_cast<int64_t>(isum);
  *out_f64 = fsum;
  g_err.clear();
  return RQ_OK;
}

}  // namespace

extern "C" {

int ref_chain_sum_binop(const rq_host_column* a_shards, const rq_host_column* b_shards,
                        int32_t nshards, int32_t nthreads, int32_t op, int32_t* out_dtype,
                        int64_t* out_i64, double* out_f64, double* seconds) {
  std::vector<Column> as, bs;
  int st = guarded([&] {
    for (int i = 0; i < nshards; ++i) {
      as.push_back(to_column(&a_shards[i]));
      bs.push_back(to_column(&b_shards[i]));
    }
  });
  if (st) return st;
  return run_sharded(
      nshards, nthreads,
      [&](int s) {
        Column sum = compute::arith(as[static_cast<size_t>(s)], bs[static_cast<size_t>(s)], bop(op));
        return agg::aggregate_all(sum, agg::AggFn::Sum);
      },
      out_dtype, out_i64, out_f64, seconds);
}

int ref_chain_filtered_sum(const rq_host_column* c_shards, const rq_host_column* a_shards,
                           const rq_host_column* b_shards, int32_t nshards, int32_t nthreads,
                           rq_scalar k, int32_t cmp, int32_t op, int32_t* out_dtype,
                           int64_t* out_i64, double* out_f64, double* seconds) {
  std::vector<Column> cs, as, bs;
  int st = guarded([&] {
    for (int i = 0; i < nshards; ++i) {
      cs.push_back(to_column(&c_shards[i]));
      as.push_back(to_column(&a_shards[i]));
      bs.push_back(to_column(&b_shards[i]));
    }
  });
  if (st) return st;
  return run_sharded(
      nshards, nthreads,
      [&](int s) {
        auto u = static_cast<size_t>(s);
        MaskColumn m = compute::compare_scalar(cs[u], scal(k), bop(cmp));
        Column fa = compute::filter(as[u], m);
        Column fb = compute::filter(bs[u], m);
        Column prod = compute::arith(fa, fb, bop(op));
        return agg::aggregate_all(prod, agg::AggFn::Sum);
      },
      out_dtype, out_i64, out_f64, seconds);
}

}  // extern "C"
