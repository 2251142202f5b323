// runq_adapter.cpp — the drop-in C++ boundary: the reference's hot-path
// operator API with its exact signatures (runq::compute align.hpp:59-95,
// runq::enc primitives.hpp:28-92, runq::masks mask_ops.hpp:18-20,
// runq::agg groupby.hpp:22-50, runq::kernels kernels.hpp:13-72), each
// implemented as upload → sm_100a kernels (librunq_b200.so, C ABI in
// include/runq_b200.h) → download, with the reference's value semantics and
// exception types (error.hpp:11-26: RQ_INVALID → runq::Error, RQ_OVERFLOW →
// OverflowError, RQ_RESOURCE → ResourceError).
//
// Compiled against the reference's public headers (the types Array, Column,
// MaskColumn, Shape … stay the reference's); it replaces the reference's
// align.cpp, primitives.cpp, mask_ops.cpp, groupby.cpp and kernels.cpp, so a
// reference program linked with this file instead of those five runs its
// operators on the B200. tests/refcheck/ links the reference's own unit
// tests and acceptance suite this way.
//
// Host code here only converts types and moves bytes: every data-touching
// step is a device kernel. One device context per host thread (device 0, or
// RQ_DEVICE).
#include <cstdlib>
#include <cstring>
#include <memory>
#include <utility>
#include <string>

#include "../../include/runq_b200.h"
#include "runq/align.hpp"
#include "runq/groupby.hpp"
#include "runq/kernels.hpp"
#include "runq/mask_ops.hpp"
#include "runq/primitives.hpp"

namespace rqa {

using namespace runq;

[[noreturn]] void raise(int st) {
  std::string msg = rq_last_error();
  switch (st) {
    case RQ_OVERFLOW: throw OverflowError(msg);
    case RQ_RESOURCE: throw ResourceError(msg);
    case RQ_INVALID: throw Error(msg);
    default: throw Error("device: " + msg);
  }
}
inline void ck(int st) {
  if (st != RQ_OK) raise(st);
}

struct Context {
  rq_ctx_t c = nullptr;
  Context() {
    const char* d = std::getenv("RQ_DEVICE");
    ck(rq_ctx_create(d ? std::atoi(d) : 0, &c));
  }
  ~Context() { rq_ctx_destroy(c); }
};
rq_ctx_t ctx() {
  thread_local Context tc;
  return tc.c;
}

// The device (CUDA context, stream, pool) is brought up when the program
// loads, like any library's static state, so the first operator call does
// not pay for driver initialisation.
const bool kWarm = [] {
  if (!std::getenv("RQ_ADAPTER_LAZY")) ctx();
  return true;
}();

// ---- owned handles -----------------------------------------------------------------

struct Arr {
  rq_arr_t h = nullptr;
  Arr() = default;
  explicit Arr(rq_arr_t x) : h(x) {}
  Arr(const Arr&) = delete;
  Arr(Arr&& o) noexcept : h(o.h) { o.h = nullptr; }
  Arr& operator=(Arr&& o) noexcept {
    std::swap(h, o.h);
    return *this;
  }
  ~Arr() {
    if (h) rq_arr_free(h);
  }
};
struct Col {
  rq_col_t h = nullptr;
  Col() = default;
  explicit Col(rq_col_t x) : h(x) {}
  Col(const Col&) = delete;
  Col(Col&& o) noexcept : h(o.h) { o.h = nullptr; }
  Col& operator=(Col&& o) noexcept {
    std::swap(h, o.h);
    return *this;
  }
  ~Col() {
    if (h) rq_col_free(h);
  }
};
struct Msk {
  rq_mask_t h = nullptr;
  Msk() = default;
  explicit Msk(rq_mask_t x) : h(x) {}
  Msk(const Msk&) = delete;
  Msk(Msk&& o) noexcept : h(o.h) { o.h = nullptr; }
  Msk& operator=(Msk&& o) noexcept {
    std::swap(h, o.h);
    return *this;
  }
  ~Msk() {
    if (h) rq_mask_free(h);
  }
};

int32_t dt(DType t) { return static_cast<int32_t>(t); }  // same order (dtype.hpp:11 / rq_dtype)

Arr up(const Array& a) {
  Arr r;
  ck(rq_arr_upload(ctx(), dt(a.dtype()), a.size() ? a.data() : nullptr, a.size(), &r.h));
  return r;
}
Arr up(std::span<const int64_t> p) {
  Arr r;
  ck(rq_arr_upload(ctx(), RQ_I64, p.empty() ? nullptr : p.data(), static_cast<int64_t>(p.size()), &r.h));
  return r;
}

Array down(rq_arr_t h) {
  int32_t t = RQ_I64;
  int64_t n = 0;
  ck(rq_arr_info(h, &t, &n));
  Array a = Array::zeros(static_cast<DType>(t), n);
  if (n) ck(rq_arr_download(ctx(), h, const_cast<std::byte*>(a.data())));
  return a;
}
Array down(const Arr& a) { return down(a.h); }
PosVec down_pos(rq_arr_t h) {
  int32_t t = RQ_I64;
  int64_t n = 0;
  ck(rq_arr_info(h, &t, &n));
  if (t != RQ_I64) throw Error("adapter: expected an int64 position array");
  PosVec v(static_cast<size_t>(n));
  if (n) ck(rq_arr_download(ctx(), h, v.data()));
  return v;
}
PosVec down_pos(const Arr& a) { return down_pos(a.h); }

void* vp(const void* p) { return const_cast<void*>(p); }
int64_t* pp(const PosVec& v) { return const_cast<int64_t*>(v.data()); }

// ---- columns / masks ------------------------------------------------------------

void fill_plain(rq_host_column& h, const PlainColumn& c) {
  h.dtype = dt(c.values.dtype());
  h.logical = dt(c.logical);
  h.has_center = c.center.has_value();
  h.center = c.center.value_or(0);
  h.n = c.values.size();
  h.total_size = c.values.size();
  h.v = vp(c.values.data());
}

Col up(const Column& col) {
  rq_host_column h{};
  h.encoding = static_cast<int32_t>(col.encoding());
  h.total_size = col.total_size();
  col.visit([&](const auto& c) {
    using T = std::decay_t<decltype(c)>;
    if constexpr (std::is_same_v<T, PlainColumn>) {
      fill_plain(h, c);
    } else if constexpr (std::is_same_v<T, RleColumn>) {
      h.dtype = dt(c.v.dtype());
      h.n = c.run_count();
      h.v = vp(c.v.data());
      h.s = pp(c.s);
      h.e = pp(c.e);
      if (h.n == 0) h.s = h.e = nullptr;
    } else if constexpr (std::is_same_v<T, IndexColumn>) {
      h.dtype = dt(c.v.dtype());
      h.n = c.point_count();
      h.v = vp(c.v.data());
      h.p = pp(c.p);
    } else if constexpr (std::is_same_v<T, PlainPlusIndexColumn>) {
      fill_plain(h, c.base);
      h.encoding = RQ_ENC_PLAIN_INDEX;
      h.dtype2 = dt(c.outliers.v.dtype());
      h.n2 = c.outliers.point_count();
      h.v2 = vp(c.outliers.v.data());
      h.p2 = pp(c.outliers.p);
    } else {
      h.dtype = dt(c.runs.v.dtype());
      h.n = c.runs.run_count();
      h.v = vp(c.runs.v.data());
      h.s = pp(c.runs.s);
      h.e = pp(c.runs.e);
      if (h.n == 0) h.s = h.e = nullptr;
      h.dtype2 = dt(c.points.v.dtype());
      h.n2 = c.points.point_count();
      h.v2 = vp(c.points.v.data());
      h.p2 = pp(c.points.p);
    }
  });
  if (h.encoding == RQ_ENC_RLE || h.encoding == RQ_ENC_RLE_INDEX) {
    // an empty s would read as "gapless, starts implied": only pass NULL when
    // there are no runs at all
    if (h.n > 0 && h.s == nullptr) throw Error("adapter: run starts missing");
  }
  Col r;
  ck(rq_col_upload(ctx(), &h, &r.h));
  return r;
}

Array make_array(int32_t t, int64_t n, void** ptr) {
  Array a = Array::zeros(static_cast<DType>(t), n);
  *ptr = n ? vp(a.data()) : nullptr;
  return a;
}

Column down(const Col& col) {
  rq_host_column h{};
  ck(rq_col_describe(col.h, &h));
  Array v = make_array(h.dtype, h.n, &h.v);
  PosVec s, e, p;
  Array v2;
  PosVec p2;
  if (h.encoding == RQ_ENC_RLE || h.encoding == RQ_ENC_RLE_INDEX) {
    s.resize(static_cast<size_t>(h.n));
    e.resize(static_cast<size_t>(h.n));
    h.s = s.data();
    h.e = e.data();
  }
  if (h.encoding == RQ_ENC_INDEX) {
    p.resize(static_cast<size_t>(h.n));
    h.p = p.data();
  }
  if (h.encoding == RQ_ENC_PLAIN_INDEX || h.encoding == RQ_ENC_RLE_INDEX) {
    v2 = make_array(h.dtype2, h.n2, &h.v2);
    p2.resize(static_cast<size_t>(h.n2));
    h.p2 = p2.data();
  }
  ck(rq_col_download(ctx(), col.h, &h));
  const std::optional<int64_t> center = h.has_center ? std::optional<int64_t>(h.center) : std::nullopt;
  switch (h.encoding) {
    case RQ_ENC_PLAIN: return PlainColumn(std::move(v), static_cast<DType>(h.logical), center);
    case RQ_ENC_RLE: return RleColumn{std::move(v), std::move(s), std::move(e), h.total_size};
    case RQ_ENC_INDEX: return IndexColumn{std::move(v), std::move(p), h.total_size};
    case RQ_ENC_PLAIN_INDEX:
      return PlainPlusIndexColumn{PlainColumn(std::move(v), static_cast<DType>(h.logical), center),
                                  IndexColumn{std::move(v2), std::move(p2), h.total_size}};
    default:
      return RlePlusIndexColumn{RleColumn{std::move(v), std::move(s), std::move(e), h.total_size},
                                IndexColumn{std::move(v2), std::move(p2), h.total_size}};
  }
}

Msk up(const MaskColumn& m) {
  rq_host_mask h{};
  h.encoding = static_cast<int32_t>(m.encoding());
  h.total_size = m.total_size();
  m.visit([&](const auto& x) {
    using T = std::decay_t<decltype(x)>;
    if constexpr (std::is_same_v<T, PlainMask>) {
      h.n = x.size();
      h.bits = const_cast<uint8_t*>(x.bits.data());
    } else if constexpr (std::is_same_v<T, RleMask>) {
      h.n = x.run_count();
      h.s = pp(x.s);
      h.e = pp(x.e);
    } else if constexpr (std::is_same_v<T, IndexMask>) {
      h.n = static_cast<int64_t>(x.p.size());
      h.p = pp(x.p);
    } else {
      h.n = x.runs.run_count();
      h.s = pp(x.runs.s);
      h.e = pp(x.runs.e);
      h.n2 = static_cast<int64_t>(x.points.p.size());
      h.p2 = pp(x.points.p);
    }
  });
  Msk r;
  ck(rq_mask_upload(ctx(), &h, &r.h));
  return r;
}

MaskColumn down(const Msk& m) {
  rq_host_mask h{};
  ck(rq_mask_describe(m.h, &h));
  TrackedVec<uint8_t> bits;
  PosVec s, e, p, p2;
  switch (h.encoding) {
    case RQ_MASK_PLAIN: bits.resize(static_cast<size_t>(h.n)); h.bits = bits.data(); break;
    case RQ_MASK_RLE: s.resize(h.n); e.resize(h.n); h.s = s.data(); h.e = e.data(); break;
    case RQ_MASK_INDEX: p.resize(h.n); h.p = p.data(); break;
    default:
      s.resize(h.n); e.resize(h.n); p2.resize(h.n2);
      h.s = s.data(); h.e = e.data(); h.p2 = p2.data();
  }
  ck(rq_mask_download(ctx(), m.h, &h));
  switch (h.encoding) {
    case RQ_MASK_PLAIN: return PlainMask{std::move(bits)};
    case RQ_MASK_RLE: return RleMask{std::move(s), std::move(e), h.total_size};
    case RQ_MASK_INDEX: return IndexMask{std::move(p), h.total_size};
    default:
      return CompositeMask{RleMask{std::move(s), std::move(e), h.total_size}, IndexMask{std::move(p2), h.total_size}};
  }
}

rq_scalar scal(compute::Scalar k) {
  rq_scalar s{};
  if (std::holds_alternative<double>(k)) {
    s.is_float = 1;
    s.f = std::get<double>(k);
  } else {
    s.i = std::get<int64_t>(k);
  }
  return s;
}

// ---- shapes (compute::Shape ↔ kind, n, s, e, p) ----------------------------------------

compute::Shape shape_down(int32_t kind, int64_t n, rq_arr_t s, rq_arr_t e, rq_arr_t p) {
  Arr S(s), E(e), P(p);
  if (kind == 1) return compute::RunShape{down_pos(S), down_pos(E)};
  if (kind == 2) return compute::PointShape{down_pos(P)};
  return compute::DenseShape{n};
}

struct ShapeUp {
  int32_t kind = 0;
  int64_t n = 0;
  Arr s, e, p;
};
ShapeUp shape_up(const compute::Shape& sh) {
  ShapeUp u;
  u.kind = static_cast<int32_t>(sh.index());
  if (auto* d = std::get_if<compute::DenseShape>(&sh)) u.n = d->n;
  if (auto* r = std::get_if<compute::RunShape>(&sh)) {
    u.s = up(r->s);
    u.e = up(r->e);
  }
  if (auto* q = std::get_if<compute::PointShape>(&sh)) u.p = up(q->p);
  return u;
}

}  // namespace rqa

// =====================================================================================
// runq::compute (align.hpp)
// =====================================================================================

namespace runq::compute {

using namespace rqa;

namespace {
template <class... Ts>
struct overloaded : Ts... {
  using Ts::operator()...;
};
template <class... Ts>
overloaded(Ts...) -> overloaded<Ts...>;
}  // namespace

int64_t shape_slots(const Shape& sh) {
  return std::visit(overloaded{[](const DenseShape& d) { return d.n; },
                               [](const RunShape& r) { return static_cast<int64_t>(r.s.size()); },
                               [](const PointShape& p) { return static_cast<int64_t>(p.p.size()); }},
                    sh);
}

int64_t shape_covered_rows(const Shape& sh) {
  if (auto* r = std::get_if<RunShape>(&sh)) {
    Arr w;
    ShapeUp u = shape_up(sh);
    ck(rq_shape_weights(ctx(), u.kind, u.n, u.s.h, u.e.h, u.p.h, &w.h));
    return kernels::checked_sum(down_pos(w));
  }
  return shape_slots(sh);
}

bool shapes_identical(const Shape& a, const Shape& b) {
  if (a.index() != b.index()) return false;
  return std::visit(overloaded{[&](const DenseShape& d) { return d.n == std::get<DenseShape>(b).n; },
                               [&](const RunShape& r) {
                                 const auto& o = std::get<RunShape>(b);
                                 return r.s == o.s && r.e == o.e;
                               },
                               [&](const PointShape& p) { return p.p == std::get<PointShape>(b).p; }},
                    a);
}

PosVec shape_weights(const Shape& sh) {
  ShapeUp u = shape_up(sh);
  Arr w;
  ck(rq_shape_weights(ctx(), u.kind, u.n, u.s.h, u.e.h, u.p.h, &w.h));
  return down_pos(w);
}

Column column_from_shape(const Shape& sh, Array values, int64_t total_size) {
  return std::visit(overloaded{[&](const DenseShape&) -> Column { return PlainColumn(std::move(values)); },
                               [&](const RunShape& r) -> Column {
                                 return RleColumn{std::move(values), r.s, r.e, total_size};
                               },
                               [&](const PointShape& p) -> Column {
                                 return IndexColumn{std::move(values), p.p, total_size};
                               }},
                    sh);
}

Decomposed decompose(const Column& col) {
  Col c = up(col);
  int32_t kind = 0;
  int64_t n = 0;
  rq_arr_t s = nullptr, e = nullptr, p = nullptr, v = nullptr;
  ck(rq_decompose(ctx(), c.h, &kind, &n, &s, &e, &p, &v));
  Arr V(v);
  return {shape_down(kind, n, s, e, p), down(V)};
}

Column normalize_basic(const Column& col) {
  Col c = up(col);
  Col r;
  ck(rq_normalize_basic(ctx(), c.h, &r.h));
  return down(r);
}

AlignedPair align(const Column& a, const Column& b) {
  Col x = up(a), y = up(b);
  int32_t kind = 0;
  rq_arr_t s = nullptr, e = nullptr, p = nullptr, v1 = nullptr, v2 = nullptr;
  ck(rq_align(ctx(), x.h, y.h, &kind, &s, &e, &p, &v1, &v2));
  Arr V1(v1), V2(v2);
  AlignedPair out;
  out.v1 = down(V1);
  out.v2 = down(V2);
  out.shape = shape_down(kind, out.v1.size(), s, e, p);
  out.total_size = a.total_size();
  return out;
}

MultiAligned align_many(std::span<const Column> cols) {
  std::vector<Col> up_cols;
  std::vector<rq_col_t> hs;
  for (const auto& c : cols) {
    up_cols.push_back(up(c));
    hs.push_back(up_cols.back().h);
  }
  std::vector<rq_arr_t> vals(cols.size(), nullptr);
  int32_t kind = 0;
  int64_t n = 0;
  rq_arr_t s = nullptr, e = nullptr, p = nullptr;
  if (cols.empty()) fail("align_many: no columns");
  ck(rq_align_many(ctx(), hs.data(), static_cast<int32_t>(hs.size()), &kind, &n, &s, &e, &p, vals.data()));
  MultiAligned out;
  out.shape = shape_down(kind, n, s, e, p);
  for (rq_arr_t v : vals) {
    Arr V(v);
    out.values.push_back(down(V));
  }
  out.total_size = cols[0].total_size();
  return out;
}

BinOp binop_from_name(std::string_view name) {
  static const char* names[] = {"+", "-", "*", "/", "<", "<=", "==", "!=", ">=", ">"};
  for (int i = 0; i < 10; ++i)
    if (name == names[i]) return static_cast<BinOp>(i);
  fail("unknown operator: " + std::string(name));
}

std::string_view binop_name(BinOp op) {
  static const char* names[] = {"+", "-", "*", "/", "<", "<=", "==", "!=", ">=", ">"};
  const int i = static_cast<int>(op);
  return (i >= 0 && i < 10) ? names[i] : "?";
}

Column arith(const Column& a, const Column& b, BinOp op) {
  Col x = up(a), y = up(b), r;
  ck(rq_arith(ctx(), x.h, y.h, static_cast<int32_t>(op), &r.h));
  return down(r);
}

MaskColumn compare(const Column& a, const Column& b, BinOp op) {
  Col x = up(a), y = up(b);
  Msk r;
  ck(rq_compare(ctx(), x.h, y.h, static_cast<int32_t>(op), &r.h));
  return down(r);
}

OpResult binary_op(const Column& a, const Column& b, BinOp op) {
  if (is_comparison(op)) return compare(a, b, op);
  return arith(a, b, op);
}

Column arith_scalar(const Column& a, Scalar k, BinOp op, bool reversed) {
  Col x = up(a), r;
  ck(rq_arith_scalar(ctx(), x.h, scal(k), static_cast<int32_t>(op), reversed ? 1 : 0, &r.h));
  return down(r);
}

MaskColumn compare_scalar(const Column& a, Scalar k, BinOp op, bool reversed) {
  Col x = up(a);
  Msk r;
  ck(rq_compare_scalar(ctx(), x.h, scal(k), static_cast<int32_t>(op), reversed ? 1 : 0, &r.h));
  return down(r);
}

OpResult scalar_op(const Column& a, Scalar k, BinOp op, bool reversed) {
  if (is_comparison(op)) return compare_scalar(a, k, op, reversed);
  return arith_scalar(a, k, op, reversed);
}

Column filter(const Column& a, const MaskColumn& m) {
  Col x = up(a), r;
  Msk y = up(m);
  ck(rq_filter(ctx(), x.h, y.h, &r.h));
  return down(r);
}

}  // namespace runq::compute

// =====================================================================================
// runq::enc (primitives.hpp)
// =====================================================================================

namespace runq::enc {

using namespace rqa;

RangeIntersection range_intersect(std::span<const int64_t> s1, std::span<const int64_t> e1,
                                  std::span<const int64_t> s2, std::span<const int64_t> e2) {
  Arr a = up(s1), b = up(e1), c = up(s2), d = up(e2);
  Arr s, e, i1, i2;
  ck(rq_range_intersect(ctx(), a.h, b.h, c.h, d.h, &s.h, &e.h, &i1.h, &i2.h));
  return {down_pos(s), down_pos(e), down_pos(i1), down_pos(i2)};
}

IndexRleIntersection idx_in_rle(std::span<const int64_t> p, std::span<const int64_t> s,
                                std::span<const int64_t> e) {
  Arr a = up(p), b = up(s), c = up(e), po, ro, io;
  ck(rq_idx_in_rle(ctx(), a.h, b.h, c.h, &po.h, &ro.h, &io.h));
  return {down_pos(po), down_pos(ro), down_pos(io)};
}

IndexRleIntersection rle_contain_idx(std::span<const int64_t> p, std::span<const int64_t> s,
                                     std::span<const int64_t> e) {
  Arr a = up(p), b = up(s), c = up(e), po, ro, io;
  ck(rq_rle_contain_idx(ctx(), a.h, b.h, c.h, &po.h, &ro.h, &io.h));
  return {down_pos(po), down_pos(ro), down_pos(io)};
}

IndexIntersection idx_in_idx(std::span<const int64_t> p1, std::span<const int64_t> p2) {
  Arr a = up(p1), b = up(p2), po, i1, i2;
  ck(rq_idx_in_idx(ctx(), a.h, b.h, &po.h, &i1.h, &i2.h));
  return {down_pos(po), down_pos(i1), down_pos(i2)};
}

RangeSet range_union(std::span<const int64_t> s1, std::span<const int64_t> e1, std::span<const int64_t> s2,
                     std::span<const int64_t> e2) {
  Arr a = up(s1), b = up(e1), c = up(s2), d = up(e2), s, e;
  ck(rq_range_union(ctx(), a.h, b.h, c.h, d.h, &s.h, &e.h));
  return {down_pos(s), down_pos(e)};
}

PosVec merge_sorted_idx(std::span<const int64_t> p1, std::span<const int64_t> p2) {
  Arr a = up(p1), b = up(p2), o;
  ck(rq_merge_sorted_idx(ctx(), a.h, b.h, &o.h));
  return down_pos(o);
}

PosVec concat_sort_idx(std::span<const int64_t> p1, std::span<const int64_t> p2) {
  Arr a = up(p1), b = up(p2), o;
  ck(rq_concat_sort_idx(ctx(), a.h, b.h, &o.h));
  return down_pos(o);
}

RangeSet complement_rle(std::span<const int64_t> s, std::span<const int64_t> e, int64_t total) {
  Arr a = up(s), b = up(e), so, eo;
  ck(rq_complement_rle(ctx(), a.h, b.h, total, &so.h, &eo.h));
  return {down_pos(so), down_pos(eo)};
}

RangeSet complement_index(std::span<const int64_t> p, int64_t total) {
  Arr a = up(p), so, eo;
  ck(rq_complement_index(ctx(), a.h, total, &so.h, &eo.h));
  return {down_pos(so), down_pos(eo)};
}

IndexColumn rle_to_index(const RleColumn& c, int64_t budget) {
  Col x = up(Column(c)), r;
  ck(rq_rle_to_index(ctx(), x.h, budget, &r.h));
  return down(r).index();
}

IndexMask rle_to_index(const RleMask& m, int64_t budget) {
  Msk x = up(MaskColumn(m)), r;
  ck(rq_mask_rle_to_index(ctx(), x.h, budget, &r.h));
  return down(r).index();
}

PlainColumn rle_to_plain(const RleColumn& c, double fill, int64_t budget) {
  Col x = up(Column(c)), r;
  ck(rq_rle_to_plain(ctx(), x.h, fill, budget, &r.h));
  return down(r).plain();
}

PlainMask rle_to_plain(const RleMask& m, int64_t budget) {
  Msk x = up(MaskColumn(m)), r;
  ck(rq_mask_rle_to_plain(ctx(), x.h, budget, &r.h));
  return down(r).plain();
}

RleColumn plain_to_rle(const PlainColumn& c) {
  Col x = up(Column(c)), r;
  ck(rq_plain_to_rle(ctx(), x.h, &r.h));
  return down(r).rle();
}

RlePlusIndexColumn plain_to_rle_index(const PlainColumn& c, int64_t min_run) {
  Col x = up(Column(c)), r;
  ck(rq_plain_to_rle_index(ctx(), x.h, min_run, &r.h));
  return down(r).rle_index();
}

PlainPlusIndexColumn plain_to_plain_index(const PlainColumn& c, double trim_fraction) {
  Col x = up(Column(c)), r;
  ck(rq_plain_to_plain_index(ctx(), x.h, trim_fraction, &r.h));
  return down(r).plain_index();
}

RleMask plain_mask_to_rle(const PlainMask& m) {
  Msk x = up(MaskColumn(m)), r;
  ck(rq_plain_mask_to_rle(ctx(), x.h, &r.h));
  return down(r).rle();
}

IndexMask plain_mask_to_index(const PlainMask& m) {
  Msk x = up(MaskColumn(m)), r;
  ck(rq_plain_mask_to_index(ctx(), x.h, &r.h));
  return down(r).index();
}

RleColumn compact_rle(const RleColumn& c) {
  Col x = up(Column(c)), r;
  ck(rq_compact_rle(ctx(), x.h, &r.h));
  return down(r).rle();
}

Column compact_rle_index(const RlePlusIndexColumn& c) {
  Col x = up(Column(c)), r;
  ck(rq_compact_rle_index(ctx(), x.h, &r.h));
  return down(r);
}

}  // namespace runq::enc

// =====================================================================================
// runq::masks (mask_ops.hpp)
// =====================================================================================

namespace runq::masks {

using namespace rqa;

MaskColumn and_mask(const MaskColumn& m1, const MaskColumn& m2) {
  Msk a = up(m1), b = up(m2), r;
  ck(rq_mask_and(ctx(), a.h, b.h, &r.h));
  return down(r);
}

MaskColumn or_mask(const MaskColumn& m1, const MaskColumn& m2) {
  Msk a = up(m1), b = up(m2), r;
  ck(rq_mask_or(ctx(), a.h, b.h, &r.h));
  return down(r);
}

MaskColumn not_mask(const MaskColumn& m) {
  Msk a = up(m), r;
  ck(rq_mask_not(ctx(), a.h, &r.h));
  return down(r);
}

}  // namespace runq::masks

// =====================================================================================
// runq::kernels (kernels.hpp)
// =====================================================================================

namespace runq::kernels {

using namespace rqa;

PosVec bucketize(std::span<const int64_t> x, std::span<const int64_t> boundaries, bool right) {
  Arr a = up(x), b = up(boundaries), o;
  ck(rq_bucketize(ctx(), a.h, b.h, right ? 1 : 0, &o.h));
  return down_pos(o);
}

PosVec cumsum(std::span<const int64_t> x, bool exclusive) {
  Arr a = up(x), o;
  ck(rq_cumsum(ctx(), a.h, exclusive ? 1 : 0, &o.h));
  return down_pos(o);
}

int64_t checked_sum(std::span<const int64_t> x) {
  Arr a = up(x);
  int64_t out = 0;
  ck(rq_checked_sum(ctx(), a.h, &out));
  return out;
}

Array repeat_interleave(const Array& values, std::span<const int64_t> counts) {
  Arr v = up(values), c = up(counts), o;
  ck(rq_repeat_interleave(ctx(), v.h, c.h, &o.h));
  return down(o);
}

PosVec range_arange(std::span<const int64_t> start, std::span<const int64_t> length) {
  Arr a = up(start), b = up(length), o;
  ck(rq_range_arange(ctx(), a.h, b.h, &o.h));
  return down_pos(o);
}

Array scatter_reduce(const Array& values, std::span<const int64_t> index, int64_t n_groups, Reduce op) {
  Arr v = up(values), i = up(index), o;
  ck(rq_scatter_reduce(ctx(), v.h, i.h, n_groups, static_cast<int32_t>(op), &o.h));
  return down(o);
}

UniqueResult unique_with_inverse(std::span<const Array> columns) {
  UniqueResult res;
  if (columns.empty()) return res;
  std::vector<Arr> ups;
  std::vector<rq_arr_t> hs;
  for (const auto& c : columns) {
    ups.push_back(up(c));
    hs.push_back(ups.back().h);
  }
  std::vector<rq_arr_t> keys(columns.size(), nullptr);
  Arr inv;
  ck(rq_unique_with_inverse(ctx(), hs.data(), static_cast<int32_t>(hs.size()), keys.data(), &inv.h, &res.n_groups));
  for (rq_arr_t k : keys) {
    Arr K(k);
    res.keys.push_back(down(K));
  }
  res.inverse = down_pos(inv);
  return res;
}

Array gather(const Array& values, std::span<const int64_t> idx) {
  Arr v = up(values), i = up(idx), o;
  ck(rq_gather(ctx(), v.h, i.h, &o.h));
  return down(o);
}

PosVec gather(std::span<const int64_t> values, std::span<const int64_t> idx) {
  Arr v = up(values), i = up(idx), o;
  ck(rq_gather(ctx(), v.h, i.h, &o.h));
  return down_pos(o);
}

SortResult sort_with_perm(const Array& values) {
  Arr v = up(values), so, pe;
  ck(rq_sort_with_perm(ctx(), v.h, &so.h, &pe.h));
  return {down(so), down_pos(pe)};
}

std::vector<uint8_t> adjacent_ne(const Array& x) {
  Arr v = up(x), o;
  ck(rq_adjacent_ne(ctx(), v.h, &o.h));
  Array a = down(o);
  std::vector<uint8_t> out(static_cast<size_t>(a.size()));
  if (!out.empty()) std::memcpy(out.data(), a.data(), out.size());
  return out;
}

}  // namespace runq::kernels

// =====================================================================================
// runq::agg (groupby.hpp)
// =====================================================================================

namespace runq::agg {

using namespace rqa;

AggFn agg_from_name(std::string_view name) {
  static const char* names[] = {"sum", "count", "min", "max", "avg", "std", "var"};
  for (int i = 0; i < 7; ++i)
    if (name == names[i]) return static_cast<AggFn>(i);
  fail("unknown aggregate function: " + std::string(name));
}

std::string_view agg_name(AggFn fn) {
  static const char* names[] = {"sum", "count", "min", "max", "avg", "std", "var"};
  const int i = static_cast<int>(fn);
  return (i >= 0 && i < 7) ? names[i] : "?";
}

GroupingResult group_on_arrays(compute::Shape shape, std::span<const Array> key_values, int64_t total_size) {
  require(!key_values.empty(), "group: empty key list");
  auto u = kernels::unique_with_inverse(key_values);
  GroupingResult g;
  g.inverse = std::move(u.inverse);
  g.n_groups = u.n_groups;
  g.keys = std::move(u.keys);
  g.shape = std::move(shape);
  g.total_size = total_size;
  return g;
}

GroupingResult group(std::span<const Column> keys) {
  require(!keys.empty(), "group: empty key list");
  std::vector<Col> ups;
  std::vector<rq_col_t> hs;
  for (const auto& k : keys) {
    ups.push_back(up(k));
    hs.push_back(ups.back().h);
  }
  std::vector<rq_arr_t> kout(keys.size(), nullptr);
  int32_t kind = 0;
  int64_t n = 0;
  rq_arr_t s = nullptr, e = nullptr, p = nullptr;
  Arr inv;
  GroupingResult g;
  ck(rq_group(ctx(), hs.data(), static_cast<int32_t>(hs.size()), &kind, &n, &s, &e, &p, &inv.h, kout.data(),
              &g.n_groups));
  g.shape = shape_down(kind, n, s, e, p);
  g.inverse = down_pos(inv);
  for (rq_arr_t k : kout) {
    Arr K(k);
    g.keys.push_back(down(K));
  }
  g.total_size = keys[0].total_size();
  return g;
}

Array aggregate_array(const compute::Shape& shape, const Array& values, const GroupingResult& g, AggFn fn) {
  ShapeUp u = shape_up(shape);
  Arr v = up(values), inv = up(g.inverse), o;
  ck(rq_aggregate_array(ctx(), u.kind, u.n, u.s.h, u.e.h, u.p.h, v.h, inv.h, g.n_groups, static_cast<int32_t>(fn),
                        &o.h));
  return down(o);
}

Array aggregate(const Column& data, const GroupingResult& g, AggFn fn) {
  auto d = compute::decompose(data);
  require(compute::shapes_identical(d.shape, g.shape), "aggregate: data shape differs from grouping shape");
  return aggregate_array(d.shape, d.values, g, fn);
}

GroupAggregateResult group_aggregate(std::span<const Column> keys, std::span<const Column> data,
                                     std::span<const AggFn> fns) {
  require(data.size() == fns.size(), "group_aggregate: data/function count mismatch");
  std::vector<Col> kc, dc;
  std::vector<rq_col_t> kh, dh;
  for (const auto& k : keys) {
    kc.push_back(up(k));
    kh.push_back(kc.back().h);
  }
  for (const auto& d : data) {
    dc.push_back(up(d));
    dh.push_back(dc.back().h);
  }
  std::vector<int32_t> f;
  for (AggFn x : fns) f.push_back(static_cast<int32_t>(x));
  std::vector<rq_arr_t> ko(keys.size(), nullptr), vo(data.size(), nullptr);
  GroupAggregateResult out;
  ck(rq_group_aggregate(ctx(), kh.data(), static_cast<int32_t>(kh.size()), dh.data(), f.data(),
                        static_cast<int32_t>(dh.size()), &out.n_groups, ko.data(), vo.data()));
  for (rq_arr_t k : ko) {
    Arr K(k);
    out.keys.push_back(down(K));
  }
  for (rq_arr_t v : vo) {
    Arr V(v);
    out.values.push_back(down(V));
  }
  return out;
}

Array aggregate_all(const Column& data, AggFn fn) {
  Col c = up(data);
  int32_t t = RQ_I64;
  int64_t i = 0;
  double f = 0;
  ck(rq_aggregate_all(ctx(), c.h, static_cast<int32_t>(fn), &t, &i, &f));
  return t == RQ_F64 ? Array::of<double>({f}) : Array::of<int64_t>({i});
}

}  // namespace runq::agg
