// ops.cpp — host dispatch of the operator API over device columns.
//
// Mirrors the reference's encoding-pair dispatch exactly, because the
// dispatch decides OUTPUT ENCODINGS:
//   compute::align/arith/compare/arith_scalar/compare_scalar/filter
//     (align.cpp:86-771), masks::and_mask (mask_ops.cpp:183-209).
// Every data-touching step is a device kernel (k_*.cu); this file only
// chooses which one and wires the outputs.
#include <cmath>

#include "rq_internal.hpp"

namespace rqb {

namespace {

constexpr double kSparseFraction = 0.05;             // mask_ops.hpp:12
constexpr int64_t kDefaultElementBudget = int64_t{1} << 33;  // primitives.hpp:12

enum ShapeKind { DENSE = 0, RUN = 1, POINT = 2 };

struct Decomposed {
  int kind = DENSE;
  int64_t n = 0;  // dense rows
  DArr s, e, p;
  DArr values;
};

// compute::decompose (align.cpp:86-100)
Decomposed decompose(const CtxPtr& ctx, const DCol& c) {
  Decomposed d;
  switch (c.enc) {
    case RQ_ENC_PLAIN:
      d.kind = DENSE;
      d.n = c.total;
      d.values = decode_plain(ctx, c);
      return d;
    case RQ_ENC_RLE:
      d.kind = RUN;
      d.s = c.s;
      d.e = c.e;
      d.values = c.v;
      return d;
    case RQ_ENC_INDEX:
      d.kind = POINT;
      d.p = c.p;
      d.values = c.v;
      return d;
    case RQ_ENC_PLAIN_INDEX:
      d.kind = DENSE;
      d.n = c.total;
      d.values = decode_plain_index(ctx, c);
      return d;
    case RQ_ENC_RLE_INDEX:
      fail("decompose: rle+index has two positional parts; distribute first");
  }
  fail("decompose: unknown encoding");
}

struct ShapeAlign {
  int kind = DENSE;
  int64_t n = 0;
  DArr s, e, p;
  bool id1 = true, id2 = true;  // identity take
  DArr take1, take2;
};

int64_t slots_of(const ShapeAlign& sa) {
  return sa.kind == DENSE ? sa.n : sa.kind == RUN ? sa.s.n : sa.p.n;
}

// align_run_dense (align.cpp:127-143)
ShapeAlign align_run_dense(const CtxPtr& ctx, const DArr& s, const DArr& e, int64_t n) {
  ShapeAlign out;
  DArr positions, run_idx;
  expand_runs(ctx, s, e, &positions, &run_idx);
  out.id1 = false;
  out.take1 = run_idx;
  if (positions.n == n) {
    out.kind = DENSE;
    out.n = n;
  } else {
    out.kind = POINT;
    out.id2 = false;
    out.take2 = positions;
    out.p = positions;
  }
  return out;
}

ShapeAlign swap_takes(ShapeAlign sa) {
  std::swap(sa.id1, sa.id2);
  std::swap(sa.take1, sa.take2);
  return sa;
}

// align_shapes (align.cpp:145-208)
ShapeAlign align_shapes(const CtxPtr& ctx, const Decomposed& a, const Decomposed& b) {
  ShapeAlign out;
  if (a.kind == DENSE && b.kind == DENSE) {
    out.kind = DENSE;
    out.n = a.n;
    return out;
  }
  if (a.kind == RUN && b.kind == RUN) {
    Intersection r = range_intersect(ctx, a.s, a.e, b.s, b.e, true, true);
    out.kind = RUN;
    out.s = r.s;
    out.e = r.e;
    out.id1 = out.id2 = false;
    out.take1 = r.idx1;
    out.take2 = r.idx2;
    return out;
  }
  if (a.kind == RUN && b.kind == POINT) {
    // idx_in_rle when |p| <= runs else rle_contain_idx: identical outputs
    PointsInRuns r = points_in_runs(ctx, b.p, a.s, a.e, true, true);
    out.kind = POINT;
    out.p = r.p_out;
    out.id1 = out.id2 = false;
    out.take1 = r.run_of;
    out.take2 = r.idx_of;
    return out;
  }
  if (a.kind == POINT && b.kind == RUN) return swap_takes(align_shapes(ctx, b, a));
  if (a.kind == POINT && b.kind == POINT) {
    PointsIntersect r = points_intersect(ctx, a.p, b.p, true, true);
    out.kind = POINT;
    out.p = r.p_out;
    out.id1 = out.id2 = false;
    out.take1 = r.idx1;
    out.take2 = r.idx2;
    return out;
  }
  if (a.kind == RUN && b.kind == DENSE) return align_run_dense(ctx, a.s, a.e, b.n);
  if (a.kind == DENSE && b.kind == RUN) return swap_takes(align_run_dense(ctx, b.s, b.e, a.n));
  if (a.kind == POINT && b.kind == DENSE) {
    out.kind = POINT;
    out.p = a.p;
    out.id2 = false;
    out.take2 = a.p;
    return out;
  }
  return swap_takes(align_shapes(ctx, b, a));  // Dense x Point
}

DArr take(const CtxPtr& ctx, const DArr& v, bool identity, const DArr& idx, int64_t slots) {
  if (identity && v.n == slots) return v;
  if (identity) return copy_prefix(ctx, v, 0);
  return gather(ctx, v, idx);
}

DCol column_from_shape(int kind, const DArr& s, const DArr& e, const DArr& p, DArr values,
                       int64_t total) {  // align.cpp:72-84
  DCol c;
  c.total = total;
  c.v = std::move(values);
  c.logical = c.v.dt;
  if (kind == DENSE) {
    c.enc = RQ_ENC_PLAIN;
    c.total = c.v.n;
  } else if (kind == RUN) {
    c.enc = RQ_ENC_RLE;
    c.s = s;
    c.e = e;
  } else {
    c.enc = RQ_ENC_INDEX;
    c.p = p;
  }
  return c;
}

DMask mask_from_shape(const CtxPtr& ctx, const Aligned& ap, const DArr& flags) {  // :352-381
  DMask m;
  m.total = ap.total;
  if (ap.kind == DENSE) {
    m.enc = RQ_MASK_PLAIN;
    m.bits = flags;
    m.total = flags.n;
  } else if (ap.kind == RUN) {
    m.enc = RQ_MASK_RLE;
    select_runs(ctx, flags, ap.s, ap.e, m.s, m.e);
  } else {
    m.enc = RQ_MASK_INDEX;
    select_points(ctx, flags, ap.p, m.p, nullptr);
  }
  return m;
}

DCol rle_part(const DCol& c) {
  DCol r;
  r.enc = RQ_ENC_RLE;
  r.total = c.total;
  r.v = c.v;
  r.logical = c.v.dt;
  r.s = c.s;
  r.e = c.e;
  return r;
}

DCol index_part(const DCol& c) {
  DCol r;
  r.enc = RQ_ENC_INDEX;
  r.total = c.total;
  r.v = c.v2;
  r.logical = c.v2.dt;
  r.p = c.p2;
  return r;
}

DCol empty_index(int64_t total, int32_t dt) {
  DCol r;
  r.enc = RQ_ENC_INDEX;
  r.total = total;
  r.v.dt = dt;
  r.logical = dt;
  return r;
}

// combine_disjoint (align.cpp:446-483)
DCol combine_disjoint(const CtxPtr& ctx, const DCol& a, const DCol& b) {
  require(a.enc != RQ_ENC_PLAIN && b.enc != RQ_ENC_PLAIN,
          "combine_disjoint: plain parts cannot carry gaps");
  const int64_t total = a.total;
  auto parts = [](const DCol& c, const DCol*& runs, const DCol*& pts, DCol& rbuf, DCol& pbuf) {
    runs = nullptr;
    pts = nullptr;
    if (c.enc == RQ_ENC_RLE) runs = &c;
    else if (c.enc == RQ_ENC_INDEX) pts = &c;
    else if (c.enc == RQ_ENC_RLE_INDEX) {
      rbuf = rle_part(c);
      pbuf = index_part(c);
      runs = &rbuf;
      pts = &pbuf;
    }
  };
  const DCol *ra, *pa, *rb, *pb;
  DCol rbuf_a, pbuf_a, rbuf_b, pbuf_b;
  parts(a, ra, pa, rbuf_a, pbuf_a);
  parts(b, rb, pb, rbuf_b, pbuf_b);

  bool have_runs_obj = ra || rb;
  DCol runs;
  if (ra && rb) {
    // merge_disjoint_runs: b's values cast to a's dtype
    DArr vb = cast_values(ctx, rb->v, ra->v.dt);
    runs.enc = RQ_ENC_RLE;
    runs.total = ra->total;
    merge_disjoint(ctx, ra->s, &ra->e, &ra->v, rb->s, &rb->e, &vb, runs.s, &runs.e, &runs.v);
    runs.logical = runs.v.dt;
  } else if (ra) {
    runs = *ra;
  } else if (rb) {
    runs = *rb;
  }
  DCol pts;
  bool have_pts_obj = pa || pb;
  if (pa && pb) {
    DArr vb = cast_values(ctx, pb->v, pa->v.dt);
    pts.enc = RQ_ENC_INDEX;
    pts.total = pa->total;
    merge_disjoint(ctx, pa->p, nullptr, &pa->v, pb->p, nullptr, &vb, pts.p, nullptr, &pts.v);
    pts.logical = pts.v.dt;
  } else if (pa) {
    pts = *pa;
  } else if (pb) {
    pts = *pb;
  }
  const bool have_runs = have_runs_obj && runs.s.n > 0;
  const bool have_pts = have_pts_obj && pts.p.n > 0;
  if (have_runs && have_pts) {
    DCol c;
    c.enc = RQ_ENC_RLE_INDEX;
    c.total = runs.total;
    c.v = runs.v;
    c.logical = runs.v.dt;
    c.s = runs.s;
    c.e = runs.e;
    c.v2 = pts.v;
    c.p2 = pts.p;
    return c;
  }
  if (have_runs) return runs;
  if (have_pts) return pts;
  if (have_runs_obj) return runs;  // empty, keep a consistent carrier
  return empty_index(total, a.value_type());
}

DMask rle_mask_part(const DMask& m) {
  DMask r;
  r.enc = RQ_MASK_RLE;
  r.total = m.total;
  r.s = m.s;
  r.e = m.e;
  return r;
}
DMask index_mask_part(const DMask& m) {
  DMask r;
  r.enc = RQ_MASK_INDEX;
  r.total = m.total;
  r.p = m.p;
  return r;
}

// combine_disjoint_masks (align.cpp:485-489)
DMask combine_disjoint_masks(const CtxPtr& ctx, const DMask& a, const DMask& b) {
  if (a.enc == RQ_MASK_RLE && b.enc == RQ_MASK_INDEX) {
    DMask c;
    c.enc = RQ_MASK_COMPOSITE;
    c.total = a.total;
    c.s = a.s;
    c.e = a.e;
    c.p = b.p;
    return c;
  }
  return mask_or(ctx, a, b);
}

// enc::rle_to_index for masks (primitives.cpp:181-190), budget-checked
DArr rle_mask_positions(const CtxPtr& ctx, const DArr& s, const DArr& e) {
  const int64_t rows = covered_rows(ctx, s, e);
  if (rows > kDefaultElementBudget)
    fail("rle_to_index: expansion of " + std::to_string(rows) + " elements exceeds budget " +
             std::to_string(kDefaultElementBudget),
         RQ_RESOURCE);
  DArr pos;
  expand_runs(ctx, s, e, &pos, nullptr);
  return pos;
}

// enc::rle_to_plain for masks (primitives.cpp:207-213)
DArr rle_mask_bits(const CtxPtr& ctx, const DArr& s, const DArr& e, int64_t total) {
  if (total > kDefaultElementBudget)
    fail("rle_to_plain: expansion of " + std::to_string(total) + " elements exceeds budget",
         RQ_RESOURCE);
  DArr bits = zeros_bytes(ctx, total);
  DArr pos;
  expand_runs(ctx, s, e, &pos, nullptr);
  set_bits(ctx, bits, pos);
  return bits;
}

bool rle_mask_sparse(const CtxPtr& ctx, const DMask& m) {  // mask_ops.cpp:13-17
  if (m.total == 0) return false;
  return static_cast<double>(covered_rows(ctx, m.s, m.e)) < kSparseFraction * static_cast<double>(m.total);
}

// Index columns sharing one position buffer (e.g. plain columns filtered
// with the same mask) have identical coverage by construction.
bool same_points(const DCol& a, const DCol& b) {
  return a.enc == RQ_ENC_INDEX && b.enc == RQ_ENC_INDEX && a.p.buf && a.p.buf == b.p.buf && a.p.n == b.p.n;
}

DMask make_index_mask(DArr p, int64_t total) {
  DMask m;
  m.enc = RQ_MASK_INDEX;
  m.total = total;
  m.p = std::move(p);
  return m;
}
DMask make_plain_mask(DArr bits) {
  DMask m;
  m.enc = RQ_MASK_PLAIN;
  m.total = bits.n;
  m.bits = std::move(bits);
  return m;
}
DMask make_rle_mask(DArr s, DArr e, int64_t total) {
  DMask m;
  m.enc = RQ_MASK_RLE;
  m.total = total;
  m.s = std::move(s);
  m.e = std::move(e);
  return m;
}

// and_plain_index (mask_ops.cpp:43-49): keep positions whose bit is set
DMask and_plain_index(const CtxPtr& ctx, const DMask& plain, const DMask& idx) {
  DArr flags = gather(ctx, plain.bits, idx.p);
  DMask out;
  out.enc = RQ_MASK_INDEX;
  out.total = idx.total;
  select_points(ctx, flags, idx.p, out.p, nullptr);
  return out;
}

DMask and_rle_index(const CtxPtr& ctx, const DMask& rle, const DMask& idx) {  // :26-34
  PointsInRuns r = points_in_runs(ctx, idx.p, rle.s, rle.e, false, false);
  return make_index_mask(r.p_out, idx.total);
}

DMask and_index_index(const CtxPtr& ctx, const DMask& a, const DMask& b) {  // :51-57
  PointsIntersect r = points_intersect(ctx, a.p, b.p, false, false);
  return make_index_mask(r.p_out, a.total);
}

DMask and_rle_rle(const CtxPtr& ctx, const DMask& a, const DMask& b) {  // :21-24
  Intersection r = range_intersect(ctx, a.s, a.e, b.s, b.e, false, false);
  return make_rle_mask(r.s, r.e, a.total);
}

DMask and_rle_plain(const CtxPtr& ctx, const DMask& rle, const DMask& plain) {  // :59-62
  if (rle_mask_sparse(ctx, rle))
    return and_plain_index(ctx, plain, make_index_mask(rle_mask_positions(ctx, rle.s, rle.e), rle.total));
  return make_plain_mask(bytes_and(ctx, rle_mask_bits(ctx, rle.s, rle.e, rle.total), plain.bits));
}

DMask or_index_index(const CtxPtr& ctx, const DMask& a, const DMask& b) {  // :81-91
  return make_index_mask(union_points(ctx, a.p, b.p), a.total);
}

DMask or_plain_index(const CtxPtr& ctx, const DMask& plain, const DMask& idx) {  // :75-79
  DArr bits = bytes_copy01(ctx, plain.bits);
  set_bits(ctx, bits, idx.p);
  return make_plain_mask(bits);
}

// and_composite (mask_ops.cpp:147-158)
DMask and_composite(const CtxPtr& ctx, const DMask& a, const DMask& b) {
  auto parts = [](const DMask& m, DMask& runs, DMask& pts) {
    if (m.enc == RQ_MASK_RLE) {
      runs = m;
      pts = make_index_mask(DArr{}, m.total);
    } else if (m.enc == RQ_MASK_INDEX) {
      runs = make_rle_mask(DArr{}, DArr{}, m.total);
      pts = m;
    } else if (m.enc == RQ_MASK_COMPOSITE) {
      runs = rle_mask_part(m);
      pts = index_mask_part(m);
    } else {
      fail("as_parts: plain mask has no positional parts");
    }
  };
  DMask ra, pa, rb, pb;
  parts(a, ra, pa);
  parts(b, rb, pb);
  DMask rr = and_rle_rle(ctx, ra, rb);
  DMask rp = and_rle_index(ctx, ra, pb);
  DMask pr = and_rle_index(ctx, rb, pa);
  DMask pp = and_index_index(ctx, pa, pb);
  DMask pts = or_index_index(ctx, or_index_index(ctx, rp, pr), pp);
  DMask c;
  c.enc = RQ_MASK_COMPOSITE;
  c.total = rr.total;
  c.s = rr.s;
  c.e = rr.e;
  c.p = pts.p;
  return c;
}

// and_composite_plain (mask_ops.cpp:168-175)
DMask and_composite_plain(const CtxPtr& ctx, const DMask& c, const DMask& plain) {
  DMask run_part = and_rle_plain(ctx, rle_mask_part(c), plain);
  DMask pt_part = and_plain_index(ctx, plain, index_mask_part(c));
  if (run_part.enc == RQ_MASK_PLAIN) return or_plain_index(ctx, run_part, pt_part);
  return or_index_index(ctx, run_part, pt_part);
}

}  // namespace

bool col_gapless(const CtxPtr& ctx, const DCol& c) {
  if (c.enc != RQ_ENC_RLE) return false;
  if (c.gapless < 0) c.gapless = runs_gapless(ctx, c.s, c.e, c.total) ? 1 : 0;
  return c.gapless == 1;
}

int64_t mask_true_count(const CtxPtr& ctx, const DMask& m) {  // column.cpp:112-128
  if (m.true_count >= 0) return m.true_count;
  int64_t n = 0;
  switch (m.enc) {
    case RQ_MASK_PLAIN: n = count_nonzero(ctx, m.bits); break;
    case RQ_MASK_RLE: n = covered_rows(ctx, m.s, m.e); break;
    case RQ_MASK_INDEX: n = m.p.n; break;
    default: n = covered_rows(ctx, m.s, m.e) + m.p.n;
  }
  m.true_count = n;
  return n;
}

Aligned align(const CtxPtr& ctx, const DCol& a, const DCol& b) {  // align.cpp:219-231
  require(a.total == b.total, "align: total_size mismatch");
  Decomposed da = decompose(ctx, a);
  Decomposed db = decompose(ctx, b);
  ShapeAlign sa = align_shapes(ctx, da, db);
  const int64_t slots = slots_of(sa);
  Aligned out;
  out.v1 = take(ctx, da.values, sa.id1, sa.take1, slots);
  out.v2 = take(ctx, db.values, sa.id2, sa.take2, slots);
  out.kind = sa.kind;
  out.s = sa.s;
  out.e = sa.e;
  out.p = sa.p;
  out.total = a.total;
  return out;
}

DCol arith(const CtxPtr& ctx, const DCol& a, const DCol& b, int op) {  // align.cpp:495-508
  require(op >= RQ_ADD && op <= RQ_DIV, "arith: comparison operator");
  if (a.enc == RQ_ENC_RLE_INDEX)
    return combine_disjoint(ctx, arith(ctx, rle_part(a), b, op), arith(ctx, index_part(a), b, op));
  if (b.enc == RQ_ENC_RLE_INDEX)
    return combine_disjoint(ctx, arith(ctx, a, rle_part(b), op), arith(ctx, a, index_part(b), op));
  if (same_points(a, b)) {
    // identical position list (one shared buffer): idx_in_idx would return
    // p itself with identity take indices, so align reduces to elementwise
    require(a.total == b.total, "align: total_size mismatch");
    return column_from_shape(POINT, {}, {}, a.p, arith_values(ctx, a.v, b.v, op), a.total);
  }
  Aligned ap = align(ctx, a, b);
  DArr vals = arith_values(ctx, ap.v1, ap.v2, op);
  return column_from_shape(ap.kind, ap.s, ap.e, ap.p, vals, ap.total);
}

DMask compare(const CtxPtr& ctx, const DCol& a, const DCol& b, int op) {  // align.cpp:510-523
  require(op >= RQ_LT && op <= RQ_GT, "compare: arithmetic operator");
  if (a.enc == RQ_ENC_RLE_INDEX)
    return combine_disjoint_masks(ctx, compare(ctx, rle_part(a), b, op),
                                  compare(ctx, index_part(a), b, op));
  if (b.enc == RQ_ENC_RLE_INDEX)
    return combine_disjoint_masks(ctx, compare(ctx, a, rle_part(b), op),
                                  compare(ctx, a, index_part(b), op));
  Aligned ap = align(ctx, a, b);
  DArr flags = cmp_values(ctx, ap.v1, ap.v2, op);
  return mask_from_shape(ctx, ap, flags);
}

DCol arith_scalar(const CtxPtr& ctx, const DCol& a, Scalar k, int op, bool reversed) {  // :571-596
  require(op >= RQ_ADD && op <= RQ_DIV, "apply_arith: not an arithmetic op");
  switch (a.enc) {
    case RQ_ENC_PLAIN: {
      DArr vals = scalar_arith_values(ctx, decode_plain(ctx, a), k, op, reversed);
      return column_from_shape(DENSE, {}, {}, {}, vals, a.total);
    }
    case RQ_ENC_RLE: {
      DCol c = a;
      c.v = scalar_arith_values(ctx, a.v, k, op, reversed);
      c.logical = c.v.dt;
      return c;
    }
    case RQ_ENC_INDEX: {
      DCol c = a;
      c.v = scalar_arith_values(ctx, a.v, k, op, reversed);
      c.logical = c.v.dt;
      return c;
    }
    case RQ_ENC_PLAIN_INDEX: {
      DArr vals = scalar_arith_values(ctx, decode_plain_index(ctx, a), k, op, reversed);
      return column_from_shape(DENSE, {}, {}, {}, vals, a.total);
    }
    case RQ_ENC_RLE_INDEX:
      return combine_disjoint(ctx, arith_scalar(ctx, rle_part(a), k, op, reversed),
                              arith_scalar(ctx, index_part(a), k, op, reversed));
  }
  fail("arith_scalar: unknown encoding");
}

DMask compare_scalar(const CtxPtr& ctx, const DCol& a, Scalar k, int op, bool reversed) {  // :598-652
  require(op >= RQ_LT && op <= RQ_GT, "apply_cmp: not a comparison");
  switch (a.enc) {
    case RQ_ENC_PLAIN:
      return make_plain_mask(plain_cmp_scalar(ctx, a, k, op, reversed));
    case RQ_ENC_RLE: {
      DMask m;
      m.enc = RQ_MASK_RLE;
      m.total = a.total;
      rle_cmp_scalar_select(ctx, a.v, a.s, a.e, k, op, reversed, m.s, m.e);
      return m;
    }
    case RQ_ENC_INDEX: {
      DMask m;
      m.enc = RQ_MASK_INDEX;
      m.total = a.total;
      index_cmp_scalar_select(ctx, a.v, a.p, k, op, reversed, m.p);
      return m;
    }
    case RQ_ENC_PLAIN_INDEX: {
      // compare the narrow base, then outlier slots take the outliers' flags
      DCol base = a;
      base.enc = RQ_ENC_PLAIN;
      DArr bits = plain_cmp_scalar(ctx, base, k, op, reversed);
      DArr oflags = scalar_cmp_values(ctx, a.v2, k, op, reversed);
      scatter_flags(ctx, bits, a.p2, oflags);
      return make_plain_mask(bits);
    }
    case RQ_ENC_RLE_INDEX:
      return combine_disjoint_masks(ctx, compare_scalar(ctx, rle_part(a), k, op, reversed),
                                    compare_scalar(ctx, index_part(a), k, op, reversed));
  }
  fail("compare_scalar: unknown encoding");
}

namespace {

DCol filter_rle(const CtxPtr& ctx, const DCol& c, const DMask& m);
DCol filter_index(const CtxPtr& ctx, const DCol& c, const DMask& m);
DCol filter_plain(const CtxPtr& ctx, const DCol& c, const DMask& m);

DCol filter_rle(const CtxPtr& ctx, const DCol& c, const DMask& m) {  // align.cpp:667-696
  switch (m.enc) {
    case RQ_MASK_RLE: {
      Intersection r = range_intersect(ctx, c.s, c.e, m.s, m.e, true, false);
      DCol out;
      out.enc = RQ_ENC_RLE;
      out.total = c.total;
      out.v = gather(ctx, c.v, r.idx1);
      out.logical = out.v.dt;
      out.s = r.s;
      out.e = r.e;
      return out;
    }
    case RQ_MASK_INDEX: {
      PointsInRuns r = points_in_runs(ctx, m.p, c.s, c.e, true, false);
      DCol out;
      out.enc = RQ_ENC_INDEX;
      out.total = c.total;
      out.v = gather(ctx, c.v, r.run_of);
      out.logical = out.v.dt;
      out.p = r.p_out;
      return out;
    }
    case RQ_MASK_PLAIN: {
      const int64_t threshold = static_cast<int64_t>(kSparseFraction * static_cast<double>(m.bits.n));
      if (mask_true_count(ctx, m) < threshold)
        return filter_rle(ctx, c, make_index_mask(plain_mask_to_index(ctx, m.bits), m.total));
      DArr s, e;
      plain_mask_to_rle(ctx, m.bits, s, e);
      return filter_rle(ctx, c, make_rle_mask(s, e, m.total));
    }
    default:
      return combine_disjoint(ctx, filter_rle(ctx, c, rle_mask_part(m)),
                              filter_rle(ctx, c, index_mask_part(m)));
  }
}

DCol filter_index(const CtxPtr& ctx, const DCol& c, const DMask& m) {  // align.cpp:698-731
  switch (m.enc) {
    case RQ_MASK_RLE: {
      PointsInRuns r = points_in_runs(ctx, c.p, m.s, m.e, false, true);
      DCol out;
      out.enc = RQ_ENC_INDEX;
      out.total = c.total;
      out.v = gather(ctx, c.v, r.idx_of);
      out.logical = out.v.dt;
      out.p = r.p_out;
      return out;
    }
    case RQ_MASK_INDEX: {
      PointsIntersect r = points_intersect(ctx, c.p, m.p, true, false);
      DCol out;
      out.enc = RQ_ENC_INDEX;
      out.total = c.total;
      out.v = gather(ctx, c.v, r.idx1);
      out.logical = out.v.dt;
      out.p = r.p_out;
      return out;
    }
    case RQ_MASK_PLAIN: {
      DArr flags = gather(ctx, m.bits, c.p);
      DCol out;
      out.enc = RQ_ENC_INDEX;
      out.total = c.total;
      DArr keep;
      select_points(ctx, flags, c.p, out.p, &keep);
      out.v = gather(ctx, c.v, keep);
      out.logical = out.v.dt;
      return out;
    }
    default:
      return combine_disjoint(ctx, filter_index(ctx, c, rle_mask_part(m)),
                              filter_index(ctx, c, index_mask_part(m)));
  }
}

DCol filter_plain(const CtxPtr& ctx, const DCol& c, const DMask& m) {  // align.cpp:733-751
  auto take_pos = [&](const DArr& pos) {
    // gather the storage first, decode only the survivors
    DCol g = c;
    g.v = gather(ctx, c.v, pos);
    DCol out;
    out.enc = RQ_ENC_INDEX;
    out.total = c.total;
    out.v = decode_plain(ctx, g);
    out.logical = out.v.dt;
    out.p = pos;
    return out;
  };
  switch (m.enc) {
    case RQ_MASK_RLE:
      if (!m.positions) m.positions = std::make_shared<DArr>(rle_mask_positions(ctx, m.s, m.e));
      return take_pos(*m.positions);
    case RQ_MASK_INDEX: return take_pos(m.p);
    case RQ_MASK_PLAIN: return take_pos(plain_mask_to_index(ctx, m.bits));
    default:
      return combine_disjoint(ctx, filter_plain(ctx, c, rle_mask_part(m)),
                              filter_plain(ctx, c, index_mask_part(m)));
  }
}

}  // namespace

DCol filter(const CtxPtr& ctx, const DCol& a, const DMask& m) {  // align.cpp:755-771
  require(a.total == m.total, "filter: total_size mismatch");
  if (mask_true_count(ctx, m) == m.total) return a;  // full cover selects everything
  switch (a.enc) {
    case RQ_ENC_PLAIN: return filter_plain(ctx, a, m);
    case RQ_ENC_RLE: return filter_rle(ctx, a, m);
    case RQ_ENC_INDEX: return filter_index(ctx, a, m);
    case RQ_ENC_PLAIN_INDEX: {
      // Reference: filter_plain(PlainColumn(decode_values(a)), m) — decodes
      // every row first. Same result with the decode restricted to the
      // selected rows: gather the narrow base at the selected positions,
      // decode, then overlay the outliers that fall on selected positions.
      if (m.enc == RQ_MASK_COMPOSITE) {
        DCol dec;
        dec.enc = RQ_ENC_PLAIN;
        dec.v = decode_plain_index(ctx, a);
        dec.logical = dec.v.dt;
        dec.total = dec.v.n;
        return filter_plain(ctx, dec, m);
      }
      DArr pos;
      if (m.enc == RQ_MASK_RLE) {
        if (!m.positions) m.positions = std::make_shared<DArr>(rle_mask_positions(ctx, m.s, m.e));
        pos = *m.positions;
      } else if (m.enc == RQ_MASK_INDEX) {
        pos = m.p;
      } else {
        pos = plain_mask_to_index(ctx, m.bits);
      }
      DCol base = a;
      base.enc = RQ_ENC_PLAIN;
      base.v = gather(ctx, a.v, pos);
      DArr vals = cast_values(ctx, decode_plain(ctx, base), a.v2.dt);
      if (vals.buf == base.v.buf) vals = copy_prefix(ctx, vals, vals.n);
      PointsIntersect hit = points_intersect(ctx, a.p2, pos, true, true);
      if (hit.p_out.n > 0) {
        DArr ov = gather(ctx, a.v2, hit.idx1);
        scatter_values(ctx, vals, hit.idx2, ov);
      }
      DCol out;
      out.enc = RQ_ENC_INDEX;
      out.total = a.total;
      out.v = vals;
      out.logical = vals.dt;
      out.p = pos;
      return out;
    }
    case RQ_ENC_RLE_INDEX:
      return combine_disjoint(ctx, filter(ctx, rle_part(a), m), filter(ctx, index_part(a), m));
  }
  fail("filter: unknown encoding");
}

DMask mask_and(const CtxPtr& ctx, const DMask& m1, const DMask& m2) {  // mask_ops.cpp:183-209
  require(m1.total == m2.total, "and_mask: total_size mismatch");
  const int e1 = m1.enc, e2 = m2.enc;
  if (e1 == RQ_MASK_COMPOSITE || e2 == RQ_MASK_COMPOSITE) {
    if (e1 == RQ_MASK_PLAIN) return and_composite_plain(ctx, m2, m1);
    if (e2 == RQ_MASK_PLAIN) return and_composite_plain(ctx, m1, m2);
    return and_composite(ctx, m1, m2);
  }
  if (e1 == RQ_MASK_RLE && e2 == RQ_MASK_RLE) return and_rle_rle(ctx, m1, m2);
  if (e1 == RQ_MASK_RLE && e2 == RQ_MASK_PLAIN) return and_rle_plain(ctx, m1, m2);
  if (e1 == RQ_MASK_PLAIN && e2 == RQ_MASK_RLE) return and_rle_plain(ctx, m2, m1);
  if (e1 == RQ_MASK_RLE && e2 == RQ_MASK_INDEX) return and_rle_index(ctx, m1, m2);
  if (e1 == RQ_MASK_INDEX && e2 == RQ_MASK_RLE) return and_rle_index(ctx, m2, m1);
  if (e1 == RQ_MASK_PLAIN && e2 == RQ_MASK_PLAIN)
    return make_plain_mask(bytes_and(ctx, m1.bits, m2.bits));
  if (e1 == RQ_MASK_PLAIN && e2 == RQ_MASK_INDEX) return and_plain_index(ctx, m1, m2);
  if (e1 == RQ_MASK_INDEX && e2 == RQ_MASK_PLAIN) return and_plain_index(ctx, m2, m1);
  return and_index_index(ctx, m1, m2);
}

namespace {

DMask or_rle_rle(const CtxPtr& ctx, const DMask& a, const DMask& b) {  // mask_ops.cpp:66-69
  // range_union (primitives.cpp:102-123): merge starts and ends separately
  DArr S = merge_keys(ctx, a.s, b.s);
  DArr E = merge_keys(ctx, a.e, b.e);
  DMask m = make_rle_mask(DArr{}, DArr{}, a.total);
  if (S.n) union_from_merged(ctx, S, E, m.s, m.e);
  return m;
}

DMask or_rle_plain(const CtxPtr& ctx, const DMask& rle, const DMask& plain) {  // :93-96
  if (rle_mask_sparse(ctx, rle))
    return or_plain_index(ctx, plain, make_index_mask(rle_mask_positions(ctx, rle.s, rle.e), rle.total));
  return make_plain_mask(bytes_or(ctx, rle_mask_bits(ctx, rle.s, rle.e, rle.total), plain.bits));
}

// points of idx not covered by rle; keeps composite parts disjoint (:98-111)
DMask subtract_runs(const CtxPtr& ctx, const DMask& idx, const DMask& rle) {
  return make_index_mask(points_not_in_runs(ctx, idx.p, rle.s, rle.e), idx.total);
}

DMask composite_of(DMask runs, DMask pts) {
  DMask c;
  c.enc = RQ_MASK_COMPOSITE;
  c.total = runs.total;
  c.s = runs.s;
  c.e = runs.e;
  c.p = pts.p;
  return c;
}

void mask_parts(const DMask& m, DMask& runs, DMask& pts) {  // as_parts (:120-133)
  if (m.enc == RQ_MASK_RLE) {
    runs = m;
    pts = make_index_mask(DArr{}, m.total);
  } else if (m.enc == RQ_MASK_INDEX) {
    runs = make_rle_mask(DArr{}, DArr{}, m.total);
    pts = m;
  } else if (m.enc == RQ_MASK_COMPOSITE) {
    runs = rle_mask_part(m);
    pts = index_mask_part(m);
  } else {
    fail("as_parts: plain mask has no positional parts");
  }
}

DMask or_composite(const CtxPtr& ctx, const DMask& a, const DMask& b) {  // :160-165
  DMask ra, pa, rb, pb;
  mask_parts(a, ra, pa);
  mask_parts(b, rb, pb);
  DMask runs = or_rle_rle(ctx, ra, rb);
  DMask pts = subtract_runs(ctx, or_index_index(ctx, pa, pb), runs);
  return composite_of(runs, pts);
}

DMask or_composite_plain(const CtxPtr& ctx, const DMask& c, const DMask& plain) {  // :177-180
  DMask with_runs = or_rle_plain(ctx, rle_mask_part(c), plain);
  return or_plain_index(ctx, with_runs, index_mask_part(c));
}

}  // namespace

DMask mask_or(const CtxPtr& ctx, const DMask& m1, const DMask& m2) {  // mask_ops.cpp:211-237
  require(m1.total == m2.total, "or_mask: total_size mismatch");
  const int e1 = m1.enc, e2 = m2.enc;
  if (e1 == RQ_MASK_COMPOSITE || e2 == RQ_MASK_COMPOSITE) {
    if (e1 == RQ_MASK_PLAIN) return or_composite_plain(ctx, m2, m1);
    if (e2 == RQ_MASK_PLAIN) return or_composite_plain(ctx, m1, m2);
    return or_composite(ctx, m1, m2);
  }
  if (e1 == RQ_MASK_RLE && e2 == RQ_MASK_RLE) return or_rle_rle(ctx, m1, m2);
  if (e1 == RQ_MASK_RLE && e2 == RQ_MASK_PLAIN) return or_rle_plain(ctx, m1, m2);
  if (e1 == RQ_MASK_PLAIN && e2 == RQ_MASK_RLE) return or_rle_plain(ctx, m2, m1);
  if (e1 == RQ_MASK_RLE && e2 == RQ_MASK_INDEX) return composite_of(m1, subtract_runs(ctx, m2, m1));
  if (e1 == RQ_MASK_INDEX && e2 == RQ_MASK_RLE) return composite_of(m2, subtract_runs(ctx, m1, m2));
  if (e1 == RQ_MASK_PLAIN && e2 == RQ_MASK_PLAIN)
    return make_plain_mask(bytes_or(ctx, m1.bits, m2.bits));
  if (e1 == RQ_MASK_PLAIN && e2 == RQ_MASK_INDEX) return or_plain_index(ctx, m1, m2);
  if (e1 == RQ_MASK_INDEX && e2 == RQ_MASK_PLAIN) return or_plain_index(ctx, m2, m1);
  return or_index_index(ctx, m1, m2);
}

DMask mask_not(const CtxPtr& ctx, const DMask& m) {  // mask_ops.cpp:239-265
  switch (m.enc) {
    case RQ_MASK_PLAIN:
      return make_plain_mask(bytes_not(ctx, m.bits));
    case RQ_MASK_RLE: {
      DMask r = make_rle_mask(DArr{}, DArr{}, m.total);
      complement_runs(ctx, m.s, m.e, m.total, r.s, r.e);
      return r;
    }
    case RQ_MASK_INDEX: {
      DMask r = make_rle_mask(DArr{}, DArr{}, m.total);
      complement_runs(ctx, m.p, m.p, m.total, r.s, r.e);
      return r;
    }
    default: {
      // ~(runs | points) = ~runs & ~points; both complements are RLE
      DArr rs, re, ps, pe;
      complement_runs(ctx, m.s, m.e, m.total, rs, re);
      complement_runs(ctx, m.p, m.p, m.total, ps, pe);
      Intersection r = range_intersect(ctx, rs, re, ps, pe, false, false);
      return make_rle_mask(r.s, r.e, m.total);
    }
  }
}

DCol normalize_basic(const CtxPtr& ctx, const DCol& c) {  // align.cpp:102-115
  if (c.enc == RQ_ENC_PLAIN_INDEX) {
    DCol out;
    out.enc = RQ_ENC_PLAIN;
    out.v = decode_plain_index(ctx, c);
    out.logical = out.v.dt;
    out.total = out.v.n;
    return out;
  }
  if (c.enc == RQ_ENC_RLE_INDEX) {
    // to_rows (column.cpp:331-376): expand runs, merge with the points
    require(c.v.dt == c.v2.dt, "array dtype mismatch");
    DArr rpos, ridx;
    expand_runs(ctx, c.s, c.e, &rpos, &ridx);
    DArr rv = gather(ctx, c.v, ridx);
    DArr pos, vals;
    merge_disjoint(ctx, rpos, nullptr, &rv, c.p2, nullptr, &c.v2, pos, nullptr, &vals);
    if (pos.n == c.total) {
      DCol out;
      out.enc = RQ_ENC_PLAIN;
      out.v = vals;
      out.logical = vals.dt;
      out.total = vals.n;
      return out;
    }
    DCol out;
    out.enc = RQ_ENC_INDEX;
    out.total = c.total;
    out.v = vals;
    out.logical = vals.dt;
    out.p = pos;
    return out;
  }
  return c;
}

}  // namespace rqb
