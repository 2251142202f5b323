// k_fused.cu — single-pass filtered aggregate (the C2 query shape).
//
// The reference evaluates
//   m  = compare_scalar(C, k, cmp)                 (align.cpp:598-652)
//   A' = filter(A, m); B' = filter(B, m)           (align.cpp:755-771)
//   aggregate_all(arith(A', B', op), fn)           (align.cpp:495-508, groupby.cpp:164-172)
// materialising the mask, two filtered columns and the product. With A RLE
// and B Index, every surviving slot is a point p of B with C(p) passing and
// A covering p, so the whole chain is
//   Σ_{p ∈ B, pred(C(p)), p ∈ cover(A)} op(A(p), B(p))
// and one merge-path walk over (B points, A run ends) computes it. C's runs
// overlapping a tile's position range are staged in shared memory (range
// located by a warp-cooperative search in the partition pass), so C is read
// once too; a narrow-plain C is decoded inline at each point. Integer sums
// wrap exactly as the chain's int64 arithmetic; f64 within tolerance.
#include <limits>

#include "merge_walk.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

struct AggPart {  // same layout as k_agg.cu
  unsigned long long isum;
  double fsum;
  long long cnt;
  long long imin, imax;
  double fmin, fmax;
  double pad;
};

enum CKind { C_RLE_GAPLESS = 0, C_RLE_GAPPED = 1, C_PLAIN = 2 };

struct CSpec {
  const void* v;
  int dt;
  const int64_t* s;
  const int64_t* e;
  int64_t n;  // runs (RLE) or rows (plain)
  int logical, has_center;
  int64_t center;
  int cmp;
  int k_float;
  int64_t ki;
  double kf;
};

template <class T>
__device__ __forceinline__ bool c_pass(const CSpec& c, T x) {
  const T k = c.k_float ? static_cast<T>(c.kf) : static_cast<T>(c.ki);
  return cmp_t<T>(x, k, c.cmp);
}

__device__ __forceinline__ bool c_value_pass(const CSpec& c, int64_t idx) {
  if (c.k_float || dt_is_float_dev(c.dt)) {
    const double x = ld_f64(c.v, c.dt, idx);
    const double k = c.k_float ? c.kf : static_cast<double>(c.ki);
    return cmp_t<double>(x, k, c.cmp);
  }
  return cmp_t<int64_t>(ld_i64(c.v, c.dt, idx), c.ki, c.cmp);
}

__device__ __forceinline__ bool c_plain_pass(const CSpec& c, int64_t row) {
  int64_t x = wrap_to(c.logical, ld_i64(c.v, c.dt, row));
  if (c.has_center)
    x = wrap_to(c.logical, static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(c.center)));
  return cmp_t<int64_t>(x, c.ki, c.cmp);
}

// partition: merge split of (points P, run ends E) at each tile boundary,
// plus the first C run whose end >= the tile's first point.
__global__ void k_fused_partition(const int64_t* __restrict__ P, int64_t np,
                                  const int64_t* __restrict__ E, int64_t ne, int64_t tile,
                                  int64_t nparts, const int64_t* __restrict__ ce, int64_t nc,
                                  int64_t* __restrict__ part, int64_t* __restrict__ cpart) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= nparts) return;
  int64_t diag = w * tile;
  if (diag > np + ne) diag = np + ne;
  const int64_t i = warp_merge_path(P, np, E, ne, diag);
  int64_t c = nc;
  if (ce != nullptr && i < np) c = warp_lower_bound(ce, nc, __ldg(reinterpret_cast<const long long*>(P) + i));
  if ((threadIdx.x & 31) == 0) {
    part[w] = i;
    if (cpart) cpart[w] = c;
  }
}

template <int BLOCK, int ITEMS, int CCAP, class T, bool X_GAPLESS, int CK>
__global__ void __launch_bounds__(BLOCK)
    k_filtered_points_reduce(MergeArgs m, const int64_t* __restrict__ xs, const void* __restrict__ xv,
                             int xdt, const void* __restrict__ yv, int ydt, CSpec c,
                             const int64_t* __restrict__ cpart, int op, int swap,
                             AggPart* __restrict__ parts, int* __restrict__ err) {
  using Tile = MergeTile<BLOCK, ITEMS>;
  __shared__ int64_t sk[Tile::TILE];
  __shared__ int64_t c_e[CK == C_PLAIN ? 1 : CCAP];
  __shared__ int64_t c_s[CK == C_RLE_GAPPED ? CCAP : 1];  // start, or INT64_MAX if failing
  __shared__ uint8_t c_ok[CK == C_PLAIN ? 1 : CCAP];
  Tile t;
  const int tile = blockIdx.x;
  int64_t c0 = 0, cn = 0;
  bool c_staged = false;
  if (CK != C_PLAIN) {
    c0 = cpart[tile];
    int64_t c1 = cpart[tile + 1];
    if (c1 >= c.n) c1 = c.n - 1;
    cn = c1 - c0 + 1;
    if (c0 >= c.n) cn = 0;
    c_staged = cn <= CCAP;
    if (c_staged) {
      for (int64_t q = threadIdx.x; q < cn; q += BLOCK) {
        c_e[q] = ldg64(c.e, c0 + q);
        if (CK == C_RLE_GAPPED) c_s[q] = ldg64(c.s, c0 + q);
        c_ok[q] = c_value_pass(c, c0 + q) ? 1 : 0;
      }
    }
  }
  t.load(m, tile, sk);  // includes __syncthreads()

  uint64_t isum = 0;
  double fsum = 0.0;
  int64_t cnt = 0;
  int lerr = 0;
  int64_t ccur = -1;  // local C cursor (staged index or global index)
  t.walk(sk, [&](int64_t i, int64_t j, bool takeP, int64_t p) {
    if (!takeP) return;  // run-end step: nothing to emit
    // A (RLE, "x") covers p?
    if (j >= m.nb) return;
    if (!X_GAPLESS && ldg64(xs, j) > p) return;
    // predicate on C at p
    bool pass;
    if (CK == C_PLAIN) {
      pass = p < c.n && c_plain_pass(c, p);
    } else if (c_staged) {
      if (ccur < 0) {  // first point of this thread: binary search the staged ends
        int64_t lo = 0, hi = cn;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (c_e[mid] < p) lo = mid + 1;
          else hi = mid;
        }
        ccur = lo;
      }
      while (ccur < cn && c_e[ccur] < p) ++ccur;
      pass = ccur < cn && c_ok[ccur] && (CK == C_RLE_GAPLESS || c_s[ccur] <= p);
    } else {
      if (ccur < 0) ccur = lower_bound_g(c.e, c.n, p);
      while (ccur < c.n && ldg64(c.e, ccur) < p) ++ccur;
      pass = ccur < c.n && (CK == C_RLE_GAPLESS || ldg64(c.s, ccur) <= p) && c_value_pass(c, ccur);
    }
    if (!pass) return;
    const T xa = ld_as<T>(xv, xdt, j);
    const T yb = ld_as<T>(yv, ydt, i);
    const T r = swap ? arith_t<T>(yb, xa, op, &lerr) : arith_t<T>(xa, yb, op, &lerr);
    isum += static_cast<uint64_t>(static_cast<int64_t>(r));
    fsum += static_cast<double>(r);
    ++cnt;
  });
  if (lerr) atomicExch(err, 1);
  // block reduction -> one partial per tile
  __shared__ uint64_t ru[BLOCK / 32 + 1];
  __shared__ double rf[BLOCK / 32 + 1];
  const uint64_t bi = block_sum<BLOCK>(isum, ru);
  const double bf = block_sum<BLOCK>(fsum, rf);
  const uint64_t bc = block_sum<BLOCK>(static_cast<uint64_t>(cnt), ru);
  if (threadIdx.x == 0) {
    AggPart pp{};
    pp.isum = bi;
    pp.fsum = bf;
    pp.cnt = static_cast<long long>(bc);
    parts[tile] = pp;
  }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_sum_parts(const AggPart* __restrict__ parts, int64_t n, AggPart* __restrict__ out) {
  __shared__ uint64_t ru[BLOCK / 32 + 1];
  __shared__ double rf[BLOCK / 32 + 1];
  uint64_t isum = 0, cnt = 0;
  double fsum = 0.0;
  for (int64_t q = threadIdx.x; q < n; q += BLOCK) {
    isum += parts[q].isum;
    fsum += parts[q].fsum;
    cnt += static_cast<uint64_t>(parts[q].cnt);
  }
  isum = block_sum<BLOCK>(isum, ru);
  fsum = block_sum<BLOCK>(fsum, rf);
  cnt = block_sum<BLOCK>(cnt, ru);
  if (threadIdx.x == 0) {
    AggPart pp{};
    pp.isum = isum;
    pp.fsum = fsum;
    pp.cnt = static_cast<long long>(cnt);
    *out = pp;
  }
}

}  // namespace dev

AggOut filtered_aggregate_binop_chain(const CtxPtr& ctx, const DCol& c, Scalar k, int cmp,
                                      const DCol& a, const DCol& b, int op, int fn);

namespace {

constexpr int FB = 256, FI = 8, FCAP = 1024;

template <class T, bool XG, int CK>
void launch_fused(const CtxPtr& ctx, unsigned g, const dev::MergeArgs& m, const DCol& x, const DCol& y,
                  const dev::CSpec& cs, const int64_t* cpart, int op, int swap, dev::AggPart* parts,
                  int* err) {
  dev::k_filtered_points_reduce<FB, FI, FCAP, T, XG, CK><<<g, FB, 0, ctx->stream>>>(
      m, x.s.pos(), x.v.raw(), x.v.dt, y.v.raw(), y.v.dt, cs, cpart, op, swap, parts, err);
}

template <class T, bool XG>
void launch_ck(int ck, const CtxPtr& ctx, unsigned g, const dev::MergeArgs& m, const DCol& x, const DCol& y,
               const dev::CSpec& cs, const int64_t* cpart, int op, int swap, dev::AggPart* parts, int* err) {
  switch (ck) {
    case dev::C_RLE_GAPLESS: launch_fused<T, XG, dev::C_RLE_GAPLESS>(ctx, g, m, x, y, cs, cpart, op, swap, parts, err); break;
    case dev::C_RLE_GAPPED: launch_fused<T, XG, dev::C_RLE_GAPPED>(ctx, g, m, x, y, cs, cpart, op, swap, parts, err); break;
    default: launch_fused<T, XG, dev::C_PLAIN>(ctx, g, m, x, y, cs, cpart, op, swap, parts, err); break;
  }
}

}  // namespace

AggOut filtered_aggregate_binop(const CtxPtr& ctx, const DCol& c, Scalar k, int cmp, const DCol& a,
                                const DCol& b, int op, int fn) {
  require(cmp >= RQ_LT && cmp <= RQ_GT, "compare_scalar: comparison operator required");
  require(op >= RQ_ADD && op <= RQ_DIV, "arith: arithmetic operator required");
  require(c.total == a.total && a.total == b.total, "filter: total_size mismatch");
  const bool shape_ok = (a.enc == RQ_ENC_RLE && b.enc == RQ_ENC_INDEX) ||
                        (a.enc == RQ_ENC_INDEX && b.enc == RQ_ENC_RLE);
  const bool c_ok = c.enc == RQ_ENC_RLE ||
                    (c.enc == RQ_ENC_PLAIN && !dt_float(c.v.dt) && !dt_float(c.logical) && !k.is_float);
  const bool fn_ok = fn == RQ_SUM || fn == RQ_COUNT || fn == RQ_AVG;
  if (!shape_ok || !c_ok || !fn_ok) return filtered_aggregate_binop_chain(ctx, c, k, cmp, a, b, op, fn);

  const DCol& x = a.enc == RQ_ENC_RLE ? a : b;  // runs
  const DCol& y = a.enc == RQ_ENC_RLE ? b : a;  // points
  const int swap = a.enc == RQ_ENC_RLE ? 0 : 1;
  const bool flt = dt_float(x.v.dt) || dt_float(y.v.dt);
  const bool xg = col_gapless(ctx, x);
  int ck = dev::C_PLAIN;
  if (c.enc == RQ_ENC_RLE) ck = col_gapless(ctx, c) ? dev::C_RLE_GAPLESS : dev::C_RLE_GAPPED;

  dev::CSpec cs{};
  cs.v = c.v.raw();
  cs.dt = c.v.dt;
  cs.s = c.s.pos();
  cs.e = c.e.pos();
  cs.n = c.enc == RQ_ENC_RLE ? c.s.n : c.v.n;
  cs.logical = c.logical;
  cs.has_center = c.has_center ? 1 : 0;
  cs.center = c.center;
  cs.cmp = cmp;
  cs.k_float = k.is_float ? 1 : 0;
  cs.ki = k.i;
  cs.kf = k.f;

  const int64_t np = y.p.n, ne = x.e.n;
  dev::AggPart res{};
  if (np > 0 && ne > 0 && cs.n > 0) {
    constexpr int64_t TILE = FB * FI;
    const int64_t ntiles = (np + ne + TILE - 1) / TILE;
    DArr part = alloc_arr(ctx, RQ_I64, ntiles + 1);
    DArr cpart = alloc_arr(ctx, RQ_I64, ntiles + 1);
    DArr parts = alloc_arr(ctx, RQ_I64, ntiles * (sizeof(dev::AggPart) / 8));
    DArr out = alloc_arr(ctx, RQ_I64, sizeof(dev::AggPart) / 8);
    DArr err = alloc_arr(ctx, RQ_I32, 2);
    RQ_CUDA_CHECK(cudaMemsetAsync(err.raw_mut(), 0, 8, ctx->stream));
    {
      KTimer timer(ctx, "filtered_points_reduce");
      const int64_t nparts = ntiles + 1;
      dev::k_fused_partition<<<static_cast<unsigned>((nparts * 32 + 255) / 256), 256, 0, ctx->stream>>>(
          y.p.pos(), np, x.e.pos(), ne, TILE, nparts, ck == dev::C_PLAIN ? nullptr : c.e.pos(), cs.n,
          part.as<int64_t>(), ck == dev::C_PLAIN ? nullptr : cpart.as<int64_t>());
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
      dev::MergeArgs m{y.p.pos(), np, x.e.pos(), ne, part.as<int64_t>()};
      const unsigned g = static_cast<unsigned>(ntiles);
      auto* P = parts.as<dev::AggPart>();
      if (flt) {
        if (xg) launch_ck<double, true>(ck, ctx, g, m, x, y, cs, cpart.pos(), op, swap, P, err.as<int>());
        else launch_ck<double, false>(ck, ctx, g, m, x, y, cs, cpart.pos(), op, swap, P, err.as<int>());
      } else {
        if (xg) launch_ck<int64_t, true>(ck, ctx, g, m, x, y, cs, cpart.pos(), op, swap, P, err.as<int>());
        else launch_ck<int64_t, false>(ck, ctx, g, m, x, y, cs, cpart.pos(), op, swap, P, err.as<int>());
      }
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
      dev::k_sum_parts<256><<<1, 256, 0, ctx->stream>>>(P, ntiles, out.as<dev::AggPart>());
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
    }
    RQ_CUDA_CHECK(cudaMemcpyAsync(ctx->pinned, out.raw(), sizeof(dev::AggPart), cudaMemcpyDeviceToHost, ctx->stream));
    RQ_CUDA_CHECK(cudaMemcpyAsync(ctx->pinned + 16, err.raw(), 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    res = *reinterpret_cast<const dev::AggPart*>(ctx->pinned);
    if (!flt && op == RQ_DIV && static_cast<int32_t>(ctx->pinned[16] & 0xffffffff))
      fail("integer division by zero");
  }
  AggOut o;
  if (fn == RQ_COUNT) {
    o.dtype = RQ_I64;
    o.i = res.cnt;
  } else if (fn == RQ_AVG) {
    o.dtype = RQ_F64;
    o.f = res.cnt > 0 ? res.fsum / static_cast<double>(res.cnt) : std::numeric_limits<double>::quiet_NaN();
  } else if (flt) {
    o.dtype = RQ_F64;
    o.f = res.fsum;
  } else {
    o.dtype = RQ_I64;
    o.i = static_cast<int64_t>(res.isum);
  }
  return o;
}

}  // namespace rqb
