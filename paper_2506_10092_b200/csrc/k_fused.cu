// k_fused.cu — single-pass filtered aggregate (the C2 query shape).
//
// The reference evaluates
//   m  = compare_scalar(C, k, cmp)                 (align.cpp:598-652)
//   A' = filter(A, m); B' = filter(B, m)           (align.cpp:755-771)
//   aggregate_all(arith(A', B', op), fn)           (align.cpp:495-508, groupby.cpp:164-172)
// materialising the mask, two filtered columns and the product. With A RLE
// and B Index, every surviving slot is a point p of B with C(p) passing and
// A covering p, so the whole chain is
//   Σ_{p ∈ B, pred(C(p)), p ∈ cover(A)} op(A(p), B(p)).
//
// Points-driven single pass: B's points are cut into fixed tiles
// (BLOCK×ITEMS points); a partition pass locates, per tile boundary, the
// first A run and first C run that can contain the boundary point (one
// warp-cooperative 32-ary search each). Each CTA stages its tile's A-run-end
// window and C window (ends + predicate flag, evaluated once per run) in
// shared memory with coalesced loads; every lane then takes one point per
// round (striped → coalesced point/value loads) and resolves it with a
// branchless binary search in shared memory — uniform trip counts, no
// divergence, no global-latency chains. Windows larger than the staging
// capacity fall back to a global binary search inside the window. Every byte
// of A's run ends, B's points and C's runs comes from HBM once; A's values
// are gathered only for covered points. (A merge-path walk over all run ends
// measured issue-bound here: most steps were run ends with no output.)
// Integer sums wrap exactly like the chain's int64 arithmetic; f64 within
// tolerance.
#include <cstdlib>
#include <limits>
#include <type_traits>

#include "device_common.cuh"
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
  int opmask;  // bit c set: comparison holds for outcome class c (<, ==, >)
};

inline int cmp_opmask(int cmp) {
  switch (cmp) {
    case RQ_LT: return 0b001;
    case RQ_LE: return 0b011;
    case RQ_EQ: return 0b010;
    case RQ_NE: return 0b101;
    case RQ_GE: return 0b110;
    default: return 0b100;  // GT
  }
}

struct XSpec {  // the RLE data column
  const int64_t* s;
  const int64_t* e;
  const void* v;
  int dt;
  int64_t n;
  int gapless;
};

__device__ __forceinline__ int64_t ld_i64_hot(const void* p, int dt, int64_t i) {
  return dt == RQ_I64 ? ldg64(static_cast<const int64_t*>(p), i) : ld_i64(p, dt, i);
}
__device__ __forceinline__ double ld_f64_hot(const void* p, int dt, int64_t i) {
  return dt == RQ_F64 ? __ldg(static_cast<const double*>(p) + i) : ld_f64(p, dt, i);
}
template <class T>
__device__ __forceinline__ T ld_hot(const void* p, int dt, int64_t i);
// storage already of the arithmetic type (the common case: int64 / f64)
template <class T>
__device__ __forceinline__ T ld_same(const void* p, int64_t i) {
  return __ldg(static_cast<const T*>(p) + i);
}
template <>
__device__ __forceinline__ int64_t ld_hot<int64_t>(const void* p, int dt, int64_t i) {
  return ld_i64_hot(p, dt, i);
}
template <>
__device__ __forceinline__ double ld_hot<double>(const void* p, int dt, int64_t i) {
  return ld_f64_hot(p, dt, i);
}

// Branch-free predicate: outcome class (0: x<k, 1: x==k, 2: x>k) selects a
// bit of the comparison's 3-bit truth mask (cmp_opmask on the host).
__device__ __forceinline__ bool c_run_pass(const CSpec& c, int64_t idx) {
  int cls;
  if (c.k_float || dt_is_float_dev(c.dt)) {
    const double x = ld_f64(c.v, c.dt, idx);
    const double k = c.k_float ? c.kf : static_cast<double>(c.ki);
    if (x != x || k != k) return c.cmp == RQ_NE;  // NaN: only != holds
    cls = x < k ? 0 : (x == k ? 1 : 2);
  } else {
    const int64_t x = ld_i64_hot(c.v, c.dt, idx);
    cls = x < c.ki ? 0 : (x == c.ki ? 1 : 2);
  }
  return (c.opmask >> cls) & 1;
}

__device__ __forceinline__ bool c_plain_pass(const CSpec& c, int64_t row) {
  int64_t x = wrap_to(c.logical, ld_i64(c.v, c.dt, row));
  if (c.has_center)
    x = wrap_to(c.logical, static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(c.center)));
  const int cls = x < c.ki ? 0 : (x == c.ki ? 1 : 2);
  return (c.opmask >> cls) & 1;
}

// first index in [lo, hi) with e[idx] >= key (hi if none)
__device__ __forceinline__ int64_t lb_window(const int64_t* __restrict__ e, int64_t lo, int64_t hi,
                                             int64_t key) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ldg64(e, mid) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// tile boundary t: first A run and first C run with end >= P[t * tile]
__global__ void k_points_partition(const int64_t* __restrict__ P, int64_t np, int64_t tile,
                                   int64_t nparts, const int64_t* __restrict__ xe, int64_t nx,
                                   const int64_t* __restrict__ ce, int64_t nc,
                                   int64_t* __restrict__ apart, int64_t* __restrict__ cpart) {
  // two warps per boundary: even warps search A's ends, odd warps C's ends
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t w = gw >> 1;
  const bool is_c = gw & 1;
  if (w >= nparts || (is_c && !ce)) return;  // warp-uniform
  const int64_t q = w * tile;
  int64_t r = is_c ? nc : nx;
  if (q < np) r = is_c ? warp_lower_bound(ce, nc, ldg64(P, q)) : warp_lower_bound(xe, nx, ldg64(P, q));
  if ((threadIdx.x & 31) == 0) (is_c ? cpart : apart)[w] = r;
}

template <class T, int OP>
__device__ __forceinline__ T apply_op(T x, T y, int* err) {
  return arith_t<T>(x, y, OP, err);
}

// Branchless lower_bound over a shared-memory window of 32-bit offsets,
// fully unrolled over the power-of-two capacity CAP (log2(CAP) steps of
// add / compare / load / select; identical trip count in every lane).
// Entries at index >= len hold INT32_MAX, so no bounds test is needed.
template <int CAP>
__device__ __forceinline__ int smem_rank32(const int32_t* w, int32_t key) {
  int pos = 0;  // number of entries < key found so far
#pragma unroll
  for (int step = CAP / 2; step > 0; step >>= 1) pos = (w[pos + step - 1] < key) ? pos + step : pos;
  return pos + (w[pos] < key ? 1 : 0);
}

template <int BLOCK, int ITEMS, int ACAP, int CCAP, class T, int OP, int CK, bool BLOCKED, bool SAME>
__global__ void __launch_bounds__(BLOCK)
    k_points_filtered_reduce(const int64_t* __restrict__ P, const void* __restrict__ yv, int ydt,
                             int64_t np, XSpec x, CSpec c, const int64_t* __restrict__ apart,
                             const int64_t* __restrict__ cpart, int swap,
                             AggPart* __restrict__ parts, int* __restrict__ err) {
  constexpr int TILE = BLOCK * ITEMS;
  static_assert((ACAP & (ACAP - 1)) == 0 && (CCAP & (CCAP - 1)) == 0, "power-of-two windows");
  __shared__ int32_t wa[ACAP];
  __shared__ int32_t wc[CK == C_PLAIN ? 1 : CCAP];
  __shared__ uint8_t wok[CK == C_PLAIN ? 1 : CCAP];
  const int tile = blockIdx.x;
  const int64_t tbase = static_cast<int64_t>(tile) * TILE;
  const int64_t tnext = tbase + TILE;
  // positions inside the tile are stored as 32-bit offsets from its first
  // point; valid when the tile spans < 2^31 - 1 rows (checked per tile)
  const int64_t p0 = ldg64(P, tbase);
  const int64_t tlast = (tnext < np ? tnext : np) - 1;
  const bool narrow = ldg64(P, tlast) - p0 < INT32_MAX - 1;
  // tile windows (from the partition pass): runs that may contain this
  // tile's points
  const int64_t a_lo = apart[tile];
  int64_t a_hi = apart[tile + 1] + 1;
  if (a_hi > x.n) a_hi = x.n;
  const int64_t alen = a_hi > a_lo ? a_hi - a_lo : 0;
  const bool a_staged = narrow && alen < ACAP;
  // search length: the power of two above the window (uniform per CTA)
  // smallest power of two > alen (alen < 2^31 whenever the window is staged)
  const int la = alen > 0 ? (1 << (32 - __clz(static_cast<int>(min(alen, static_cast<int64_t>(INT32_MAX / 2)))))) : 1;
  int64_t c_lo = 0, clen = 0;
  bool c_staged = false;
  int lc = 1;
  if (CK != C_PLAIN) {
    c_lo = cpart[tile];
    int64_t c_hi = cpart[tile + 1] + 1;
    if (c_hi > c.n) c_hi = c.n;
    clen = c_hi > c_lo ? c_hi - c_lo : 0;
    c_staged = narrow && clen < CCAP;
    lc = clen > 0 ? (1 << (32 - __clz(static_cast<int>(min(clen, static_cast<int64_t>(INT32_MAX / 2)))))) : 1;
  }
  // coalesced staging of the run windows as 32-bit offsets from p0 (C's
  // predicate evaluated once per run); [len, L) padded with INT32_MAX. All
  // loads of a thread are issued before any store.
  static_assert(ACAP % BLOCK == 0 && CCAP % BLOCK == 0, "window capacity multiple of BLOCK");
  constexpr int AU = ACAP / BLOCK, CU = CCAP / BLOCK;
  const int64_t pad = p0 + INT32_MAX;
  if (a_staged) {
    int64_t t[AU];
#pragma unroll
    for (int u = 0; u < AU; ++u) {
      const int q = u * BLOCK + threadIdx.x;
      t[u] = q < alen ? ldg64(x.e, a_lo + q) : pad;
    }
#pragma unroll
    for (int u = 0; u < AU; ++u) {
      const int q = u * BLOCK + threadIdx.x;
      if (q < la) wa[q] = static_cast<int32_t>(min(t[u] - p0, static_cast<int64_t>(INT32_MAX)));
    }
  }
  if (CK != C_PLAIN && c_staged) {
    int64_t te[CU];
    bool tok[CU];
#pragma unroll
    for (int u = 0; u < CU; ++u) {
      const int q = u * BLOCK + threadIdx.x;
      te[u] = q < clen ? ldg64(c.e, c_lo + q) : pad;
      tok[u] = q < clen && c_run_pass(c, c_lo + q);
    }
#pragma unroll
    for (int u = 0; u < CU; ++u) {
      const int q = u * BLOCK + threadIdx.x;
      if (q < lc) {
        wc[q] = static_cast<int32_t>(min(te[u] - p0, static_cast<int64_t>(INT32_MAX)));
        wok[q] = tok[u] ? 1 : 0;
      }
    }
  }
  __syncthreads();

  uint64_t isum = 0;
  double fsum = 0.0;
  int64_t cnt = 0;
  int lerr = 0;
  // point q of lane k: striped (coalesced scalar loads, lockstep searches)
  // or blocked (ITEMS consecutive points per lane: one full search for the
  // first point, short forward scans for the rest — the points are sorted)
  auto qof = [&](int k) -> int64_t {
    return BLOCKED ? tbase + static_cast<int64_t>(threadIdx.x) * ITEMS + k
                   : tbase + static_cast<int64_t>(k) * BLOCK + threadIdx.x;
  };
  int64_t pts[ITEMS];
  int32_t key[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t q = qof(k);
    pts[k] = q < np ? ldg64(P, q) : INT64_MAX;
    key[k] = static_cast<int32_t>(pts[k] - p0);  // used only when narrow
  }
  int ra[ITEMS], rc[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) ra[k] = rc[k] = 0;
  const bool do_c = CK != C_PLAIN && c_staged;
  constexpr int NS = BLOCKED ? 1 : ITEMS;  // points searched from scratch
  // search over [0, L) with L the window's power of two (trip count log2 L,
  // uniform per CTA); both searches advance in the same step loop
#pragma unroll
  for (int step = (ACAP > CCAP ? ACAP : CCAP) / 2; step > 0; step >>= 1) {
    if (a_staged && step < la) {
#pragma unroll
      for (int k = 0; k < NS; ++k) ra[k] = (wa[ra[k] + step - 1] < key[k]) ? ra[k] + step : ra[k];
    }
    if (do_c && step < lc) {
#pragma unroll
      for (int k = 0; k < NS; ++k) rc[k] = (wc[rc[k] + step - 1] < key[k]) ? rc[k] + step : rc[k];
    }
  }
  if (a_staged) {
#pragma unroll
    for (int k = 0; k < NS; ++k) ra[k] += wa[ra[k]] < key[k] ? 1 : 0;
  }
  if (do_c) {
#pragma unroll
    for (int k = 0; k < NS; ++k) rc[k] += wc[rc[k]] < key[k] ? 1 : 0;
  }
  if (BLOCKED) {  // forward scans; padding (INT32_MAX) stops every scan
#pragma unroll
    for (int k = 1; k < ITEMS; ++k) {
      // two branchless steps cover the usual gap between neighbouring
      // points; the loop only runs for longer gaps
      int r = ra[k - 1];
      if (a_staged) {
        r += wa[r] < key[k] ? 1 : 0;
        r += wa[r] < key[k] ? 1 : 0;
        while (wa[r] < key[k]) ++r;
      }
      ra[k] = r;
      int t = rc[k - 1];
      if (do_c) {
        t += wc[t] < key[k] ? 1 : 0;
        while (wc[t] < key[k]) ++t;
      }
      rc[k] = t;
    }
  }
  // qualify every point (A covers it, C's run passes) ...
  int64_t arun[ITEMS];
  bool take[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t q = qof(k);
    const int64_t p = pts[k];
    take[k] = false;
    arun[k] = a_lo;
    if (q >= np) continue;
    const int64_t ar = a_staged ? a_lo + ra[k] : lb_window(x.e, a_lo, a_hi, p);
    if (ar >= a_hi) continue;
    if (!x.gapless && ldg64(x.s, ar) > p) continue;
    bool pass;
    if (CK == C_PLAIN) {
      pass = p < c.n && c_plain_pass(c, p);
    } else if (c_staged) {
      const int cr = rc[k];
      pass = cr < clen && wok[cr] && (CK == C_RLE_GAPLESS || ldg64(c.s, c_lo + cr) <= p);
    } else {
      const int64_t cr = lb_window(c.e, c_lo, c_lo + clen, p);
      pass = cr < c_lo + clen && (CK == C_RLE_GAPLESS || ldg64(c.s, cr) <= p) && c_run_pass(c, cr);
    }
    take[k] = pass;
    arun[k] = ar;
  }
  // ... then gather both operands for all points at once (independent loads)
  T xa[ITEMS], yb[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t q = qof(k);
    if (SAME) {
      xa[k] = take[k] ? ld_same<T>(x.v, arun[k]) : T(0);
      yb[k] = take[k] ? ld_same<T>(yv, q) : T(0);
    } else {
      xa[k] = take[k] ? ld_hot<T>(x.v, x.dt, arun[k]) : T(0);
      yb[k] = take[k] ? ld_hot<T>(yv, ydt, q) : T(0);
    }
  }
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (!take[k]) continue;
    const T r = swap ? apply_op<T, OP>(yb[k], xa[k], &lerr) : apply_op<T, OP>(xa[k], yb[k], &lerr);
    isum += static_cast<uint64_t>(static_cast<int64_t>(r));
    fsum += static_cast<double>(r);
    ++cnt;
  }
  if (lerr) atomicExch(err, 1);
  // one block reduction of the three accumulators
  __shared__ uint64_t ru[BLOCK / 32];
  __shared__ double rf[BLOCK / 32];
  __shared__ uint64_t rn[BLOCK / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  isum = warp_sum(isum);
  fsum = warp_sum(fsum);
  const uint64_t ucnt = warp_sum(static_cast<uint64_t>(cnt));
  if (lane == 0) {
    ru[wid] = isum;
    rf[wid] = fsum;
    rn[wid] = ucnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    AggPart pp{};
    for (int w = 0; w < BLOCK / 32; ++w) {
      pp.isum += ru[w];
      pp.fsum += rf[w];
      pp.cnt += static_cast<long long>(rn[w]);
    }
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
  // fixed-order strided fold; 8 partials per thread per batch so the loads
  // of a batch are in flight together
  constexpr int U = 8;
  for (int64_t q0 = 0; q0 < n; q0 += static_cast<int64_t>(BLOCK) * U) {
    unsigned long long bi[U];
    double bf[U];
    long long bc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + static_cast<int64_t>(u) * BLOCK + threadIdx.x;
      const bool ok = q < n;
      bi[u] = ok ? parts[q].isum : 0ull;
      bf[u] = ok ? parts[q].fsum : 0.0;
      bc[u] = ok ? parts[q].cnt : 0ll;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      isum += bi[u];
      fsum += bf[u];
      cnt += static_cast<uint64_t>(bc[u]);
    }
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

constexpr int FB = 256, FI = 4, FACAP = 2048, FCCAP = 1024;

struct FusedLaunch {
  unsigned grid;
  const DCol* y;
  dev::XSpec xs;
  dev::CSpec cs;
  const int64_t* apart;
  const int64_t* cpart;
  int swap;
  dev::AggPart* parts;
  int* err;
};

// (4 points per thread measured equal to 8 with a 2×-wider window, r1)
template <class T, int OP, int CK>
void launch3(const CtxPtr& ctx, const FusedLaunch& f) {
  const int32_t tdt = std::is_same<T, double>::value ? RQ_F64 : RQ_I64;
  const bool same = f.xs.dt == tdt && f.y->v.dt == tdt;
#define RQ_LAUNCH_C2(B, S)                                                                          \
  dev::k_points_filtered_reduce<FB, FI, FACAP, FCCAP, T, OP, CK, B, S><<<f.grid, FB, 0, ctx->stream>>>( \
      f.y->p.pos(), f.y->v.raw(), f.y->v.dt, f.y->p.n, f.xs, f.cs, f.apart, f.cpart, f.swap, f.parts, f.err)
  // blocked points per lane (r1: 0.145 ms vs 0.162 ms striped at C2 1B rows)
  if (same) RQ_LAUNCH_C2(true, true);
  else RQ_LAUNCH_C2(true, false);
#undef RQ_LAUNCH_C2
}

template <class T, int OP>
void launch2(int ck, const CtxPtr& ctx, const FusedLaunch& f) {
  switch (ck) {
    case dev::C_RLE_GAPLESS: launch3<T, OP, dev::C_RLE_GAPLESS>(ctx, f); break;
    case dev::C_RLE_GAPPED: launch3<T, OP, dev::C_RLE_GAPPED>(ctx, f); break;
    default: launch3<T, OP, dev::C_PLAIN>(ctx, f); break;
  }
}

template <class T>
void launch1(int op, int ck, const CtxPtr& ctx, const FusedLaunch& f) {
  switch (op) {
    case RQ_ADD: launch2<T, RQ_ADD>(ck, ctx, f); break;
    case RQ_SUB: launch2<T, RQ_SUB>(ck, ctx, f); break;
    case RQ_MUL: launch2<T, RQ_MUL>(ck, ctx, f); break;
    default: launch2<T, RQ_DIV>(ck, ctx, f); break;
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
  const bool flt = dt_float(x.v.dt) || dt_float(y.v.dt);
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
  cs.opmask = dev::cmp_opmask(cmp);
  dev::XSpec xs{x.s.pos(), x.e.pos(), x.v.raw(), x.v.dt, x.e.n, col_gapless(ctx, x) ? 1 : 0};

  const int64_t np = y.p.n;
  dev::AggPart res{};
  if (np > 0 && xs.n > 0 && cs.n > 0) {
    constexpr int64_t TILE = static_cast<int64_t>(FB) * FI;
    const int64_t ntiles = (np + TILE - 1) / TILE;
    DArr apart = alloc_arr(ctx, RQ_I64, ntiles + 1);
    DArr cpart = alloc_arr(ctx, RQ_I64, ntiles + 1);
    DArr parts = alloc_arr(ctx, RQ_I64, ntiles * (sizeof(dev::AggPart) / 8));
    DArr out = alloc_arr(ctx, RQ_I64, sizeof(dev::AggPart) / 8 + 1);
    int* err = reinterpret_cast<int*>(out.as<int64_t>() + sizeof(dev::AggPart) / 8);
    RQ_CUDA_CHECK(cudaMemsetAsync(err, 0, 8, ctx->stream));
    {
      KTimer timer(ctx, "filtered_points_reduce");
      const int64_t nparts = ntiles + 1;
      dev::k_points_partition<<<static_cast<unsigned>((nparts * 64 + 255) / 256), 256, 0, ctx->stream>>>(
          y.p.pos(), np, TILE, nparts, x.e.pos(), xs.n, ck == dev::C_PLAIN ? nullptr : c.e.pos(), cs.n,
          apart.as<int64_t>(), ck == dev::C_PLAIN ? nullptr : cpart.as<int64_t>());
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
      FusedLaunch f{static_cast<unsigned>(ntiles), &y, xs, cs, apart.pos(), cpart.pos(),
                    a.enc == RQ_ENC_RLE ? 0 : 1, parts.as<dev::AggPart>(), err};
      if (flt) launch1<double>(op, ck, ctx, f);
      else launch1<int64_t>(op, ck, ctx, f);
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
      dev::k_sum_parts<1024><<<1, 1024, 0, ctx->stream>>>(parts.as<dev::AggPart>(), ntiles,
                                                        out.as<dev::AggPart>());
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
    }
    const int64_t* h = ctx->readback(out.raw(), sizeof(dev::AggPart) + 8);
    res = *reinterpret_cast<const dev::AggPart*>(h);
    const int32_t e = static_cast<int32_t>(h[sizeof(dev::AggPart) / 8] & 0xffffffff);
    if (!flt && op == RQ_DIV && e) fail("integer division by zero");
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
