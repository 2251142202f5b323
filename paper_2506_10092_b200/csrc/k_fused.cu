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
#include <cstring>
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

// ---------------------------------------------------------------------------
// Persistent TMA variant (the production path when every buffer is 16-B
// aligned). Each CTA owns a CONTIGUOUS range of point tiles, so the first
// A/C run a tile can touch is the run of the previous tile's last point:
// one warp-level search per CTA replaces the per-tile partition pass, and
// the tile windows are chained forward. Per tile, one elected thread issues
// 1-D bulk copies (cp.async.bulk, completing on an mbarrier) of the tile's
// points and B values, A's run-end window and C's run-end + value window, in
// the stored int64 / storage-width form (no register staging, no
// conversion); lanes then resolve ITEMS consecutive points each with one
// branch-free shared-memory lower_bound and short forward scans. The window
// length is predicted from the previous tile's span (×1.25 + 32, at most
// AW / CW runs); a point past a window's last staged run falls back to a
// global search, so the prediction affects only speed. The per-CTA partials
// are folded by the last CTA to finish (ticket counter that wraps back to 0),
// in a fixed order.
// ---------------------------------------------------------------------------

template <class T>
__device__ __forceinline__ T lds_as(const unsigned char* base, int dt, int i);
template <>
__device__ __forceinline__ int64_t lds_as<int64_t>(const unsigned char* b, int dt, int i) {
  switch (dt) {
    case RQ_I8: return reinterpret_cast<const int8_t*>(b)[i];
    case RQ_I16: return reinterpret_cast<const int16_t*>(b)[i];
    case RQ_I32: return reinterpret_cast<const int32_t*>(b)[i];
    case RQ_I64: return reinterpret_cast<const int64_t*>(b)[i];
    case RQ_F32: return static_cast<int64_t>(reinterpret_cast<const float*>(b)[i]);
    default: return static_cast<int64_t>(reinterpret_cast<const double*>(b)[i]);
  }
}
template <>
__device__ __forceinline__ double lds_as<double>(const unsigned char* b, int dt, int i) {
  switch (dt) {
    case RQ_I8: return reinterpret_cast<const int8_t*>(b)[i];
    case RQ_I16: return reinterpret_cast<const int16_t*>(b)[i];
    case RQ_I32: return reinterpret_cast<const int32_t*>(b)[i];
    case RQ_I64: return static_cast<double>(reinterpret_cast<const int64_t*>(b)[i]);
    case RQ_F32: return reinterpret_cast<const float*>(b)[i];
    default: return reinterpret_cast<const double*>(b)[i];
  }
}

// c_run_pass on a value staged in shared memory
__device__ __forceinline__ bool c_smem_pass(const CSpec& c, const unsigned char* sv, int idx) {
  if (c.dt == RQ_I64 && !c.k_float) {  // dictionary codes as int64 (the common case)
    const int64_t x = reinterpret_cast<const int64_t*>(sv)[idx];
    return (c.opmask >> (x < c.ki ? 0 : (x == c.ki ? 1 : 2))) & 1;
  }
  int cls;
  if (c.k_float || dt_is_float_dev(c.dt)) {
    const double x = lds_as<double>(sv, c.dt, idx);
    const double k = c.k_float ? c.kf : static_cast<double>(c.ki);
    if (x != x || k != k) return c.cmp == RQ_NE;
    cls = x < k ? 0 : (x == k ? 1 : 2);
  } else {
    const int64_t x = lds_as<int64_t>(sv, c.dt, idx);
    cls = x < c.ki ? 0 : (x == c.ki ? 1 : 2);
  }
  return (c.opmask >> cls) & 1;
}

struct TmaWin {
  int64_t lo16;  // first staged run (multiple of 16)
  int n;         // staged runs
};

__device__ __forceinline__ TmaWin tma_window(int64_t lo, int est, int cap, int64_t total) {
  TmaWin w;
  w.lo16 = lo & ~int64_t(15);
  int64_t n = static_cast<int64_t>(est) + (lo - w.lo16);
  if (n > cap) n = cap;
  if (n > total - w.lo16) n = total - w.lo16;
  w.n = n > 0 ? static_cast<int>(n) : 0;
  return w;
}
__device__ __forceinline__ uint32_t ceil16(uint32_t x) { return (x + 15u) & ~15u; }

// one pipeline stage: A's run-end window, C's run-end window and C's values
template <int AW, int CW>
struct C2Stage {
  // staged runs n < W (W a power of two), padded with INT64_MAX up to the
  // power of two above n (<= W); + 16 for the bulk copy's round-up
  static constexpr int A_CAP = AW + 16;  // >= max(ceil16(AW - 1), AW + 8)
  static constexpr int C_CAP = CW + 16;
  static constexpr size_t A_OFF = 0;
  static constexpr size_t C_OFF = A_OFF + A_CAP * 8;
  static constexpr size_t CV_OFF = C_OFF + C_CAP * 8;
  static constexpr size_t F_OFF = CV_OFF + C_CAP * 8;  // C's predicate per staged run (producer-written)
  static constexpr size_t BYTES = F_OFF + ((C_CAP + 15) & ~15);
};

template <int BLOCK, int ITEMS>
__device__ __forceinline__ void load_keys(const int64_t* __restrict__ P, int64_t np, int64_t q0,
                                          int64_t (&k)[ITEMS]) {
  static_assert(ITEMS % 2 == 0, "pairs of points per 128-bit load");
  if (q0 + ITEMS <= np) {
#pragma unroll
    for (int j = 0; j < ITEMS; j += 2) {
      const longlong2 v = __ldg(reinterpret_cast<const longlong2*>(P + q0 + j));
      k[j] = v.x;
      k[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) k[j] = q0 + j < np ? ldg64(P, q0 + j) : INT64_MAX;
  }
}

template <int BLOCK, int ITEMS, int AW, int CW, int NS, class T, int OP, int CK, bool SAME, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
    k_points_filtered_reduce_tma(const int64_t* __restrict__ P, const void* __restrict__ yv, int ydt,
                                 int64_t np, XSpec x, CSpec c, int64_t ntiles, int swap,
                                 AggPart* __restrict__ parts, unsigned* __restrict__ ticket,
                                 AggPart* __restrict__ out, int* __restrict__ err) {
  constexpr int NCW = BLOCK / 32 - 1;  // consumer warps; warp 0 produces
  constexpr int TILE = NCW * 32 * ITEMS;
  constexpr bool HAS_C = CK != C_PLAIN;
  using S = C2Stage<AW, CW>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[NS], empty[NS], ready[NS];
  __shared__ int64_t s_lo[NS][2];  // [stage][A, C] first staged run
  __shared__ int s_n[NS][2];       // [stage][A, C] staged runs

  const int64_t t_begin = static_cast<int64_t>(blockIdx.x) * ntiles / gridDim.x;
  const int64_t t_end = static_cast<int64_t>(blockIdx.x + 1) * ntiles / gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wc = HAS_C ? dt_width_dev(c.dt) : 1;
  auto sA = [&](int st) { return reinterpret_cast<int64_t*>(smem + st * S::BYTES + S::A_OFF); };
  auto sC = [&](int st) { return reinterpret_cast<int64_t*>(smem + st * S::BYTES + S::C_OFF); };
  auto sCv = [&](int st) { return smem + st * S::BYTES + S::CV_OFF; };
  auto sF = [&](int st) { return smem + st * S::BYTES + S::F_OFF; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 32);  // every producer lane arrives (releasing its own stores)
      mbar_init(&empty[i], NCW);
      mbar_init(&ready[i], 32);  // producer lanes, after C's predicate flags of the landed stage
    }
  }
  __syncthreads();

  uint64_t isum = 0;
  double fsum = 0.0;
  int64_t cnt = 0;
  int lerr = 0;
  if (wid == 0) {
    // ---- producer warp: window chain + staging -------------------------------
    // Tile t's windows start at the runs of its first point, ranked in tile
    // t-1's (landed, padded) windows — a global warp search only when the
    // point lies past them. Full 16-run chunks are bulk-copied; the tail
    // chunk at a column's end and the INT64_MAX pad up to the power-of-two
    // capacity (+8 for the fixed-width forward steps) are written by the
    // lanes, outside the copied range, before the arrive that publishes them.
    int64_t a_cur = 0, c_cur = 0, a_lo16 = 0, c_lo16 = 0;
    // per stage: entries [hw, W + 8) still hold the pad (only what earlier
    // copies into a stage overwrote is re-padded)
    int hwA[NS], hwC[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) hwA[i] = AW + 8, hwC[i] = CW + 8;
    int a_est = AW, c_est = CW, a_n = 0, c_n = 0;
    int64_t pf = t_begin < t_end ? ldg64(P, t_begin * TILE) : 0;
    // last run ends (interpolation round of the start-up search), loaded beside pf
    const int64_t a_last = x.n > 0 ? ldg64(x.e, x.n - 1) : -1;
    const int64_t c_last = HAS_C && c.n > 0 ? ldg64(c.e, c.n - 1) : -1;
    for (int64_t t = t_begin; t < t_end; ++t) {
      const int st = static_cast<int>((t - t_begin) % NS);
      const uint32_t use = static_cast<uint32_t>((t - t_begin) / NS);
      const int pst = static_cast<int>((t - 1 - t_begin + NS) % NS);  // tile t-1's stage
      const int64_t p_first = pf;
      if (t + 1 < t_end) pf = ldg64(P, (t + 1) * TILE);
      if (t == t_begin) {
        warp_lower_bound_pair(x.e, x.n, a_last, p_first, HAS_C ? c.e : nullptr, HAS_C ? c.n : 0, c_last,
                              p_first, a_cur, c_cur);
      } else {
        mbar_wait(&full[pst], ((t - 1 - t_begin) / NS) & 1);  // tile t-1 landed
        // C's predicate once per staged run of tile t-1 (the consumers read a
        // flag byte per point instead of comparing the value), then publish
        if (HAS_C)
          for (int i = lane; i < c_n; i += 32) sF(pst)[i] = c_smem_pass(c, sCv(pst), i) ? 1 : 0;
        mbar_arrive(&ready[pst]);
        const int ra = smem_lb_pow2<AW>(sA(pst), AW, p_first);
        int64_t an = a_lo16 + ra;
        if (ra >= a_n && an < x.n) an += warp_lower_bound(x.e + an, x.n - an, p_first);
        const int64_t ua = an - a_cur;  // runs spanned by tile t-1
        a_est = static_cast<int>(min(static_cast<int64_t>(AW), ua + (ua >> 2) + 32));
        a_cur = an;
        if (HAS_C) {
          const int rc = smem_lb_pow2<CW>(sC(pst), CW, p_first);
          int64_t cn = c_lo16 + rc;
          if (rc >= c_n && cn < c.n) cn += warp_lower_bound(c.e + cn, c.n - cn, p_first);
          const int64_t uc = cn - c_cur;
          c_est = static_cast<int>(min(static_cast<int64_t>(CW), uc + (uc >> 2) + 32));
          c_cur = cn;
        }
      }
      if (t - t_begin >= NS) mbar_wait(&empty[st], (use - 1) & 1);  // consumers done with tile t-NS
      // staged counts: whole 16-run chunks (< W), clipped at the column end
      auto stage_n = [](int64_t lo, int est, int W, int64_t total, int64_t& lo16) {
        lo16 = lo & ~int64_t(15);
        int64_t n = static_cast<int64_t>(est) + (lo - lo16);
        if (n > W - 16) n = W - 16;
        n = (n + 15) & ~int64_t(15);
        if (n > total - lo16) n = total - lo16;
        return n > 0 ? static_cast<int>(n) : 0;
      };
      a_n = stage_n(a_cur, a_est, AW, x.n, a_lo16);
      c_n = HAS_C ? stage_n(c_cur, c_est, CW, c.n, c_lo16) : 0;
      int64_t* wA = sA(st);
      int64_t* wC = sC(st);
      unsigned char* wCv = sCv(st);
      const int a_bulk = a_n & ~15, c_bulk = c_n & ~15;
      for (int i = a_bulk + lane; i < a_n; i += 32) wA[i] = ldg64(x.e, a_lo16 + i);
      int hwa = hwA[0], hwc = hwC[0];
#pragma unroll
      for (int i = 1; i < NS; ++i)
        if (st == i) hwa = hwA[i], hwc = hwC[i];
      for (int i = a_n + lane; i < hwa; i += 32) wA[i] = INT64_MAX;
      if (HAS_C) {
        for (int i = c_bulk + lane; i < c_n; i += 32) {
          wC[i] = ldg64(c.e, c_lo16 + i);
          const unsigned char* src = static_cast<const unsigned char*>(c.v) + (c_lo16 + i) * wc;
          for (int j = 0; j < wc; ++j) wCv[i * wc + j] = src[j];
        }
        for (int i = c_n + lane; i < hwc; i += 32) wC[i] = INT64_MAX;
      }
#pragma unroll
      for (int i = 0; i < NS; ++i)
        if (st == i) hwA[i] = a_n, hwC[i] = c_n;
      if (lane != 0) mbar_arrive(&full[st]);
      if (lane == 0) {
        s_lo[st][0] = a_lo16;
        s_n[st][0] = a_n;
        s_lo[st][1] = c_lo16;
        s_n[st][1] = c_n;
        const uint32_t ba = static_cast<uint32_t>(a_bulk) * 8u;
        const uint32_t bc = static_cast<uint32_t>(c_bulk) * 8u;
        const uint32_t bcv = static_cast<uint32_t>(c_bulk) * static_cast<uint32_t>(wc);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[st], ba + (HAS_C ? bc + bcv : 0u));
        if (ba) bulk_g2s(wA, x.e + a_lo16, ba, &full[st]);
        if (HAS_C && bc) {
          bulk_g2s(wC, c.e + c_lo16, bc, &full[st]);
          bulk_g2s(wCv, static_cast<const unsigned char*>(c.v) + c_lo16 * wc, bcv, &full[st]);
        }
      }
      __syncwarp();
    }
    if (t_begin < t_end) {  // the last tile's flags
      const int lst = static_cast<int>((t_end - 1 - t_begin) % NS);
      mbar_wait(&full[lst], ((t_end - 1 - t_begin) / NS) & 1);
      if (HAS_C)
        for (int i = lane; i < c_n; i += 32) sF(lst)[i] = c_smem_pass(c, sCv(lst), i) ? 1 : 0;
      mbar_arrive(&ready[lst]);
    }
  } else {
    // ---- consumer warps: ITEMS consecutive points per lane ---------------------
    const int i0 = ((wid - 1) * 32 + lane) * ITEMS;
    int64_t cur[ITEMS], nxt[ITEMS];
    if (t_begin < t_end) load_keys<BLOCK, ITEMS>(P, np, t_begin * TILE + i0, cur);
    for (int64_t t = t_begin; t < t_end; ++t) {
      const int st = static_cast<int>((t - t_begin) % NS);
      const uint32_t use = static_cast<uint32_t>((t - t_begin) / NS);
      const int64_t tbase = t * TILE;
      const int npt = static_cast<int>(np - tbase < TILE ? np - tbase : TILE);
      if (t + 1 < t_end) load_keys<BLOCK, ITEMS>(P, np, tbase + TILE + i0, nxt);
      mbar_wait(&ready[st], use & 1u);  // landed (the producer saw `full`) and flagged
      const int64_t a16 = s_lo[st][0], c16 = s_lo[st][1];
      const int na = s_n[st][0], nc = s_n[st][1];
      const int64_t* wA = sA(st);
      const int64_t* wC = sC(st);

      int ra[ITEMS], rc[ITEMS];
      {  // both windows searched in one unrolled loop: two independent chains
        int pa = 0, pc = 0;
#pragma unroll
        for (int step = AW / 2; step > 0; step >>= 1) {
          pa = wA[pa + step - 1] < cur[0] ? pa + step : pa;
          if (HAS_C && step < CW) pc = wC[pc + step - 1] < cur[0] ? pc + step : pc;
        }
        ra[0] = pa + (wA[pa] < cur[0] ? 1 : 0);
        if (HAS_C) rc[0] = pc + (wC[pc] < cur[0] ? 1 : 0);
      }
      // forward from the previous point: a branch-free search over the next 8
      // (A) / 4 (C) runs covers the usual gap between neighbouring points; the
      // loop runs only for longer gaps (rare, so warps seldom diverge). The pad
      // entries stop every scan.
#pragma unroll
      for (int k = 1; k < ITEMS; ++k) {
        int r = ra[k - 1];
        r = wA[r + 3] < cur[k] ? r + 4 : r;
        r = wA[r + 1] < cur[k] ? r + 2 : r;
        r = wA[r] < cur[k] ? r + 1 : r;
        while (wA[r] < cur[k]) ++r;
        ra[k] = r;
        if (HAS_C) {
          int q = rc[k - 1];
          q = wC[q + 1] < cur[k] ? q + 2 : q;
          q = wC[q] < cur[k] ? q + 1 : q;
          while (wC[q] < cur[k]) ++q;
          rc[k] = q;
        }
      }
      int64_t arun[ITEMS];
      bool take[ITEMS];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int64_t p = cur[k];
        int64_t ar = a16 + ra[k];
        if (ra[k] >= na && ar < x.n) ar = lb_window(x.e, ar, x.n, p);  // past the window
        arun[k] = ar;
        bool pass = i0 + k < npt && ar < x.n && (x.gapless || ldg64(x.s, ar) <= p);
        if (CK == C_PLAIN) {
          pass = pass && p < c.n && c_plain_pass(c, p);
        } else {
          int64_t cr = c16 + rc[k];
          if (rc[k] >= nc) {
            if (cr < c.n) cr = lb_window(c.e, cr, c.n, p);
            pass = pass && cr < c.n && (CK == C_RLE_GAPLESS || ldg64(c.s, cr) <= p) && c_run_pass(c, cr);
          } else {
            pass = pass && (CK == C_RLE_GAPLESS || ldg64(c.s, cr) <= p) && sF(st)[rc[k]];
          }
        }
        take[k] = pass;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // stage reads done (the gathers below are global)
      T xa[ITEMS], yb[ITEMS];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int64_t q = tbase + i0 + k;
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
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) cur[k] = nxt[k];
    }
  }
  if (lerr) atomicOr(err, 1);

  __shared__ uint64_t ru[BLOCK / 32 + 1];
  __shared__ double rf[BLOCK / 32 + 1];
  __shared__ uint64_t rn[BLOCK / 32 + 1];
  __shared__ bool last;
  isum = warp_sum(isum);
  fsum = warp_sum(fsum);
  uint64_t ucnt = warp_sum(static_cast<uint64_t>(cnt));
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
    parts[blockIdx.x] = pp;
    __threadfence();
    last = atomicInc(ticket, gridDim.x - 1) == gridDim.x - 1;  // wraps to 0 for the next launch
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last CTA folds every partial in a fixed order
  isum = 0;
  fsum = 0.0;
  ucnt = 0;
  for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += BLOCK) {
    isum += __ldcg(&parts[i].isum);
    fsum += __ldcg(&parts[i].fsum);
    ucnt += static_cast<uint64_t>(__ldcg(&parts[i].cnt));
  }
  isum = block_sum<BLOCK>(isum, ru);
  fsum = block_sum<BLOCK>(fsum, rf);
  ucnt = block_sum<BLOCK>(ucnt, rn);
  if (threadIdx.x == 0) {
    AggPart pp{};
    pp.isum = isum;
    pp.fsum = fsum;
    pp.cnt = static_cast<long long>(ucnt);
    pp.imin = atomicExch(err, 0);  // error flag travels with the result; reset for the next launch
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

// ---- persistent TMA path ----
// (overridable at build time for A/B sweeps: -DRQ_C2_TB=… etc.)
#ifndef RQ_C2_TB
#define RQ_C2_TB 256
#endif
#ifndef RQ_C2_TI
#define RQ_C2_TI 4
#endif
#ifndef RQ_C2_TAW
#define RQ_C2_TAW 2048
#endif
#ifndef RQ_C2_TCW
#define RQ_C2_TCW 512
#endif
#ifndef RQ_C2_TNS
#define RQ_C2_TNS 2
#endif
#ifndef RQ_C2_MINB
#define RQ_C2_MINB 4
#endif
constexpr int TB = RQ_C2_TB, TI = RQ_C2_TI, TAW = RQ_C2_TAW, TCW = RQ_C2_TCW;
constexpr int TNS = RQ_C2_TNS;  // 3 stages measured slower (3 CTAs/SM)
constexpr int TMINB = RQ_C2_MINB;
using TmaSmem = dev::C2Stage<TAW, TCW>;
constexpr size_t TMA_SMEM = TNS * TmaSmem::BYTES;

struct TmaLaunch {
  const DCol* y;
  dev::XSpec xs;
  dev::CSpec cs;
  int64_t ntiles;
  int swap;
  dev::AggPart* parts;
  unsigned* ticket;
  dev::AggPart* out;
  int* err;
};


template <class T, int OP, int CK>
int64_t launch_tma3(const CtxPtr& ctx, const TmaLaunch& f, bool dry) {
  const int32_t tdt = std::is_same<T, double>::value ? RQ_F64 : RQ_I64;
  const bool same = f.xs.dt == tdt && f.y->v.dt == tdt;
  auto k_same = dev::k_points_filtered_reduce_tma<TB, TI, TAW, TCW, TNS, T, OP, CK, true, TMINB>;
  auto k_gen = dev::k_points_filtered_reduce_tma<TB, TI, TAW, TCW, TNS, T, OP, CK, false, TMINB>;
  const int occ = kernel_occupancy(ctx, same ? k_same : k_gen, TB, TMA_SMEM);
  int64_t grid = static_cast<int64_t>(ctx->sm_count) * occ;
  if (grid > f.ntiles) grid = f.ntiles;
  if (dry) return grid;
  (same ? k_same : k_gen)<<<static_cast<unsigned>(grid), TB, TMA_SMEM, ctx->stream>>>(
      f.y->p.pos(), f.y->v.raw(), f.y->v.dt, f.y->p.n, f.xs, f.cs, f.ntiles, f.swap, f.parts, f.ticket,
      f.out, f.err);
  return grid;
}

template <class T, int OP>
int64_t launch_tma2(int ck, const CtxPtr& ctx, const TmaLaunch& f, bool dry) {
  switch (ck) {
    case dev::C_RLE_GAPLESS: return launch_tma3<T, OP, dev::C_RLE_GAPLESS>(ctx, f, dry);
    case dev::C_RLE_GAPPED: return launch_tma3<T, OP, dev::C_RLE_GAPPED>(ctx, f, dry);
    default: return launch_tma3<T, OP, dev::C_PLAIN>(ctx, f, dry);
  }
}

template <class T>
int64_t launch_tma1(int op, int ck, const CtxPtr& ctx, const TmaLaunch& f, bool dry) {
  switch (op) {
    case RQ_ADD: return launch_tma2<T, RQ_ADD>(ck, ctx, f, dry);
    case RQ_SUB: return launch_tma2<T, RQ_SUB>(ck, ctx, f, dry);
    case RQ_MUL: return launch_tma2<T, RQ_MUL>(ck, ctx, f, dry);
    default: return launch_tma2<T, RQ_DIV>(ck, ctx, f, dry);
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
  const bool use_tma = tma_ok(y.p) && tma_ok(y.v) && tma_ok(x.e) &&
                       (ck == dev::C_PLAIN || (tma_ok(c.e) && tma_ok(c.v)));
  if (np > 0 && xs.n > 0 && cs.n > 0 && use_tma) {
    constexpr int64_t TILE = static_cast<int64_t>(TB - 32) * TI;  // warp 0 produces
    const int64_t ntiles = (np + TILE - 1) / TILE;
    TmaLaunch f{&y, xs, cs, ntiles, a.enc == RQ_ENC_RLE ? 0 : 1, nullptr, ctx->tickets, nullptr, nullptr};
    const int64_t grid = flt ? launch_tma1<double>(op, ck, ctx, f, true) : launch_tma1<int64_t>(op, ck, ctx, f, true);
    // per-CTA partials in the context's scratch; the last CTA writes the
    // folded result straight into mapped pinned host memory
    f.parts = static_cast<dev::AggPart*>(ctx->get_scratch(static_cast<size_t>(grid) * sizeof(dev::AggPart)));
    f.out = static_cast<dev::AggPart*>(ctx->result_dev);
    f.err = reinterpret_cast<int*>(ctx->tickets + 1);  // zero between launches (the kernel resets it)
    {
      KTimer timer(ctx, "filtered_points_reduce");
      if (flt) launch_tma1<double>(op, ck, ctx, f, false);
      else launch_tma1<int64_t>(op, ck, ctx, f, false);
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
    }
    ctx->sync();
    std::memcpy(&res, ctx->result_host, sizeof(res));
    if (!flt && op == RQ_DIV && res.imin) fail("integer division by zero");
  } else if (np > 0 && xs.n > 0 && cs.n > 0) {
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
