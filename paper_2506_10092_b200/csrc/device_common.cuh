// device_common.cuh — device building blocks shared by the sm_100a kernels:
// dtype-tagged value loads, the reference's arithmetic/comparison semantics,
// warp/block scans and reductions, single-pass decoupled look-back, and
// merge-path partitioning (the data-parallel replacement for the
// reference's bucketize/repeat_interleave pipeline, kernels.cpp:10-60).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/runq_b200.h"

namespace rqb {
namespace dev {

constexpr unsigned FULL = 0xffffffffu;
constexpr int64_t KEY_MAX = INT64_MAX;

// ---- dtype-tagged loads (runq::Array::to_i64 / to_f64, array.cpp:44-61) ---------

__device__ __forceinline__ bool dt_is_float_dev(int dt) { return dt == RQ_F32 || dt == RQ_F64; }
__device__ __forceinline__ int dt_width_dev(int dt) {
  return dt == RQ_I8 ? 1 : dt == RQ_I16 ? 2 : (dt == RQ_I32 || dt == RQ_F32) ? 4 : 8;
}

__device__ __forceinline__ int64_t ld_i64(const void* p, int dt, int64_t i) {
  switch (dt) {
    case RQ_I8: return static_cast<const int8_t*>(p)[i];
    case RQ_I16: return static_cast<const int16_t*>(p)[i];
    case RQ_I32: return static_cast<const int32_t*>(p)[i];
    case RQ_I64: return __ldg(static_cast<const long long*>(p) + i);
    case RQ_F32: return static_cast<int64_t>(static_cast<const float*>(p)[i]);
    default: return static_cast<int64_t>(static_cast<const double*>(p)[i]);
  }
}

__device__ __forceinline__ double ld_f64(const void* p, int dt, int64_t i) {
  switch (dt) {
    case RQ_I8: return static_cast<double>(static_cast<const int8_t*>(p)[i]);
    case RQ_I16: return static_cast<double>(static_cast<const int16_t*>(p)[i]);
    case RQ_I32: return static_cast<double>(static_cast<const int32_t*>(p)[i]);
    case RQ_I64: return static_cast<double>(__ldg(static_cast<const long long*>(p) + i));
    case RQ_F32: return static_cast<double>(static_cast<const float*>(p)[i]);
    default: return __ldg(static_cast<const double*>(p) + i);
  }
}

template <class T>
__device__ __forceinline__ T ld_as(const void* p, int dt, int64_t i);
template <>
__device__ __forceinline__ int64_t ld_as<int64_t>(const void* p, int dt, int64_t i) {
  return ld_i64(p, dt, i);
}
template <>
__device__ __forceinline__ double ld_as<double>(const void* p, int dt, int64_t i) {
  return ld_f64(p, dt, i);
}

// Wrap an int64 to a narrower logical width (static_cast<T> in
// column.cpp:289-294 decode).
__device__ __forceinline__ int64_t wrap_to(int dt, int64_t x) {
  switch (dt) {
    case RQ_I8: return static_cast<int8_t>(static_cast<uint8_t>(x));
    case RQ_I16: return static_cast<int16_t>(static_cast<uint16_t>(x));
    case RQ_I32: return static_cast<int32_t>(static_cast<uint32_t>(x));
    default: return x;
  }
}

// ---- operator semantics (align.cpp:290-318: apply_arith / apply_cmp) -------------

// Integer arithmetic wraps modulo 2^64 (unsigned) so results are bit-exact
// regardless of evaluation order. Division by zero sets *err (the reference
// throws runq::Error "integer division by zero", align.cpp:297-299).
__device__ __forceinline__ int64_t arith_i64(int64_t x, int64_t y, int op, int* err) {
  switch (op) {
    case RQ_ADD: return static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(y));
    case RQ_SUB: return static_cast<int64_t>(static_cast<uint64_t>(x) - static_cast<uint64_t>(y));
    case RQ_MUL: return static_cast<int64_t>(static_cast<uint64_t>(x) * static_cast<uint64_t>(y));
    default:
      if (y == 0) {
        if (err) *err = 1;
        return 0;
      }
      if (x == INT64_MIN && y == -1) return INT64_MIN;  // wraps like two's complement
      return x / y;
  }
}
__device__ __forceinline__ double arith_f64(double x, double y, int op, int*) {
  switch (op) {
    case RQ_ADD: return x + y;
    case RQ_SUB: return x - y;
    case RQ_MUL: return x * y;
    default: return x / y;  // IEEE inf/nan
  }
}
template <class T>
__device__ __forceinline__ T arith_t(T x, T y, int op, int* err);
template <>
__device__ __forceinline__ int64_t arith_t<int64_t>(int64_t x, int64_t y, int op, int* err) {
  return arith_i64(x, y, op, err);
}
template <>
__device__ __forceinline__ double arith_t<double>(double x, double y, int op, int* err) {
  return arith_f64(x, y, op, err);
}

template <class T>
__device__ __forceinline__ bool cmp_t(T x, T y, int op) {
  switch (op) {
    case RQ_LT: return x < y;
    case RQ_LE: return x <= y;
    case RQ_EQ: return x == y;
    case RQ_NE: return x != y;
    case RQ_GE: return x >= y;
    default: return x > y;
  }
}

// ---- warp / block primitives ------------------------------------------------------

template <class T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}
template <class T>
__device__ __forceinline__ T warp_min(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T y = __shfl_xor_sync(FULL, x, o);
    x = y < x ? y : x;
  }
  return x;
}
template <class T>
__device__ __forceinline__ T warp_max(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T y = __shfl_xor_sync(FULL, x, o);
    x = y > x ? y : x;
  }
  return x;
}

// inclusive warp scan
template <class T>
__device__ __forceinline__ T warp_inclusive(T x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Block-wide exclusive scan. `warp_tot` must hold BLOCK/32 elements.
template <int BLOCK, class T>
__device__ __forceinline__ T block_exclusive(T x, T& total, T* warp_tot) {
  constexpr int NW = BLOCK / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = warp_inclusive(x);
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T w = lane < NW ? warp_tot[lane] : T(0);
    T wi = warp_inclusive(w);
    if (lane < NW) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == NW - 1) warp_tot[NW] = wi;   // block total (needs NW+1 slots)
  }
  __syncthreads();
  total = warp_tot[NW];
  T res = warp_tot[wid] + inc - x;
  __syncthreads();
  return res;
}

// Block sum; result valid in every thread. `red` must hold BLOCK/32 + 1.
template <int BLOCK, class T>
__device__ __forceinline__ T block_sum(T x, T* red) {
  constexpr int NW = BLOCK / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  x = warp_sum(x);
  if (lane == 0) red[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T w = lane < NW ? red[lane] : T(0);
    w = warp_sum(w);
    if (lane == 0) red[NW] = w;
  }
  __syncthreads();
  T r = red[NW];
  __syncthreads();
  return r;
}

// ---- single-pass decoupled look-back (Merrill & Garland) -----------------------------
//
// Status word: [63:62] flag (1 = tile aggregate, 2 = inclusive prefix),
// [61:40] launch epoch (so the status buffer never needs zeroing between
// launches), [39:0] value (counts up to 2^40).
struct LookBack {
  unsigned long long* status;
  uint32_t epoch;

  static constexpr uint64_t VMASK = (1ull << 40) - 1;

  __device__ __forceinline__ unsigned long long pack(uint64_t flag, uint64_t v) const {
    return (flag << 62) | ((static_cast<uint64_t>(epoch) & 0x3fffffull) << 40) | (v & VMASK);
  }
  __device__ __forceinline__ int flag_of(unsigned long long w) const {
    if (((w >> 40) & 0x3fffffull) != (epoch & 0x3fffffu)) return 0;
    return static_cast<int>(w >> 62);
  }
  __device__ __forceinline__ void store(int tile, unsigned long long w) const {
    atomicExch(status + tile, w);
  }
  __device__ __forceinline__ unsigned long long load(int tile) const {
    return *reinterpret_cast<volatile unsigned long long*>(status + tile);
  }

  // Called by all 32 lanes of ONE warp. Returns the exclusive prefix of
  // `tile` (sum of the aggregates of tiles < tile) and publishes this tile's
  // inclusive prefix.
  __device__ uint64_t exclusive(int tile, uint64_t aggregate) const {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
      if (lane == 0) store(0, pack(2, aggregate));
      return 0;
    }
    if (lane == 0) store(tile, pack(1, aggregate));
    uint64_t excl = 0;
    int pred = tile - 1;
    while (true) {
      const int t = pred - lane;
      int flag = 2;
      uint64_t val = 0;
      if (t >= 0) {
        unsigned long long w;
        do {
          w = load(t);
          flag = flag_of(w);
        } while (flag == 0);
        val = w & VMASK;
      }
      const unsigned inc = __ballot_sync(FULL, flag == 2);
      const int stop = inc ? (__ffs(inc) - 1) : 32;
      if (lane > stop) val = 0;
      excl += warp_sum(val);
      if (inc) break;
      pred -= 32;
    }
    if (lane == 0) store(tile, pack(2, excl + aggregate));
    return excl;
  }
};

// ---- merge path -------------------------------------------------------------------
//
// For the merge of sorted A and B where ties take A first (A[i] <= B[j] ⇒ A[i]
// precedes B[j]), returns how many A elements precede diagonal `diag`.
template <class FA, class FB>
__device__ __forceinline__ int64_t merge_path(FA a, int64_t na, FB b, int64_t nb, int64_t diag) {
  int64_t lo = diag > nb ? diag - nb : 0;
  int64_t hi = diag < na ? diag : na;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a(mid) <= b(diag - 1 - mid)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Warp-cooperative 32-ary version of merge_path (one warp per diagonal):
// ~log32(n) rounds of two independent loads per lane instead of log2(n)
// dependent loads. All lanes return the same value.
__device__ __forceinline__ int64_t warp_merge_path(const int64_t* __restrict__ A, int64_t na,
                                                   const int64_t* __restrict__ B, int64_t nb,
                                                   int64_t diag) {
  const int lane = threadIdx.x & 31;
  int64_t lo = diag > nb ? diag - nb : 0;
  int64_t hi = diag < na ? diag : na;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int64_t span = hi - lo;
    const int64_t step = (span + 31) / 32;
    int64_t x = lo + (static_cast<int64_t>(lane) + 1) * step - 1;
    if (x > hi - 1) x = hi - 1;
    const bool pred = __ldg(reinterpret_cast<const long long*>(A) + x) <=
                      __ldg(reinterpret_cast<const long long*>(B) + (diag - 1 - x));
    const unsigned bal = __ballot_sync(FULL, pred);
    const int c = __popc(bal);  // predicate is monotone: true for lanes < c
    const int64_t nlo = c == 0 ? lo : __shfl_sync(FULL, x, c - 1) + 1;
    const int64_t nhi = c == 32 ? hi : __shfl_sync(FULL, x, c);
    lo = nlo;
    hi = nhi;
  }
  const int64_t x = lo + lane;
  bool pred = false;
  if (x < hi)
    pred = __ldg(reinterpret_cast<const long long*>(A) + x) <=
           __ldg(reinterpret_cast<const long long*>(B) + (diag - 1 - x));
  return lo + __popc(__ballot_sync(FULL, pred));
}

// Warp-cooperative 32-ary lower_bound (first index with a[i] >= key).
__device__ __forceinline__ int64_t warp_lower_bound(const int64_t* __restrict__ a, int64_t n,
                                                    int64_t key) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    int64_t x = lo + (static_cast<int64_t>(lane) + 1) * step - 1;
    if (x > hi - 1) x = hi - 1;
    const bool pred = __ldg(reinterpret_cast<const long long*>(a) + x) < key;
    const int c = __popc(__ballot_sync(FULL, pred));
    const int64_t nlo = c == 0 ? lo : __shfl_sync(FULL, x, c - 1) + 1;
    const int64_t nhi = c == 32 ? hi : __shfl_sync(FULL, x, c);
    lo = nlo;
    hi = nhi;
  }
  const int64_t x = lo + lane;
  const bool pred = x < hi && __ldg(reinterpret_cast<const long long*>(a) + x) < key;
  return lo + __popc(__ballot_sync(FULL, pred));
}

// One narrowing round of a 32-ary warp search: lane splitters x (monotone
// over lanes, inside [lo, hi)), answer kept in [lo, hi].
__device__ __forceinline__ void warp_lb_narrow(int64_t x, bool pred, int64_t& lo, int64_t& hi) {
  const int c = __popc(__ballot_sync(FULL, pred));
  const int64_t nlo = c == 0 ? lo : __shfl_sync(FULL, x, c - 1) + 1;
  const int64_t nhi = c == 32 ? hi : __shfl_sync(FULL, x, c);
  lo = nlo;
  hi = nhi;
}

// Splitter of lane `lane` for a 32-ary round over [lo, hi) (hi - lo > 32).
__device__ __forceinline__ int64_t warp_lb_splitter(int64_t lo, int64_t hi, int lane) {
  const int64_t step = (hi - lo + 31) / 32;
  const int64_t x = lo + (static_cast<int64_t>(lane) + 1) * step - 1;
  return x > hi - 1 ? hi - 1 : x;
}

// First round of an interpolation search: splitters spaced S apart around
// the position the key would have if the ends were evenly spread over
// [0, last] (run ends of a synthetic or real column are close to that), so
// a typical answer is bracketed to S entries in one load latency; any key
// still lands in a correct [lo, hi] (the outer brackets), only slower.
__device__ __forceinline__ int64_t warp_lb_interp_splitter(int64_t n, int64_t last, int64_t key,
                                                           int lane) {
  const int64_t S = max(int64_t(1), min(int64_t(1024), n >> 14));
  double f = last >= 0 ? static_cast<double>(key) / (static_cast<double>(last) + 1.0) : 0.0;
  f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
  const int64_t g = static_cast<int64_t>(f * static_cast<double>(n));
  int64_t x = g + (static_cast<int64_t>(lane) - 16) * S;
  return x < 0 ? 0 : (x > n - 1 ? n - 1 : x);
}

// Two independent warp lower_bounds (first index with a[i] >= ka, b[i] >= kb)
// advanced in lockstep so every round issues both lists' loads together:
// an interpolation round (the last end of each list, loaded beside the keys by
// the caller, places the splitters), then 32-ary rounds. CTA start-up cost of
// the persistent kernels: ~4 load latencies instead of ~11 for two sequential
// 32-ary searches. nb == 0 (or b == nullptr) searches only a.
__device__ __forceinline__ void warp_lower_bound_pair(const int64_t* __restrict__ a, int64_t na,
                                                      int64_t a_last, int64_t ka,
                                                      const int64_t* __restrict__ b, int64_t nb,
                                                      int64_t b_last, int64_t kb, int64_t& ra,
                                                      int64_t& rb) {
  const int lane = threadIdx.x & 31;
  const auto* A = reinterpret_cast<const long long*>(a);
  const auto* B = reinterpret_cast<const long long*>(b);
  int64_t alo = 0, ahi = na, blo = 0, bhi = b ? nb : 0;
  if (ahi > 32 || bhi > 32) {  // interpolation round
    const bool ua = ahi > 32, ub = bhi > 32;
    const int64_t xa = ua ? warp_lb_interp_splitter(na, a_last, ka, lane) : 0;
    const int64_t xb = ub ? warp_lb_interp_splitter(nb, b_last, kb, lane) : 0;
    const bool pa = ua && __ldg(A + xa) < ka;
    const bool pb = ub && __ldg(B + xb) < kb;
    if (ua) warp_lb_narrow(xa, pa, alo, ahi);
    if (ub) warp_lb_narrow(xb, pb, blo, bhi);
  }
  while (ahi - alo > 32 || bhi - blo > 32) {
    const bool ua = ahi - alo > 32, ub = bhi - blo > 32;
    const int64_t xa = ua ? warp_lb_splitter(alo, ahi, lane) : 0;
    const int64_t xb = ub ? warp_lb_splitter(blo, bhi, lane) : 0;
    const bool pa = ua && __ldg(A + xa) < ka;
    const bool pb = ub && __ldg(B + xb) < kb;
    if (ua) warp_lb_narrow(xa, pa, alo, ahi);
    if (ub) warp_lb_narrow(xb, pb, blo, bhi);
  }
  const int64_t xa = alo + lane, xb = blo + lane;
  const bool pa = xa < ahi && __ldg(A + xa) < ka;
  const bool pb = xb < bhi && __ldg(B + xb) < kb;
  ra = alo + __popc(__ballot_sync(FULL, pa));
  rb = blo + __popc(__ballot_sync(FULL, pb));
}

// upper_bound / lower_bound over a sorted global int64 array
__device__ __forceinline__ int64_t upper_bound_g(const int64_t* __restrict__ a, int64_t n,
                                                 int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(reinterpret_cast<const long long*>(a) + mid) <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t lower_bound_g(const int64_t* __restrict__ a, int64_t n,
                                                 int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(reinterpret_cast<const long long*>(a) + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t ldg64(const int64_t* p, int64_t i) {
  return __ldg(reinterpret_cast<const long long*>(p) + i);
}

// ---- TMA 1-D bulk copies (cp.async.bulk → UBLKCP) completing on an mbarrier ----
// Source and destination 16-B aligned, size a multiple of 16 B. A CTA launched
// without a cluster is its own cluster, so the shared::cluster destination
// form addresses this CTA's shared memory.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// orders this thread's generic-proxy shared-memory accesses before later
// async-proxy (bulk copy) writes to the same bytes
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// raises the transaction count of the current phase without arriving
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// waits with a short sleep between probes so that waiting warps do not
// take issue slots from the warps that are working
#ifndef RQ_MBAR_MAXSLEEP
#define RQ_MBAR_MAXSLEEP 32  // A/B on C2: 0.1188 vs 0.1193 ms at 256 (3 of 3 runs), C1 even
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  unsigned ns = 32;
  while (!mbar_try_wait(bar, parity)) {
    __nanosleep(ns);
    ns = ns < RQ_MBAR_MAXSLEEP ? ns * 2 : RQ_MBAR_MAXSLEEP;
  }
}

// lower_bound over a shared-memory window padded with INT64_MAX up to the
// power of two L (uniform per CTA; L <= CAP): log2(L) steps of
// load / compare / select / add, no bounds tests
template <int CAP>
__device__ __forceinline__ int smem_lb_pow2(const int64_t* a, int L, int64_t key) {
  int pos = 0;
#pragma unroll
  for (int step = CAP / 2; step > 0; step >>= 1)
    if (step < L) pos = a[pos + step - 1] < key ? pos + step : pos;
  return pos + (a[pos] < key ? 1 : 0);
}
__device__ __forceinline__ int pow2_above(int n) {  // smallest power of two > n (n >= 0)
  return n > 0 ? 1 << (32 - __clz(n)) : 1;
}

// Branch-free lower_bound over a shared-memory array of n >= 1 sorted int64
// (first index with a[i] >= key, n if none). The trip count depends on n
// only, so every lane of a CTA runs the same steps; no padding is needed.
__device__ __forceinline__ int smem_lower_bound(const int64_t* a, int n, int64_t key) {
  int base = 0;
  while (n > 1) {
    const int half = n >> 1;
    base = a[base + half] < key ? base + half : base;
    n -= half;
  }
  return base + (a[base] < key ? 1 : 0);
}

// Warp-cooperative lower_bound over n <= 1024 sorted shared-memory int64
// (all 32 lanes, same key; entries past the valid ones padded with
// INT64_MAX): 32 evenly spaced probes and a ballot pick the block, a second
// ballot over the block's <= 32 entries gives the rank. Two dependent
// shared-memory rounds instead of log2(n).
__device__ __forceinline__ int warp_smem_lower_bound(const int64_t* a, int n, int64_t key) {
  const int lane = threadIdx.x & 31;
  const int step = (n + 31) >> 5;
  const int probe = min((lane + 1) * step, n) - 1;
  const int c = __popc(__ballot_sync(FULL, a[probe] < key));
  const int base = c * step;
  const int i = base + lane;
  return base + __popc(__ballot_sync(FULL, lane < step && i < n && a[i] < key));
}

}  // namespace dev
}  // namespace rqb
