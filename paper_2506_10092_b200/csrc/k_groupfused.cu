// k_groupfused.cu — K10 fused group-by over RLE dictionary-code keys.
//
// agg::group_aggregate (groupby.cpp:144-162) left-fold aligns keys and every
// data column onto one shape (align_many, align.cpp:233-254 — per-row when
// any input is plain) and then sorts slots (unique_with_inverse,
// kernels.cpp:127-187). When every input covers every row, each aggregate
// only depends on (key, value) per covered row, so each data column is
// aligned with the key runs alone ("per-aggregate minimal alignment",
// SURVEY.md §7 hard part 5) and folded straight into a dense group table
// indexed by slot = key − min (ascending slot order = ascending key order):
//   * RLE data       — merge-path walk over (key run ends, data run ends),
//                      value·fragment length per step (K2 walk, K5 shape)
//   * plain data     — warp-segment row kernel: 128-bit loads, inline
//                      bit-width-reduced decode (K9), warp-uniform key-run
//                      cursor, register accumulation flushed per key run
//   * index data     — the same warp-segment kernel over point positions
//   * RLE+Index      — its runs part (walk) + points part (points kernel)
//   * Plain+Index    — base (plain kernel) + per-outlier correction
// COUNT and group presence come from the key runs alone (Σ run lengths per
// slot). Tables are per-CTA shared memory when they fit, global otherwise;
// integer sums wrap like the reference's int64 accumulators.
#include <algorithm>
#include <cmath>
#include <memory>
#include <cstdlib>
#include <limits>

#include "merge_walk.cuh"
#include "rq_internal.hpp"
#include "xg_plan.hpp"

namespace rqb {
namespace dev {

enum GKind { G_SUM_I = 0, G_SUM_F = 1, G_MIN_I = 2, G_MAX_I = 3, G_MIN_F = 4, G_MAX_F = 5, G_SQ = 6 };

template <int KIND>
struct GTraits;
template <> struct GTraits<G_SUM_I> { using T = int64_t; };
template <> struct GTraits<G_SUM_F> { using T = double; };
template <> struct GTraits<G_MIN_I> { using T = int64_t; };
template <> struct GTraits<G_MAX_I> { using T = int64_t; };
template <> struct GTraits<G_MIN_F> { using T = double; };
template <> struct GTraits<G_MAX_F> { using T = double; };
template <> struct GTraits<G_SQ> { using T = double; };

__device__ __forceinline__ void atomic_min_f(double* a, double v) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(a);
  unsigned long long old = *p;
  while (__longlong_as_double(old) > v) {
    const unsigned long long prev = atomicCAS(p, old, __double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}
__device__ __forceinline__ void atomic_max_f(double* a, double v) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(a);
  unsigned long long old = *p;
  while (__longlong_as_double(old) < v) {
    const unsigned long long prev = atomicCAS(p, old, __double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}

template <int KIND>
__device__ __forceinline__ unsigned long long g_identity() {
  switch (KIND) {
    case G_MIN_I: return static_cast<unsigned long long>(INT64_MAX);
    case G_MAX_I: return static_cast<unsigned long long>(INT64_MIN);
    case G_MIN_F: return 0x7ff0000000000000ull;  // +inf
    case G_MAX_F: return 0xfff0000000000000ull;  // -inf
    default: return 0ull;
  }
}

template <int KIND>
__device__ __forceinline__ typename GTraits<KIND>::T g_zero() {
  using T = typename GTraits<KIND>::T;
  switch (KIND) {
    case G_MIN_I: return static_cast<T>(INT64_MAX);
    case G_MAX_I: return static_cast<T>(INT64_MIN);
    case G_MIN_F: return static_cast<T>(INFINITY);
    case G_MAX_F: return static_cast<T>(-INFINITY);
    default: return T(0);
  }
}

// fold one (value, weight) into a register accumulator
template <int KIND>
__device__ __forceinline__ void g_fold(typename GTraits<KIND>::T& acc, typename GTraits<KIND>::T v,
                                       int64_t w, double mean) {
  if (KIND == G_SUM_I)
    acc = static_cast<int64_t>(static_cast<uint64_t>(acc) + static_cast<uint64_t>(v) * static_cast<uint64_t>(w));
  else if (KIND == G_SUM_F) acc += static_cast<double>(v) * static_cast<double>(w);
  else if (KIND == G_MIN_I || KIND == G_MIN_F) acc = v < acc ? v : acc;
  else if (KIND == G_MAX_I || KIND == G_MAX_F) acc = v > acc ? v : acc;
  else {
    const double d = static_cast<double>(v) - mean;
    acc += d * d * static_cast<double>(w);
  }
}

template <int KIND>
__device__ __forceinline__ typename GTraits<KIND>::T g_combine(typename GTraits<KIND>::T a,
                                                               typename GTraits<KIND>::T b) {
  if (KIND == G_SUM_I) return static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
  if (KIND == G_MIN_I || KIND == G_MIN_F) return b < a ? b : a;
  if (KIND == G_MAX_I || KIND == G_MAX_F) return b > a ? b : a;
  return a + b;
}

// merge a register accumulator into a table slot (shared or global)
template <int KIND>
__device__ __forceinline__ void g_atomic(unsigned long long* tab, int64_t slot, typename GTraits<KIND>::T v) {
  if (KIND == G_SUM_I) atomicAdd(tab + slot, static_cast<unsigned long long>(v));
  else if (KIND == G_SUM_F || KIND == G_SQ) atomicAdd(reinterpret_cast<double*>(tab) + slot, static_cast<double>(v));
  else if (KIND == G_MIN_I) atomicMin(reinterpret_cast<long long*>(tab) + slot, static_cast<long long>(v));
  else if (KIND == G_MAX_I) atomicMax(reinterpret_cast<long long*>(tab) + slot, static_cast<long long>(v));
  else if (KIND == G_MIN_F) atomic_min_f(reinterpret_cast<double*>(tab) + slot, static_cast<double>(v));
  else atomic_max_f(reinterpret_cast<double*>(tab) + slot, static_cast<double>(v));
}

// per-CTA table: shared memory when G fits, else straight to global
struct GTable {
  unsigned long long* g;  // global table (G slots)
  int64_t G;
  int64_t kmin;
  // f64 sums (G_SUM_F / G_SQ): each warp adds into its own row part[warp * G]
  // in its fixed item order, the rows are folded in warp order afterwards
  // (k_gk_pfold) — the same bits on every run. Null: atomics.
  double* part = nullptr;
};

template <int KIND>
__device__ __forceinline__ constexpr bool g_fsum() {
  return KIND == G_SUM_F || KIND == G_SQ;
}

constexpr int kSmemSlots = 4096;

template <int KIND>
__device__ __forceinline__ unsigned long long* g_table_begin(unsigned long long* smem, const GTable& t) {
  if (t.G > kSmemSlots || (g_fsum<KIND>() && t.part)) return t.g;
  for (int64_t s = threadIdx.x; s < t.G; s += blockDim.x) smem[s] = g_identity<KIND>();
  __syncthreads();
  return smem;
}

template <int KIND>
__device__ __forceinline__ void g_table_end(unsigned long long* smem, const GTable& t) {
  if (t.G > kSmemSlots || (g_fsum<KIND>() && t.part)) return;
  __syncthreads();
  using T = typename GTraits<KIND>::T;
  const unsigned long long idn = g_identity<KIND>();
  for (int64_t s = threadIdx.x; s < t.G; s += blockDim.x) {
    const unsigned long long bits = smem[s];
    if (bits == idn) continue;
    T v;
    if (KIND == G_SUM_I || KIND == G_MIN_I || KIND == G_MAX_I) v = static_cast<T>(static_cast<long long>(bits));
    else v = static_cast<T>(__longlong_as_double(bits));
    g_atomic<KIND>(t.g, s, v);
  }
}

// value sources --------------------------------------------------------------


template <class T>
__device__ __forceinline__ T plain_value(const PlainSrc& s, int64_t row) {
  if (s.flt) return static_cast<T>(ld_f64(s.v, s.dt, row));
  int64_t x = wrap_to(s.logical, ld_i64(s.v, s.dt, row));
  if (s.has_center)
    x = wrap_to(s.logical, static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(s.center)));
  return static_cast<T>(x);
}

// COUNT / presence: Σ key run lengths per slot
__global__ void k_gk_count(const int64_t* __restrict__ ks, const int64_t* __restrict__ ke,
                           const void* __restrict__ kv, int kdt, int64_t nk, GTable t) {
  __shared__ unsigned long long smem[kSmemSlots];
  unsigned long long* tab = g_table_begin<G_SUM_I>(smem, t);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nk;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t len = ldg64(ke, i) - ldg64(ks, i) + 1;
    atomicAdd(tab + (ld_i64(kv, kdt, i) - t.kmin), static_cast<unsigned long long>(len));
  }
  g_table_end<G_SUM_I>(smem, t);
}

// RLE data: merge walk over (key ends A, data ends B). Key runs may have
// gaps only where the data has no rows (uniform coverage, checked on host).
template <int BLOCK, int ITEMS, int KIND>
__global__ void __launch_bounds__(BLOCK)
    k_gk_rle(MergeArgs m, const int64_t* __restrict__ kst, const void* __restrict__ kv, int kdt,
             const int64_t* __restrict__ ds, const void* __restrict__ dv, int ddt, GTable t,
             const double* __restrict__ mean) {
  using T = typename GTraits<KIND>::T;
  using Tile = MergeTile<BLOCK, ITEMS>;
  __shared__ int64_t sk[Tile::TILE];
  __shared__ unsigned long long smem[kSmemSlots];
  unsigned long long* tab = g_table_begin<KIND>(smem, t);
  Tile tl;
  tl.load(m, blockIdx.x, sk);
  T acc = g_zero<KIND>();
  int64_t cur = -1;  // current slot
  double mu = 0.0;
  // deterministic f64 mode: this thread's flushes, in walk order (at most one
  // per merge item plus the last), combined by the warp in lane order below
  constexpr int NREC = g_fsum<KIND>() ? ITEMS + 1 : 1;
  int64_t rslot[NREC];
  T racc[NREC];
  int nrec = 0;
  const bool det = g_fsum<KIND>() && t.part;
  auto flush = [&](int64_t sl, T a) {
    if (det) {
      rslot[nrec < NREC ? nrec : NREC - 1] = sl;
      racc[nrec < NREC ? nrec : NREC - 1] = a;
      ++nrec;
    } else {
      g_atomic<KIND>(tab, sl, a);
    }
  };
  tl.walk(sk, [&](int64_t i, int64_t j, bool takeA, int64_t key) {
    if (i >= m.na || j >= m.nb) return;
    // key run i starts after key run i-1's end; data run j starts at ds[j]
    const int64_t ks = ldg64(kst, i);
    const int64_t lo = max(ks, ldg64(ds, j));
    const int64_t len = key - lo + 1;
    if (len <= 0) return;
    const int64_t slot = ld_i64(kv, kdt, i) - t.kmin;
    if (slot != cur) {
      if (cur >= 0) flush(cur, acc);
      acc = g_zero<KIND>();
      cur = slot;
      if (KIND == G_SQ) mu = mean[slot];
    }
    g_fold<KIND>(acc, ld_as<T>(dv, ddt, j), len, mu);
  });
  if (cur >= 0) flush(cur, acc);
  if (det) {
    // lane 0 walks the warp's records in (lane, record) order, adding runs of
    // one slot in a register and each finished run into the warp's row
    const int lane = threadIdx.x & 31;
    double* row = t.part + ((static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x) >> 5) * t.G;
    int64_t cs = -1;
    double ca = 0.0;
    for (int l = 0; l < 32; ++l) {
      const int nl = __shfl_sync(FULL, nrec, l);
#pragma unroll
      for (int r = 0; r < NREC; ++r) {
        const int64_t sl = __shfl_sync(FULL, rslot[r], l);
        const double a = __shfl_sync(FULL, static_cast<double>(racc[r]), l);
        if (lane == 0 && r < nl) {
          if (sl != cs) {
            if (cs >= 0) row[cs] += ca;
            cs = sl;
            ca = 0.0;
          }
          ca += a;
        }
      }
    }
    if (lane == 0 && cs >= 0) row[cs] += ca;
  }
  g_table_end<KIND>(smem, t);
}

// Plain rows or index points: each warp owns a contiguous segment of items;
// per iteration lane l takes items [base + 8l, base + 8l + 8). A warp-uniform
// cursor over the (gapless) key runs tracks the run at the window start;
// windows inside one run take the fast path (pure register accumulation).
// eight consecutive storage values with one or more vector loads
template <class S>
__device__ __forceinline__ void load8(const S* __restrict__ p, S (&out)[8]) {
  constexpr int B = 8 * sizeof(S);
  if constexpr (B >= 16) {
    union {
      uint4 v[B / 16];
      S s[8];
    } u;
#pragma unroll
    for (int k = 0; k < B / 16; ++k) u.v[k] = __ldg(reinterpret_cast<const uint4*>(p) + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) out[k] = u.s[k];
  } else {
    union {
      uint2 v;
      S s[8];
    } u;
    u.v = __ldg(reinterpret_cast<const uint2*>(p));
#pragma unroll
    for (int k = 0; k < 8; ++k) out[k] = u.s[k];
  }
}

// bit-width-reduced decode of one storage value (column.cpp:283-297)
template <class T, class S>
__device__ __forceinline__ T plain_decode(const PlainSrc& s, S raw) {
  if constexpr (std::is_floating_point<S>::value) {
    return static_cast<T>(raw);
  } else {
    int64_t x = static_cast<int64_t>(raw);
    if (s.logical != RQ_I64) x = wrap_to(s.logical, x);
    if (s.has_center) {
      x = static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(s.center));
      if (s.logical != RQ_I64) x = wrap_to(s.logical, x);
    }
    return static_cast<T>(x);
  }
}

template <int KIND, bool POINTS, class S = int64_t>
__global__ void __launch_bounds__(256)
    k_gk_items(const int64_t* __restrict__ kst, const int64_t* __restrict__ ke, const void* __restrict__ kv,
               int kdt, int64_t nk,
               PlainSrc ps, const int64_t* __restrict__ pp, const void* __restrict__ pv, int pdt,
               int64_t n, int64_t seg, GTable t, const double* __restrict__ mean,
               const PlainSrc* corr) {
  using T = typename GTraits<KIND>::T;
  __shared__ unsigned long long smem[kSmemSlots];
  unsigned long long* tab = g_table_begin<KIND>(smem, t);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  constexpr int PER = 8, WIN = 32 * PER;
  const bool vec_pts = POINTS && (reinterpret_cast<uintptr_t>(pp) & 15) == 0 && (reinterpret_cast<uintptr_t>(pv) & 15) == 0;
  for (int64_t s0 = warp * seg; s0 < n; s0 += nwarps * seg) {
    const int64_t s1 = min(s0 + seg, n);
    // key run containing the segment's first position
    const int64_t pos0 = POINTS ? ldg64(pp, s0) : s0;
    int64_t kr = warp_lower_bound(ke, nk, pos0);
    int64_t kend = kr < nk ? ldg64(ke, kr) : INT64_MAX;
    int64_t slot = kr < nk ? ld_i64(kv, kdt, kr) - t.kmin : -1;
    double mu = (KIND == G_SQ && slot >= 0) ? mean[slot] : 0.0;
    T acc = g_zero<KIND>();
    for (int64_t b = s0; b < s1; b += WIN) {
      const int64_t i0 = b + lane * PER;
      int64_t pos[PER];
      T val[PER];
      if (!POINTS && i0 + PER <= s1 && (reinterpret_cast<uintptr_t>(ps.v) & 15) == 0) {
        // 8 rows of narrow storage per lane in one 64/128-bit load set, decoded in registers
        S raw[PER];
        load8<S>(static_cast<const S*>(ps.v) + i0, raw);
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          pos[u] = i0 + u;
          val[u] = plain_decode<T, S>(ps, raw[u]);
        }
      } else if (POINTS && i0 + PER <= s1 && vec_pts) {
        // 8 consecutive points per lane: 4 x 16-B loads of positions (and of
        // 8-byte values), instead of 8 strided scalar loads each
        load8<int64_t>(pp + i0, pos);
        if (pdt == RQ_I64 || pdt == RQ_F64) {
          int64_t raw[PER];
          load8<int64_t>(static_cast<const int64_t*>(pv) + i0, raw);
#pragma unroll
          for (int u = 0; u < PER; ++u)
            val[u] = pdt == RQ_I64 ? static_cast<T>(raw[u]) : static_cast<T>(__longlong_as_double(raw[u]));
        } else {
#pragma unroll
          for (int u = 0; u < PER; ++u) val[u] = ld_as<T>(pv, pdt, i0 + u);
        }
        if (corr) {
#pragma unroll
          for (int u = 0; u < PER; ++u) val[u] -= plain_value<T>(*corr, pos[u]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int64_t q = i0 + u;
          const bool ok = q < s1;
          if (POINTS) {
            pos[u] = ok ? ldg64(pp, q) : INT64_MAX;
            T x = ok ? ld_as<T>(pv, pdt, q) : T(0);
            if (corr && ok) x -= plain_value<T>(*corr, pos[u]);  // plain+index outlier correction
            val[u] = x;
          } else {
            pos[u] = ok ? q : INT64_MAX;
            val[u] = ok ? plain_value<T>(ps, q) : T(0);
          }
        }
      }
      // last valid position of the window (warp-wide)
      const int64_t qlast = min(b + WIN, s1) - 1;
      const int64_t plast = POINTS ? ldg64(pp, qlast) : qlast;
      if (plast <= kend) {  // fast path: whole window inside the current key run
#pragma unroll
        for (int u = 0; u < PER; ++u)
          if (pos[u] != INT64_MAX) g_fold<KIND>(acc, val[u], 1, mu);
        continue;
      }
      // slow path: walk the key runs overlapping the window (warp-uniform)
      int64_t kstart = kr < nk ? ldg64(kst, kr) : INT64_MAX;
      while (true) {
#pragma unroll
        for (int u = 0; u < PER; ++u)
          if (pos[u] >= kstart && pos[u] <= kend && pos[u] != INT64_MAX) g_fold<KIND>(acc, val[u], 1, mu);
        if (plast <= kend || kr >= nk) break;
        // run kr ends inside this window: flush the warp's partial for it
        T r = acc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = g_combine<KIND>(r, __shfl_xor_sync(FULL, r, o));
        if (lane == 0 && slot >= 0) {
          if (g_fsum<KIND>() && t.part) t.part[warp * t.G + slot] += static_cast<double>(r);
          else g_atomic<KIND>(tab, slot, r);
        }
        acc = g_zero<KIND>();
        ++kr;
        kstart = kr < nk ? ldg64(kst, kr) : INT64_MAX;
        kend = kr < nk ? ldg64(ke, kr) : INT64_MAX;
        slot = kr < nk ? ld_i64(kv, kdt, kr) - t.kmin : -1;
        if (KIND == G_SQ) mu = slot >= 0 ? mean[slot] : 0.0;
      }
    }
    T r = acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r = g_combine<KIND>(r, __shfl_xor_sync(FULL, r, o));
    if (lane == 0 && slot >= 0) {
      if (g_fsum<KIND>() && t.part) t.part[warp * t.G + slot] += static_cast<double>(r);
      else g_atomic<KIND>(tab, slot, r);
    }
  }
  g_table_end<KIND>(smem, t);
}

// the warps' rows of a deterministic f64 table folded per slot in warp order
__global__ void k_gk_pfold(const double* __restrict__ part, int64_t rows, int64_t G,
                           unsigned long long* __restrict__ tab) {
  __shared__ double red[256];
  const int64_t g = blockIdx.x;
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < rows; q += 256) acc += part[q * G + g];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) tab[g] = static_cast<unsigned long long>(__double_as_longlong(red[0]));
}

__global__ void k_gk_init(unsigned long long* __restrict__ t, int64_t G, unsigned long long v) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < G;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    t[s] = v;
}

__global__ void k_gk_mean(const unsigned long long* __restrict__ fsum, const unsigned long long* __restrict__ cnt,
                          int64_t G, double* __restrict__ mean) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < G;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    mean[s] = cnt[s] ? __longlong_as_double(fsum[s]) / static_cast<double>(cnt[s]) : 0.0;
}

__global__ void k_gk_flags(const unsigned long long* __restrict__ cnt, int64_t G, uint8_t* __restrict__ f) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < G;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    f[s] = cnt[s] > 0;
}

// results of present slots (groupby.cpp:67-135 conventions)
__global__ void k_gk_finish(const int64_t* __restrict__ slots, int64_t ng, int fn,
                            const unsigned long long* __restrict__ acc,
                            const unsigned long long* __restrict__ cnt,
                            const unsigned long long* __restrict__ sq, void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < ng;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = ldg64(slots, i);
    const double c = static_cast<double>(cnt[g]);
    switch (fn) {
      case RQ_COUNT: static_cast<long long*>(out)[i] = static_cast<long long>(cnt[g]); break;
      case RQ_AVG: static_cast<double*>(out)[i] = __longlong_as_double(acc[g]) / c; break;
      case RQ_VAR:
      case RQ_STD: {
        const double var = __longlong_as_double(sq[g]) / c;
        static_cast<double*>(out)[i] = fn == RQ_VAR ? var : sqrt(var);
        break;
      }
      default: static_cast<unsigned long long*>(out)[i] = acc[g];  // SUM / MIN / MAX bits
    }
  }
}

// slot -> key component: kmin_c + (slot / stride_c) % range_c
__global__ void k_gk_keys(const int64_t* __restrict__ slots, int64_t ng, int64_t kmin, int64_t stride,
                          int64_t range, int dt, void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < ng;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = kmin + (ldg64(slots, i) / stride) % range;
    switch (dt) {
      case RQ_I8: static_cast<int8_t*>(out)[i] = static_cast<int8_t>(k); break;
      case RQ_I16: static_cast<int16_t*>(out)[i] = static_cast<int16_t>(k); break;
      case RQ_I32: static_cast<int32_t*>(out)[i] = static_cast<int32_t>(k); break;
      default: static_cast<int64_t*>(out)[i] = k; break;
    }
  }
}

// composite key slot for aligned key runs: Σ (k_c - min_c) * stride_c
struct KeyCols {
  const void* v[8];
  int dt[8];
  int64_t mn[8];
  int64_t stride[8];
  int nk;
};
__global__ void k_gk_compose(KeyCols kc, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t s = 0;
    for (int c = 0; c < kc.nk; ++c) s += (ld_i64(kc.v[c], kc.dt[c], i) - kc.mn[c]) * kc.stride[c];
    out[i] = s;
  }
}

template <int BLOCK>
__global__ void k_gk_minmax(const void* __restrict__ v, int dt, int64_t n, long long* __restrict__ out) {
  int64_t mn = INT64_MAX, mx = INT64_MIN;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * BLOCK) {
    const int64_t x = ld_i64(v, dt, i);
    mn = x < mn ? x : mn;
    mx = x > mx ? x : mx;
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, static_cast<long long>(mn));
    atomicMax(out + 1, static_cast<long long>(mx));
  }
}

}  // namespace dev

namespace {

constexpr int64_t kFusedSlotLimit = int64_t{1} << 22;

int grid_cap(const CtxPtr& ctx, int64_t n, int block = 256, int per_sm = 8) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

void launched(const CtxPtr& ctx) {
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
}

bool full_cover(const CtxPtr& ctx, const DCol& c) {
  switch (c.enc) {
    case RQ_ENC_PLAIN:
    case RQ_ENC_PLAIN_INDEX: return true;
    case RQ_ENC_RLE: return col_gapless(ctx, c);
    case RQ_ENC_INDEX: return c.p.n == c.total;
    default: {  // RLE+Index: runs and points are disjoint
      if (c.gapless < 0) c.gapless = (covered_rows(ctx, c.s, c.e) + c.p2.n == c.total) ? 1 : 0;
      return c.gapless == 1;
    }
  }
}

std::pair<int64_t, int64_t> minmax(const CtxPtr& ctx, const DArr& v);
// a key column's value range, cached on the column
std::pair<int64_t, int64_t> col_minmax(const CtxPtr& ctx, const DCol& c) {
  if (!c.has_minmax) {
    auto mm = minmax(ctx, c.v);
    c.vmin = mm.first;
    c.vmax = mm.second;
    c.has_minmax = true;
  }
  return {c.vmin, c.vmax};
}

std::pair<int64_t, int64_t> minmax(const CtxPtr& ctx, const DArr& v) {
  DArr mm = alloc_arr(ctx, RQ_I64, 2);
  const int64_t init[2] = {INT64_MAX, INT64_MIN};
  RQ_CUDA_CHECK(cudaMemcpyAsync(mm.raw_mut(), init, 16, cudaMemcpyHostToDevice, ctx->stream));
  dev::k_gk_minmax<256><<<grid_cap(ctx, v.n), 256, 0, ctx->stream>>>(v.raw(), v.dt, v.n, mm.as<long long>());
  launched(ctx);
  const int64_t* h = ctx->readback(mm.raw(), 16);
  return {h[0], h[1]};
}

struct GroupKey {
  DArr s, e;  // key runs (aligned over all key columns); gaps allowed
  DArr slot;  // slot id per run (i64)
  int64_t G = 0;
  std::vector<int64_t> kmin, stride, range;
  std::vector<int32_t> kdt;
};

template <int KIND>
void run_rle(const CtxPtr& ctx, const GroupKey& K, const DArr& ds, const DArr& de, const DArr& dv,
             dev::GTable t, const double* mean) {
  const int64_t nk = K.e.n, n = de.n;
  if (nk == 0 || n == 0) return;
  constexpr int B = 256, IT = 8, TILE = B * IT;
  const int64_t ntiles = (nk + n + TILE - 1) / TILE;
  DArr part = alloc_arr(ctx, RQ_I64, ntiles + 1);
  dev::k_merge_partition<<<static_cast<unsigned>(((ntiles + 1) * 32 + 255) / 256), 256, 0, ctx->stream>>>(
      K.e.pos(), nk, de.pos(), n, TILE, ntiles + 1, part.as<int64_t>());
  launched(ctx);
  dev::MergeArgs m{K.e.pos(), nk, de.pos(), n, part.as<int64_t>()};
  dev::k_gk_rle<B, IT, KIND><<<static_cast<unsigned>(ntiles), B, 0, ctx->stream>>>(
      m, K.s.pos(), K.slot.raw(), K.slot.dt, ds.pos(), dv.raw(), dv.dt, t, mean);
  launched(ctx);
}

template <int KIND, bool POINTS>
void run_items(const CtxPtr& ctx, const GroupKey& K, const dev::PlainSrc& ps, const DArr* p, const DArr* v,
               int64_t n, dev::GTable t, const double* mean, const dev::PlainSrc* corr) {
  if (n == 0) return;
  // segment per warp: long enough to amortise the key-run search
  int64_t seg = 1 << 16;
  const int64_t warps_wanted = static_cast<int64_t>(ctx->sm_count) * 64;
  if (n / seg < warps_wanted) seg = std::max<int64_t>(256, ((n / warps_wanted) + 255) / 256 * 256);
  const int64_t warps = (n + seg - 1) / seg;
  int64_t blocks = (warps + 7) / 8;
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 8;
  if (blocks > cap) blocks = cap;
  dev::PlainSrc* dcorr = nullptr;
  DArr corr_buf;
  if (corr) {
    corr_buf = alloc_arr(ctx, RQ_I8, sizeof(dev::PlainSrc));
    RQ_CUDA_CHECK(cudaMemcpyAsync(corr_buf.raw_mut(), corr, sizeof(dev::PlainSrc), cudaMemcpyHostToDevice,
                                  ctx->stream));
    dcorr = corr_buf.as<dev::PlainSrc>();
  }
  auto go = [&](auto tag) {
    using S = decltype(tag);
    dev::k_gk_items<KIND, POINTS, S><<<static_cast<unsigned>(blocks), 256, 0, ctx->stream>>>(
        K.s.pos(), K.e.pos(), K.slot.raw(), K.slot.dt, K.e.n, ps, p ? p->pos() : nullptr,
        v ? v->raw() : nullptr, v ? v->dt : RQ_I64, n, seg, t, mean, dcorr);
  };
  if constexpr (POINTS) {
    go(int64_t{});
  } else {
    switch (ps.dt) {
      case RQ_I8: go(int8_t{}); break;
      case RQ_I16: go(int16_t{}); break;
      case RQ_I32: go(int32_t{}); break;
      case RQ_F32: go(float{}); break;
      case RQ_F64: go(double{}); break;
      default: go(int64_t{}); break;
    }
  }
  launched(ctx);
}

dev::PlainSrc plain_src(const DCol& c) {
  dev::PlainSrc ps{};
  ps.v = c.v.raw();
  ps.dt = c.v.dt;
  ps.logical = c.logical;
  ps.has_center = c.has_center ? 1 : 0;
  ps.center = c.center;
  ps.flt = (dt_float(c.v.dt) || dt_float(c.logical)) ? 1 : 0;
  return ps;
}

// accumulate one data column into table t with kind KIND
template <int KIND>
void fold_column(const CtxPtr& ctx, const GroupKey& K, const DCol& d, dev::GTable t, const double* mean) {
  switch (d.enc) {
    case RQ_ENC_RLE: run_rle<KIND>(ctx, K, d.s, d.e, d.v, t, mean); break;
    case RQ_ENC_INDEX: run_items<KIND, true>(ctx, K, {}, &d.p, &d.v, d.p.n, t, mean, nullptr); break;
    case RQ_ENC_PLAIN: run_items<KIND, false>(ctx, K, plain_src(d), nullptr, nullptr, d.v.n, t, mean, nullptr); break;
    case RQ_ENC_RLE_INDEX:
      run_rle<KIND>(ctx, K, d.s, d.e, d.v, t, mean);
      run_items<KIND, true>(ctx, K, {}, &d.p2, &d.v2, d.p2.n, t, mean, nullptr);
      break;
    case RQ_ENC_PLAIN_INDEX: {
      if (KIND == dev::G_SUM_I || KIND == dev::G_SUM_F) {
        // base over every row, then outlier rows add (outlier − decoded base)
        dev::PlainSrc base = plain_src(d);
        run_items<KIND, false>(ctx, K, base, nullptr, nullptr, d.v.n, t, mean, nullptr);
        run_items<KIND, true>(ctx, K, {}, &d.p2, &d.v2, d.p2.n, t, mean, &base);
      } else {
        DCol dec;
        dec.enc = RQ_ENC_PLAIN;
        dec.v = decode_plain_index(ctx, d);
        dec.logical = dec.v.dt;
        dec.total = dec.v.n;
        run_items<KIND, false>(ctx, K, plain_src(dec), nullptr, nullptr, dec.v.n, t, mean, nullptr);
      }
      break;
    }
    default: fail("group: unsupported encoding");
  }
}

DArr new_table(const CtxPtr& ctx, int64_t G, unsigned long long init) {
  DArr t = alloc_arr(ctx, RQ_I64, G);
  if (init == 0) {  // a memset, not a kernel
    if (G) RQ_CUDA_CHECK(cudaMemsetAsync(t.raw_mut(), 0, static_cast<size_t>(G) * 8, ctx->stream));
    return t;
  }
  dev::k_gk_init<<<grid_cap(ctx, G), 256, 0, ctx->stream>>>(reinterpret_cast<unsigned long long*>(t.raw_mut()), G, init);
  launched(ctx);
  return t;
}

template <int KIND>
DArr table_for(const CtxPtr& ctx, const GroupKey& K, const DCol& d, const double* mean) {
  unsigned long long init = 0;
  if (KIND == dev::G_MIN_I) init = static_cast<unsigned long long>(INT64_MAX);
  if (KIND == dev::G_MAX_I) init = static_cast<unsigned long long>(INT64_MIN);
  if (KIND == dev::G_MIN_F) init = 0x7ff0000000000000ull;
  if (KIND == dev::G_MAX_F) init = 0xfff0000000000000ull;
  DArr tab = new_table(ctx, K.G, init);
  dev::GTable t{reinterpret_cast<unsigned long long*>(tab.raw_mut()), K.G, 0};
  DArr part;
  int64_t rows = 0;
  if (KIND == dev::G_SUM_F || KIND == dev::G_SQ) {
    // deterministic f64: one row per warp of the widest launch fold_column makes
    rows = static_cast<int64_t>(ctx->sm_count) * 8 * 8;  // run_items' grid cap
    if (d.enc == RQ_ENC_RLE || d.enc == RQ_ENC_RLE_INDEX)
      rows = std::max<int64_t>(rows, (K.e.n + d.e.n + 2047) / 2048 * 8);  // run_rle: a warp per 256 merge items
    if (rows * K.G <= (int64_t{8} << 20)) {
      part = alloc_arr(ctx, RQ_F64, rows * K.G);
      RQ_CUDA_CHECK(cudaMemsetAsync(part.raw_mut(), 0, static_cast<size_t>(rows * K.G) * 8, ctx->stream));
      t.part = part.as<double>();
    }
  }
  fold_column<KIND>(ctx, K, d, t, mean);
  if (t.part && K.G) {
    dev::k_gk_pfold<<<static_cast<unsigned>(K.G), 256, 0, ctx->stream>>>(t.part, rows, K.G,
                                                                        reinterpret_cast<unsigned long long*>(tab.raw_mut()));
    launched(ctx);
  }
  return tab;
}

// Builds the key run column: single gapless RLE key, or several RLE keys
// aligned by range_intersect into one gapless run list of composite slots.
bool build_key(const CtxPtr& ctx, const std::vector<const DCol*>& keys, GroupKey& K) {
  for (auto* k : keys)
    if (k->enc != RQ_ENC_RLE || dt_float(k->v.dt)) return false;
  const DArr& e = keys[0]->e;
  std::vector<DArr> vals{keys[0]->v};
  K.s = keys[0]->s;
  K.e = e;
  auto mm = col_minmax(ctx, *keys[0]);
  const int64_t range = mm.second - mm.first + 1;
  if (vals[0].n == 0 || range <= 0 || range > kFusedSlotLimit) return false;
  K.G = range;
  K.kmin = {mm.first};
  K.stride = {1};
  K.range = {range};
  K.kdt = {vals[0].dt};
  // slot = key - min, as i64 per run
  DArr slot = alloc_arr(ctx, RQ_I64, vals[0].n);
  dev::KeyCols kc{};
  kc.nk = 1;
  kc.v[0] = vals[0].raw();
  kc.dt[0] = vals[0].dt;
  kc.mn[0] = mm.first;
  kc.stride[0] = 1;
  dev::k_gk_compose<<<grid_cap(ctx, vals[0].n), 256, 0, ctx->stream>>>(kc, vals[0].n, slot.as<int64_t>());
  launched(ctx);
  K.slot = slot;
  return true;
}

bool build_multi_key(const CtxPtr& ctx, const std::vector<const DCol*>& keys, GroupKey& K) {
  for (auto* k : keys)
    if (k->enc != RQ_ENC_RLE || dt_float(k->v.dt)) return false;
  // fold-align the key runs (range_intersect; coverage = ∩ of the keys)
  DArr s = keys[0]->s, e = keys[0]->e;
  std::vector<DArr> vals{keys[0]->v};
  for (size_t c = 1; c < keys.size(); ++c) {
    Intersection r = range_intersect(ctx, s, e, keys[c]->s, keys[c]->e, true, true);
    for (auto& v : vals) v = gather(ctx, v, r.idx1);
    vals.push_back(gather(ctx, keys[c]->v, r.idx2));
    s = r.s;
    e = r.e;
  }
  dev::KeyCols kc{};
  kc.nk = static_cast<int>(keys.size());
  int64_t G = 1;
  std::vector<int64_t> mn(keys.size()), range(keys.size()), stride(keys.size());
  for (size_t c = 0; c < keys.size(); ++c) {
    if (vals[c].n == 0) return false;
    // the column's range (cached) bounds the aligned values: slots of absent
    // combinations stay empty and are dropped by the count > 0 test
    auto mm = col_minmax(ctx, *keys[c]);
    mn[c] = mm.first;
    range[c] = mm.second - mm.first + 1;
    if (range[c] <= 0 || range[c] > kFusedSlotLimit) return false;
    G *= range[c];
    if (G > kFusedSlotLimit) return false;
  }
  int64_t st = 1;
  for (size_t c = keys.size(); c-- > 0;) {
    stride[c] = st;
    st *= range[c];
  }
  for (size_t c = 0; c < keys.size(); ++c) {
    kc.v[c] = vals[c].raw();
    kc.dt[c] = vals[c].dt;
    kc.mn[c] = mn[c];
    kc.stride[c] = stride[c];
  }
  DArr slot = alloc_arr(ctx, RQ_I64, e.n);
  dev::k_gk_compose<<<grid_cap(ctx, e.n), 256, 0, ctx->stream>>>(kc, e.n, slot.as<int64_t>());
  launched(ctx);
  K.s = s;
  K.e = e;
  K.slot = slot;
  K.G = G;
  K.kmin = mn;
  K.stride = stride;
  K.range = range;
  for (auto& v : vals) K.kdt.push_back(v.dt);
  return true;
}

}  // namespace

namespace {
bool xg_fused(const CtxPtr& ctx, const DMask* mask, const std::vector<const DCol*>& keys,
              const std::vector<XExpr>& exprs, const std::vector<int>& fns, GroupAggOut& out,
              const GroupKey* preK = nullptr, const std::vector<XPred>* preds = nullptr);
}  // namespace

// Returns false when the inputs are not in the fused shape (caller then runs
// the general aligned path).
bool group_aggregate_fused(const CtxPtr& ctx, const std::vector<const DCol*>& keys,
                           const std::vector<const DCol*>& data, const std::vector<int>& fns,
                           GroupAggOut& out) {
  if (keys.empty() || keys.size() > 8) return false;
  const int64_t total = keys[0]->total;
  for (auto* k : keys)
    if (k->total != total || k->enc != RQ_ENC_RLE) return false;
  for (auto* d : data)
    if (d->total != total) return false;
  GroupKey K;
  if (!(keys.size() == 1 ? build_key(ctx, keys, K) : build_multi_key(ctx, keys, K))) return false;
  // Per-aggregate alignment is exact when every input covers exactly the
  // rows the (aligned) key runs cover: full tables, or columns all filtered
  // by the same mask (query runner Filter → GroupAgg).
  const int64_t kcov = covered_rows(ctx, K.s, K.e);
  if (kcov == total) {
    for (auto* d : data)
      if (!full_cover(ctx, *d)) return false;
  } else {
    const void* checked_p = nullptr;  // Index columns sharing one position buffer: check once
    for (auto* d : data) {
      if (d->enc == RQ_ENC_INDEX) {
        if (d->p.n != kcov) return false;
        if (d->p.raw() != checked_p) {
          PointsInRuns r = points_in_runs(ctx, d->p, K.s, K.e, false, false);
          if (r.p_out.n != d->p.n) return false;
          checked_p = d->p.raw();
        }
      } else if (d->enc == RQ_ENC_RLE) {
        if (covered_rows(ctx, d->s, d->e) != kcov) return false;
        Intersection r = range_intersect(ctx, K.s, K.e, d->s, d->e, false, false);
        if (covered_rows(ctx, r.s, r.e) != kcov) return false;
      } else {
        return false;  // plain / composite data with filtered keys: general path
      }
    }
  }
  auto to_rows = [&](size_t i, size_t taken) {
    const DCol& d = *data[i];
    return kcov == total && (d.enc == RQ_ENC_PLAIN || d.enc == RQ_ENC_PLAIN_INDEX) &&
           (fns[i] == RQ_SUM || fns[i] == RQ_AVG) && taken < 4;
  };
  KTimer timer(ctx, "group_fused");
  // Plain / Plain+Index SUM and AVG over fully covered keys: one K12 row pass
  // streams all of them together (decode baked into the generated kernel)
  std::vector<size_t> x_idx;
  GroupAggOut x_out;
  bool x_ok = false;
  if (kcov == total) {
    std::vector<XExpr> xe;
    std::vector<int> xf;
    for (size_t i = 0; i < data.size(); ++i) {
      const DCol& d = *data[i];
      if (to_rows(i, xe.size())) {
        XExpr x;
        XTerm t;
        t.col = &d;
        x.terms.push_back(t);
        xe.push_back(x);
        xf.push_back(fns[i]);
        x_idx.push_back(i);
      }
    }
    if (!xe.empty()) x_ok = xg_fused(ctx, nullptr, keys, xe, xf, x_out, &K);
    if (!x_ok) x_idx.clear();
  }
  // counts / presence from the key runs
  DArr cnt = new_table(ctx, K.G, 0);
  {
    dev::GTable t{reinterpret_cast<unsigned long long*>(cnt.raw_mut()), K.G, 0};
    dev::k_gk_count<<<grid_cap(ctx, K.e.n), 256, 0, ctx->stream>>>(K.s.pos(), K.e.pos(), K.slot.raw(),
                                                                    K.slot.dt, K.e.n, t);
    launched(ctx);
  }
  DArr flags = alloc_arr(ctx, RQ_I8, K.G);
  dev::k_gk_flags<<<grid_cap(ctx, K.G), 256, 0, ctx->stream>>>(
      reinterpret_cast<const unsigned long long*>(cnt.raw()), K.G, flags.as<uint8_t>());
  launched(ctx);
  DArr present;
  flagged_indices(ctx, flags, K.G, present);
  const int64_t ng = present.n;
  out.n_groups = ng;
  for (size_t c = 0; c < keys.size(); ++c) {
    DArr kout = alloc_arr(ctx, K.kdt[c], ng);
    if (ng) {
      dev::k_gk_keys<<<grid_cap(ctx, ng), 256, 0, ctx->stream>>>(present.pos(), ng, K.kmin[c], K.stride[c],
                                                                 K.range[c], K.kdt[c], kout.raw_mut());
      launched(ctx);
    }
    out.keys.push_back(kout);
  }
  for (size_t i = 0; i < data.size(); ++i) {
    bool taken = false;
    for (size_t j = 0; j < x_idx.size(); ++j)
      if (x_idx[j] == i && x_out.n_groups == ng) {
        out.vals.push_back(x_out.vals[j]);
        taken = true;
      }
    if (taken) continue;
    const DCol& d = *data[i];
    const int fn = fns[i];
    const bool flt = dt_float(d.value_type());
    DArr acc, sq;
    int32_t odt = RQ_F64;
    switch (fn) {
      case RQ_SUM:
        acc = flt ? table_for<dev::G_SUM_F>(ctx, K, d, nullptr) : table_for<dev::G_SUM_I>(ctx, K, d, nullptr);
        odt = flt ? RQ_F64 : RQ_I64;
        break;
      case RQ_COUNT: odt = RQ_I64; break;
      case RQ_MIN:
        acc = flt ? table_for<dev::G_MIN_F>(ctx, K, d, nullptr) : table_for<dev::G_MIN_I>(ctx, K, d, nullptr);
        odt = flt ? RQ_F64 : RQ_I64;
        break;
      case RQ_MAX:
        acc = flt ? table_for<dev::G_MAX_F>(ctx, K, d, nullptr) : table_for<dev::G_MAX_I>(ctx, K, d, nullptr);
        odt = flt ? RQ_F64 : RQ_I64;
        break;
      default: {  // AVG / VAR / STD: f64 sum of value·weight, then Σ (v - mean)²·w
        acc = table_for<dev::G_SUM_F>(ctx, K, d, nullptr);
        if (fn != RQ_AVG) {
          DArr mean = alloc_arr(ctx, RQ_F64, K.G);
          dev::k_gk_mean<<<grid_cap(ctx, K.G), 256, 0, ctx->stream>>>(
              reinterpret_cast<const unsigned long long*>(acc.raw()),
              reinterpret_cast<const unsigned long long*>(cnt.raw()), K.G, mean.as<double>());
          launched(ctx);
          sq = table_for<dev::G_SQ>(ctx, K, d, mean.as<double>());
        }
      }
    }
    DArr res = alloc_arr(ctx, odt, ng);
    if (ng) {
      dev::k_gk_finish<<<grid_cap(ctx, ng), 256, 0, ctx->stream>>>(
          present.pos(), ng, fn, acc.n ? reinterpret_cast<const unsigned long long*>(acc.raw()) : nullptr,
          reinterpret_cast<const unsigned long long*>(cnt.raw()),
          sq.n ? reinterpret_cast<const unsigned long long*>(sq.raw()) : nullptr, res.raw_mut());
      launched(ctx);
    }
    out.vals.push_back(res);
  }
  return true;
}



// ===========================================================================
// K12 — filtered group-aggregate over expression aggregates.
//
// The query runner evaluates Filter → arith / arith_scalar → GroupAgg
// (runner.cpp:243-336): every scanned column is filtered by the predicate
// mask (a plain column becomes an IndexColumn of survivors, align.cpp:733-751),
// each aggregate expression is materialised by binary / scalar operators
// (align.cpp:495-508, :571-596) and group_aggregate aligns keys and data
// (groupby.cpp:144-162). Here the rows that survive are described by a
// SEGMENT table — the key runs ∩ the mask's runs ∩ the runs of every RLE
// operand (the joint alignment of align_many, computed on the small run
// lists) — each segment carrying its group slot and its RLE operands'
// values. One row kernel then streams the plain operand columns once
// (128-bit / narrow vector loads, bit-width-reduced decode in registers),
// evaluates every expression per row with the reference's promotion rules
// (any float → f64, else wrapping int64; int ÷0 raises) and accumulates
// per-lane partials that are flushed per segment into a (slot × expression)
// table. Covered rows are split evenly over warps (a prefix over segment
// lengths), so only selected rows are read. Plain+Index operands (SUM/AVG of
// the bare column) add a per-outlier correction; COUNT and expressions over
// RLE operands only are evaluated once per segment (value × length, the
// reference's run weights, groupby.cpp:67-135).
// ===========================================================================

namespace dev {

__device__ __forceinline__ double xg_f(uint64_t b, int f) {
  return f ? __longlong_as_double(static_cast<long long>(b)) : static_cast<double>(static_cast<int64_t>(b));
}
// binary op with the reference's promotion (align.cpp:290-305)
__device__ __forceinline__ uint64_t xg_op(uint64_t a, int fa, uint64_t b, int fb, int op, int* err) {
  if (fa || fb) return static_cast<uint64_t>(__double_as_longlong(arith_f64(xg_f(a, fa), xg_f(b, fb), op, nullptr)));
  return static_cast<uint64_t>(arith_i64(static_cast<int64_t>(a), static_cast<int64_t>(b), op, err));
}
__device__ __forceinline__ uint64_t xg_term(const XgTerm& t, uint64_t x, int* err) {
  if (t.sop < 0) return x;
  const uint64_t k = t.kflt ? static_cast<uint64_t>(__double_as_longlong(t.kf)) : static_cast<uint64_t>(t.ki);
  return t.rev ? xg_op(k, t.kflt, x, t.flt, t.sop, err) : xg_op(x, t.flt, k, t.kflt, t.sop, err);
}

// decode of one storage value to the logical value bits (column.cpp:283-297)
template <class S>
__device__ __forceinline__ uint64_t xg_decode(const PlainSrc& s, S raw) {
  if constexpr (std::is_same<S, double>::value) {
    return static_cast<uint64_t>(__double_as_longlong(raw));
  } else if constexpr (std::is_same<S, float>::value) {
    return static_cast<uint64_t>(__double_as_longlong(static_cast<double>(raw)));
  } else {
    int64_t x = static_cast<int64_t>(raw);
    if (s.logical != RQ_I64) x = wrap_to(s.logical, x);
    if (s.has_center) {
      x = static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(s.center));
      if (s.logical != RQ_I64) x = wrap_to(s.logical, x);
    }
    if (s.flt) return static_cast<uint64_t>(__double_as_longlong(static_cast<double>(x)));
    return static_cast<uint64_t>(x);
  }
}

// four consecutive rows (row0 % 4 == 0) of a plain column, decoded
__device__ __forceinline__ void xg_load4(const PlainSrc& s, int64_t row0, uint64_t (&o)[4]) {
  switch (s.dt) {
    case RQ_I8: {
      const uint32_t w = __ldg(reinterpret_cast<const unsigned int*>(static_cast<const int8_t*>(s.v) + row0));
#pragma unroll
      for (int u = 0; u < 4; ++u) o[u] = xg_decode<int8_t>(s, static_cast<int8_t>((w >> (8 * u)) & 0xff));
      break;
    }
    case RQ_I16: {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(static_cast<const int16_t*>(s.v) + row0));
      o[0] = xg_decode<int16_t>(s, static_cast<int16_t>(w.x & 0xffff));
      o[1] = xg_decode<int16_t>(s, static_cast<int16_t>(w.x >> 16));
      o[2] = xg_decode<int16_t>(s, static_cast<int16_t>(w.y & 0xffff));
      o[3] = xg_decode<int16_t>(s, static_cast<int16_t>(w.y >> 16));
      break;
    }
    case RQ_I32: {
      const int4 w = __ldg(reinterpret_cast<const int4*>(static_cast<const int32_t*>(s.v) + row0));
      o[0] = xg_decode<int32_t>(s, w.x);
      o[1] = xg_decode<int32_t>(s, w.y);
      o[2] = xg_decode<int32_t>(s, w.z);
      o[3] = xg_decode<int32_t>(s, w.w);
      break;
    }
    case RQ_F32: {
      const float4 w = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(s.v) + row0));
      o[0] = xg_decode<float>(s, w.x);
      o[1] = xg_decode<float>(s, w.y);
      o[2] = xg_decode<float>(s, w.z);
      o[3] = xg_decode<float>(s, w.w);
      break;
    }
    case RQ_F64: {
      const double2* p = reinterpret_cast<const double2*>(static_cast<const double*>(s.v) + row0);
      const double2 a = __ldg(p), b = __ldg(p + 1);
      o[0] = xg_decode<double>(s, a.x);
      o[1] = xg_decode<double>(s, a.y);
      o[2] = xg_decode<double>(s, b.x);
      o[3] = xg_decode<double>(s, b.y);
      break;
    }
    default: {
      const longlong2* p = reinterpret_cast<const longlong2*>(static_cast<const int64_t*>(s.v) + row0);
      const longlong2 a = __ldg(p), b = __ldg(p + 1);
      o[0] = xg_decode<int64_t>(s, a.x);
      o[1] = xg_decode<int64_t>(s, a.y);
      o[2] = xg_decode<int64_t>(s, b.x);
      o[3] = xg_decode<int64_t>(s, b.y);
    }
  }
}


// dp (deterministic mode): this chunk's f64 partial table, written by lane 0 only
__device__ __forceinline__ void xg_flush(const XgPlan& P, unsigned long long* tab, int64_t slot,
                                         uint64_t (&acc)[XG_EXPRS], double* dp) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < XG_EXPRS; ++e) {
    if (e >= P.ne || !P.e[e].rows) continue;
    if (P.e[e].acc_f) {
      double v = __longlong_as_double(static_cast<long long>(acc[e]));
      v = warp_sum(v);
      if (dp) {
        if (lane == 0) dp[slot * P.ne + e] += v;
      } else if (lane == 0 && v != 0.0) {
        atomicAdd(reinterpret_cast<double*>(tab) + slot * P.ne + e, v);
      }
    } else {
      unsigned long long v = warp_sum(static_cast<unsigned long long>(acc[e]));
      if (lane == 0 && v != 0ull) atomicAdd(tab + slot * P.ne + e, v);
    }
    acc[e] = 0;
  }
}

// v[u] = v[u] op x[u] for the lane's 4 rows; the type / operator dispatch
// is uniform and hoisted out of the row loop
// Integer division only divides the rows that count (ok[u]: inside the
// segment's [r0, r1]); the window's other rows (dropped by the WHERE, a
// neighbouring segment, padding past the last covered row) divide by 1, so a
// zero there cannot raise — the reference divides only the filtered rows
// (align.cpp:290-305 after filter, :755-771).
__device__ __forceinline__ void xg_op4(uint64_t (&v)[4], int vf, const uint64_t (&x)[4], int xf, int op, int* err,
                                       const bool (&ok)[4]) {
  if (vf || xf) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = xg_f(v[u], vf);
      b[u] = xg_f(x[u], xf);
    }
    switch (op) {
      case RQ_ADD:
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = a[u] + b[u];
        break;
      case RQ_SUB:
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = a[u] - b[u];
        break;
      case RQ_MUL:
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = a[u] * b[u];
        break;
      default:
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = a[u] / b[u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = static_cast<uint64_t>(__double_as_longlong(a[u]));
  } else {
    switch (op) {
      case RQ_ADD:
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = v[u] + x[u];
        break;
      case RQ_SUB:
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = v[u] - x[u];
        break;
      case RQ_MUL:
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = v[u] * x[u];
        break;
      default:
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = static_cast<uint64_t>(
              arith_i64(static_cast<int64_t>(v[u]), ok[u] ? static_cast<int64_t>(x[u]) : int64_t(1), RQ_DIV, err));
    }
  }
}

// Row kernel: warp w takes covered rows [w·chunk, (w+1)·chunk) (segment
// order), lanes take 4 consecutive rows each per 128-row window. Every
// operand column is decoded once per window into the lane's slice of a
// shared-memory tile (so a term's source is an address, not a register
// select); expressions are then evaluated term by term over the 4 rows with
// the operator / type dispatch hoisted out of the row loop.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_xg_rows(const __grid_constant__ XgPlan P, const __grid_constant__ XgSegs S, int64_t chunk, unsigned long long* __restrict__ gtab, int64_t G,
              int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned long long xsm[];
  const int64_t cells = G * P.ne;
  const bool in_smem = cells <= kSmemSlots;
  unsigned long long* stab = xsm;                                   // kSmemSlots
  uint64_t* ctile = reinterpret_cast<uint64_t*>(xsm + kSmemSlots);  // [XG_COLS][BLOCK * 4]
  uint64_t* kcs = ctile + XG_COLS * BLOCK * 4;                      // [BLOCK / 32][XG_CONSTS]
  if (in_smem) {
    for (int64_t i = threadIdx.x; i < cells; i += BLOCK) stab[i] = 0ull;
    __syncthreads();
  }
  unsigned long long* tab = in_smem ? stab : gtab;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * BLOCK) >> 5;
  uint64_t* my = ctile + threadIdx.x * 4;  // this lane's 4 rows of column c at my[c * BLOCK * 4]
  uint64_t* wk = kcs + wid * XG_CONSTS;
  int lerr = 0;
  uint64_t acc[XG_EXPRS];
#pragma unroll
  for (int e = 0; e < XG_EXPRS; ++e) acc[e] = 0;
  const int64_t nseg = S.dims ? ldg64(S.dims, 0) : S.n, ncov = S.dims ? ldg64(S.dims, 1) : S.ncov;
  if (chunk <= 0) chunk = xg_chunk(ncov, nwarps);
  for (int64_t c0 = warp * chunk; c0 < ncov; c0 += nwarps * chunk) {
    const int64_t c1 = min(c0 + chunk, ncov);
    // segment holding covered row c0
    int64_t k = S.cstart ? ldg64(S.cstart, c0 / chunk) : warp_lower_bound(S.off, nseg, c0 + 1) - 1;
    int64_t c = c0;
    while (c < c1) {
      const int64_t off = ldg64(S.off, k), s = ldg64(S.s, k), e = ldg64(S.e, k);
      const int64_t slot = ldg64(S.slot, k);
      if (lane < P.ncst) wk[lane] = __ldg(S.cst + lane * S.cstride + k);
      __syncwarp();
      const int64_t r0 = s + (c - off);
      const int64_t r1 = min(e, s + (c1 - off) - 1);
      for (int64_t b = r0 & ~int64_t(3); b <= r1; b += 128) {
        const int64_t row = b + lane * 4;
        if (row > r1) continue;  // lane past the piece (no cross-lane traffic below)
        for (int ci = 0; ci < P.nc; ++ci) {
          uint64_t t[4];
          xg_load4(P.col[ci], row, t);
          uint64_t* d = my + ci * BLOCK * 4;
          reinterpret_cast<ulonglong2*>(d)[0] = make_ulonglong2(t[0], t[1]);
          reinterpret_cast<ulonglong2*>(d)[1] = make_ulonglong2(t[2], t[3]);
        }
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) ok[u] = row + u >= r0 && row + u <= r1;
#pragma unroll
        for (int ei = 0; ei < XG_EXPRS; ++ei) {
          if (ei >= P.ne || !P.e[ei].rows) continue;
          uint64_t v[4];
          int vf = 0;
          for (int ti = 0; ti < P.e[ei].nt; ++ti) {
            const XgTerm& T = P.e[ei].t[ti];
            uint64_t x[4];
            if (T.src < XG_COLS) {
              const ulonglong2* q = reinterpret_cast<const ulonglong2*>(my + T.src * BLOCK * 4);
              const ulonglong2 p0 = q[0], p1 = q[1];
              x[0] = p0.x;
              x[1] = p0.y;
              x[2] = p1.x;
              x[3] = p1.y;
            } else {
              const uint64_t kv = wk[T.src - XG_COLS];
#pragma unroll
              for (int u = 0; u < 4; ++u) x[u] = kv;
            }
            int xf = T.flt;
            if (T.sop >= 0) {  // scalar op: x op k, or k op x
              const uint64_t kb = T.kflt ? static_cast<uint64_t>(__double_as_longlong(T.kf)) : static_cast<uint64_t>(T.ki);
              uint64_t kk[4] = {kb, kb, kb, kb};
              if (T.rev) {
                xg_op4(kk, T.kflt, x, xf, T.sop, &lerr, ok);
#pragma unroll
                for (int u = 0; u < 4; ++u) x[u] = kk[u];
              } else {
                xg_op4(x, xf, kk, T.kflt, T.sop, &lerr, ok);
              }
              xf = xf || T.kflt;
            }
            if (ti == 0) {
#pragma unroll
              for (int u = 0; u < 4; ++u) v[u] = x[u];
              vf = xf;
            } else {
              xg_op4(v, vf, x, xf, P.e[ei].op[ti - 1], &lerr, ok);
              vf = vf || xf;
            }
          }
          if (P.e[ei].acc_f) {
            double a = __longlong_as_double(static_cast<long long>(acc[ei]));
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (ok[u]) a += xg_f(v[u], vf);
            acc[ei] = static_cast<uint64_t>(__double_as_longlong(a));
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (ok[u]) acc[ei] += v[u];
          }
        }
      }
      c = min(c1, off + (e - s + 1));
      // flush at segment ends where the slot changes, and at the chunk end
      const int64_t next_slot = (c < c1 && k + 1 < nseg) ? ldg64(S.slot, k + 1) : -1;
      if (next_slot != slot) xg_flush(P, tab, slot, acc, S.dpart ? S.dpart + (c0 / chunk) * S.dcells : nullptr);
      __syncwarp();
      ++k;
    }
  }
  if (lerr) atomicOr(err, 1);
  if (in_smem) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < cells; i += BLOCK) {
      const unsigned long long v = stab[i];
      if (!v) continue;
      const int ei = static_cast<int>(i % P.ne);
      if (P.e[ei].acc_f) atomicAdd(reinterpret_cast<double*>(gtab) + i, __longlong_as_double(static_cast<long long>(v)));
      else atomicAdd(gtab + i, v);
    }
  }
}

template <int BLOCK>
constexpr size_t xg_rows_smem() {
  return (static_cast<size_t>(kSmemSlots) + XG_COLS * BLOCK * 4 + (BLOCK / 32) * XG_CONSTS) * 8;
}

// Per segment: COUNT (Σ lengths) and expressions over RLE operands only
// (value × length, the reference's run weights).
// Warp-aggregated add: lanes holding the same cell combine first (segments
// come in position order, so neighbouring segments mostly share a slot) and
// one lane per distinct cell issues the atomic.
__device__ __forceinline__ void xg_add_u64(unsigned long long* base, int64_t cell, uint64_t v) {
  const unsigned same = __match_any_sync(__activemask(), static_cast<unsigned long long>(cell));
  uint64_t sum = 0;
  for (unsigned m = same; m; m &= m - 1) sum += __shfl_sync(same, v, __ffs(m) - 1);
  if ((threadIdx.x & 31) == __ffs(same) - 1 && sum) atomicAdd(base + cell, static_cast<unsigned long long>(sum));
}
// f64 adds of a warp, lanes of one cell summed in lane order; then either an
// atomic add (order-dependent last bits) or — `part` given — a plain add into
// this warp's own partial-table row, folded over warps in a fixed order later
// (k_xg_dfold): bit-identical run to run.
__device__ __forceinline__ void xg_add_f64(double* base, int64_t cell, double v, double* part = nullptr) {
  const unsigned same = __match_any_sync(__activemask(), static_cast<unsigned long long>(cell));
  double sum = 0.0;
  for (unsigned m = same; m; m &= m - 1) sum += __shfl_sync(same, v, __ffs(m) - 1);
  if ((threadIdx.x & 31) != __ffs(same) - 1) return;
  if (part) part[cell] += sum;
  else if (sum != 0.0) atomicAdd(base + cell, sum);
}

__global__ void k_xg_segs(const __grid_constant__ XgPlan P, const __grid_constant__ XgSegs S, unsigned long long* __restrict__ tab,
                          unsigned long long* __restrict__ cnt, int* __restrict__ err, double* __restrict__ part,
                          int64_t cells) {
  int lerr = 0;
  // this warp's row of the f64 partial table (null: atomics)
  double* prow = part ? part + ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * cells : nullptr;
  // every lane of a warp runs the same number of iterations (warp-collective adds)
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t first = static_cast<int64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31);
  const int64_t nseg = S.dims ? ldg64(S.dims, 0) : S.n;
  for (int64_t base = first; base < nseg; base += stride) {
    const int64_t k = base + (threadIdx.x & 31);
    const bool ok = k < nseg;
    const int64_t len = ok ? ldg64(S.e, k) - ldg64(S.s, k) + 1 : 0;
    const int64_t slot = ok ? ldg64(S.slot, k) : 0;
    xg_add_u64(cnt, slot, static_cast<uint64_t>(len));
    for (int ei = 0; ei < P.ne; ++ei) {
      const XgExpr& X = P.e[ei];
      if (X.rows || X.nt == 0) continue;
      uint64_t v = 0;
      int vf = 0;
      for (int ti = 0; ti < X.nt; ++ti) {
        const XgTerm& T = X.t[ti];
        const uint64_t y = ok ? xg_term(T, __ldg(S.cst + (T.src - XG_COLS) * S.cstride + k), &lerr) : 0;
        const int yf = T.flt || (T.sop >= 0 && T.kflt);
        if (ti == 0) {
          v = y;
          vf = yf;
        } else {
          v = ok ? xg_op(v, vf, y, yf, X.op[ti - 1], &lerr) : 0;
          vf = vf || yf;
        }
      }
      const int64_t cell = slot * P.ne + ei;
      if (X.acc_f)
        xg_add_f64(reinterpret_cast<double*>(tab), cell, ok ? xg_f(v, vf) * static_cast<double>(len) : 0.0, prow);
      else xg_add_u64(tab, cell, static_cast<uint64_t>(v) * static_cast<uint64_t>(len));
    }
  }
  if (lerr) atomicOr(err, 1);
}

// Plain+Index operand: outlier rows inside segments replace the base's
// decoded value (column.cpp:299-309).
__global__ void k_xg_outliers(PlainSrc base, const int64_t* __restrict__ p, const void* __restrict__ v2, int v2dt,
                              const int64_t* __restrict__ idx_of, const int64_t* __restrict__ run_of, int64_t n,
                              const int64_t* __restrict__ seg_slot, int ne, int ei, int acc_f,
                              unsigned long long* __restrict__ tab) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t first = static_cast<int64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31);
  for (int64_t b = first; b < n; b += stride) {  // warp-uniform trip count (warp-collective adds)
    const int64_t i = b + (threadIdx.x & 31);
    const bool ok = i < n;
    const int64_t pos = ok ? ldg64(p, i) : 0;
    const int64_t slot = ok ? ldg64(seg_slot, ldg64(run_of, i)) : 0;
    const int64_t q = ok ? ldg64(idx_of, i) : 0;
    if (acc_f) {
      const double d = ok ? ld_f64(v2, v2dt, q) - plain_value<double>(base, pos) : 0.0;
      xg_add_f64(reinterpret_cast<double*>(tab), slot * ne + ei, d);
    } else {
      const uint64_t d = ok ? static_cast<uint64_t>(ld_i64(v2, v2dt, q)) - static_cast<uint64_t>(plain_value<int64_t>(base, pos)) : 0;
      xg_add_u64(tab, slot * ne + ei, d);
    }
  }
}

__global__ void k_xg_finish(const int64_t* __restrict__ slots, int64_t ng, int ne, int ei, int fn, int acc_f,
                            const unsigned long long* __restrict__ tab, const unsigned long long* __restrict__ cnt,
                            void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < ng;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = ldg64(slots, i);
    const unsigned long long c = cnt[g];
    if (fn == RQ_COUNT) {
      static_cast<long long*>(out)[i] = static_cast<long long>(c);
    } else if (fn == RQ_AVG) {
      static_cast<double*>(out)[i] = c ? __longlong_as_double(static_cast<long long>(tab[g * ne + ei])) / static_cast<double>(c)
                                       : __longlong_as_double(0x7ff8000000000000ll);
    } else {
      static_cast<unsigned long long*>(out)[i] = tab[g * ne + ei];
    }
    (void)acc_f;
  }
}

struct XgFinish {
  int ne;
  int fn[XG_EXPRS];
  int isf[XG_EXPRS];  // the table cell holds f64 bits (else a wrapping int64 sum)
  void* out[XG_EXPRS];
};
__global__ void k_xg_finish_all(const __grid_constant__ XgFinish F, const int64_t* __restrict__ slots, int64_t ng,
                                const unsigned long long* __restrict__ tab, const unsigned long long* __restrict__ cnt) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < ng;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = slots ? ldg64(slots, i) : i;  // null: the slots are 0..ng-1 (no keys: one group)
    const unsigned long long c = cnt[g];
    for (int ei = 0; ei < F.ne; ++ei) {
      const int fn = F.fn[ei];
      if (fn == RQ_COUNT) {
        static_cast<long long*>(F.out[ei])[i] = static_cast<long long>(c);
      } else if (fn == RQ_AVG) {  // f64(Σ) / count (groupby.cpp:103-106); an integer Σ is exact in int64
        const unsigned long long t = tab[g * F.ne + ei];
        const double sum = F.isf[ei] ? __longlong_as_double(static_cast<long long>(t))
                                     : static_cast<double>(static_cast<long long>(t));
        static_cast<double*>(F.out[ei])[i] = c ? sum / static_cast<double>(c) : __longlong_as_double(0x7ff8000000000000ll);
      } else {
        static_cast<unsigned long long*>(F.out[ei])[i] = tab[g * F.ne + ei];
      }
    }
  }
}

// The keyed output stage in ONE block (tables of up to XG_TAIL_MAX slots):
// present slots (count > 0) ranked by a block scan over contiguous slot
// ranges, keys decoded from the slot (ascending slot = ascending key) and
// every expression's result written at the slot's rank, the group count into
// *ng. Replaces flags → select (size readback) → keys → finish: the host
// reads the count once, after all the work is queued.
constexpr int XG_TAIL_B = 1024;
constexpr int64_t XG_TAIL_MAX = 32768;
struct XgTailKeys {
  int nk;
  int dt[8];
  int64_t kmin[8], stride[8], range[8];
  void* out[8];
};
__global__ void __launch_bounds__(XG_TAIL_B)
    k_xg_tail(const __grid_constant__ XgFinish F, const __grid_constant__ XgTailKeys KT, int64_t G,
              const unsigned long long* __restrict__ tab, const unsigned long long* __restrict__ cnt,
              int64_t* __restrict__ ng) {
  __shared__ int64_t wt[XG_TAIL_B / 32 + 1];
  const int64_t per = (G + XG_TAIL_B - 1) / XG_TAIL_B;
  const int64_t g0 = min(G, threadIdx.x * per), g1 = min(G, g0 + per);
  int64_t mine = 0;
  for (int64_t g = g0; g < g1; ++g) mine += cnt[g] > 0;
  int64_t total;
  int64_t i = block_exclusive<XG_TAIL_B>(mine, total, wt);
  if (threadIdx.x == 0) *ng = total;
  for (int64_t g = g0; g < g1; ++g) {
    const unsigned long long c = cnt[g];
    if (!c) continue;
    for (int k = 0; k < KT.nk; ++k) {
      const int64_t key = KT.kmin[k] + (g / KT.stride[k]) % KT.range[k];
      switch (KT.dt[k]) {
        case RQ_I8: static_cast<int8_t*>(KT.out[k])[i] = static_cast<int8_t>(key); break;
        case RQ_I16: static_cast<int16_t*>(KT.out[k])[i] = static_cast<int16_t>(key); break;
        case RQ_I32: static_cast<int32_t*>(KT.out[k])[i] = static_cast<int32_t>(key); break;
        default: static_cast<int64_t*>(KT.out[k])[i] = key; break;
      }
    }
    for (int ei = 0; ei < F.ne; ++ei) {  // k_xg_finish_all's conventions (groupby.cpp:67-135)
      const int fn = F.fn[ei];
      if (fn == RQ_COUNT) {
        static_cast<long long*>(F.out[ei])[i] = static_cast<long long>(c);
      } else if (fn == RQ_AVG) {
        const unsigned long long t = tab[g * F.ne + ei];
        const double sum = F.isf[ei] ? __longlong_as_double(static_cast<long long>(t))
                                     : static_cast<double>(static_cast<long long>(t));
        static_cast<double*>(F.out[ei])[i] = sum / static_cast<double>(c);
      } else {
        static_cast<unsigned long long*>(F.out[ei])[i] = tab[g * F.ne + ei];
      }
    }
    ++i;
  }
}

// deterministic f64 fold: cell blockIdx.x of every chunk's partial table,
// a fixed strided split over the block's threads and a fixed-shape tree
struct XgIsF {
  int f[XG_EXPRS];
};
constexpr int DFOLD_B = 512;
__global__ void __launch_bounds__(DFOLD_B)
    k_xg_dfold(const double* __restrict__ dpart, int64_t nchunks, int64_t cells, int ne, XgIsF is_f,
               unsigned long long* __restrict__ tab, int add = 0) {
  __shared__ double red[DFOLD_B];
  const int64_t cell = blockIdx.x;
  if (!is_f.f[cell % ne]) return;
  // four independent partial sums per thread (loads in flight), combined in
  // a fixed order: the same bits on every run
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t q = threadIdx.x;
  for (; q + 3 * DFOLD_B < nchunks; q += 4 * DFOLD_B) {
    a0 += dpart[q * cells + cell];
    a1 += dpart[(q + DFOLD_B) * cells + cell];
    a2 += dpart[(q + 2 * DFOLD_B) * cells + cell];
    a3 += dpart[(q + 3 * DFOLD_B) * cells + cell];
  }
  for (; q < nchunks; q += DFOLD_B) a0 += dpart[q * cells + cell];
  red[threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  for (int w = DFOLD_B / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double v = add ? __longlong_as_double(static_cast<long long>(tab[cell])) + red[0] : red[0];
    tab[cell] = static_cast<unsigned long long>(__double_as_longlong(v));
  }
}

__global__ void k_xg_lengths(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t n,
                             int64_t* __restrict__ len) {  // len[n] = 0
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    len[i] = i < n ? ldg64(e, i) - ldg64(s, i) + 1 : 0;
}

}  // namespace dev

namespace dev {
__global__ void k_xg_fill1(int64_t* __restrict__ out, int64_t v) { *out = v; }
__global__ void k_xg_fill3(int64_t* a, int64_t va, int64_t* b, int64_t vb, int64_t* c, int64_t vc) {
  *a = va;
  *b = vb;
  *c = vc;
}

constexpr int XG_GATHER = 8;
struct XgGather {
  int n;
  const void* src[XG_GATHER];
  const int64_t* idx[XG_GATHER];  // each array's own index (all of length n)
  int dt[XG_GATHER];
  int to_f[XG_GATHER];
  void* dst[XG_GATHER];
};
__global__ void k_xg_gather(const __grid_constant__ XgGather G, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    for (int a = 0; a < G.n; ++a) {
      const int64_t j = ldg64(G.idx[a], i);
      if (G.to_f[a]) static_cast<double*>(G.dst[a])[i] = ld_f64(G.src[a], G.dt[a], j);
      else static_cast<int64_t*>(G.dst[a])[i] = ld_i64(G.src[a], G.dt[a], j);
    }
  }
}

// WHERE pushdown: one conjunct per entry, `col op k` or `col IN (list)`,
// evaluated once per segment on the segment's value of the predicate column
// (compare_scalar semantics, align.cpp:551-567: f64 if either side is float)
constexpr int XG_PREDS = 8, XG_IN = 16;
struct XgPred {
  int src;  // index of the predicate column's per-segment value array
  int flt;  // column values are f64
  int op;   // RQ_LT..RQ_GT, or -1 for IN
  int n_in;
  int kflt[XG_IN];
  int64_t ki[XG_IN];
  double kf[XG_IN];
};
struct XgPreds {
  int n;
  const uint64_t* val[XG_PREDS];
  XgPred p[XG_PREDS];
};
__device__ __forceinline__ bool xg_cmp1(uint64_t v, int vf, int64_t ki, double kf, int kflt, int op) {
  if (vf || kflt) {
    const double x = vf ? __longlong_as_double(static_cast<long long>(v)) : static_cast<double>(static_cast<int64_t>(v));
    const double k = kflt ? kf : static_cast<double>(ki);
    return cmp_t<double>(x, k, op);
  }
  return cmp_t<int64_t>(static_cast<int64_t>(v), ki, op);
}
__global__ void k_xg_where(const __grid_constant__ XgPreds W, int64_t n, uint8_t* __restrict__ flags) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    bool pass = true;
    for (int i = 0; i < W.n && pass; ++i) {
      const XgPred& P = W.p[i];
      const uint64_t v = __ldg(reinterpret_cast<const unsigned long long*>(W.val[P.src]) + k);
      if (P.op >= 0) {
        pass = xg_cmp1(v, P.flt, P.ki[0], P.kf[0], P.kflt[0], P.op);
      } else {
        bool any = false;
        for (int j = 0; j < P.n_in && !any; ++j) any = xg_cmp1(v, P.flt, P.ki[j], P.kf[j], P.kflt[j], RQ_EQ);
        pass = any;
      }
    }
    flags[k] = pass ? 1 : 0;
  }
}

// ---- k-way segment table (joint alignment of every run list in one pass) ----
//
// The joint shape of the key runs, the WHERE columns' runs, the mask's runs
// and the RLE operands' runs (align_many's left fold, align.cpp:233-254) is
// the set of fragments [max_l s_l(r_l), min_l e_l(r_l)] over one run r_l per
// list; every fragment ends at a run end of some list. So every run end x of
// every list is a candidate fragment end: it is kept when every list covers x
// (its run containing x starts at or before x), when no lower-numbered list
// also ends a run at x (one owner per fragment), and when the WHERE conjuncts
// pass on the lists' values at x. A candidate's position in the merged
// (stable, list-index tie-broken) order of all run ends is Σ_l lower_bound(e_l, x)
// plus the lower-numbered lists ending at x — known from the searches the
// coverage test does anyway — so the fragments come out in row order without
// a sort; two scans (kept flags, lengths) give every fragment's output slot
// and covered-row offset.
constexpr int KW_LISTS = 12;
constexpr int64_t KW_MAX_ROWS = int64_t{1} << 40;  // the look-back scan carries 40-bit prefixes
struct KwList {
  const int64_t* s;
  const int64_t* e;
  int64_t n;
  const void* v;  // run values (keys / predicate columns / RLE operands), or null
  int dt;
  int role;       // bits: 1 key, 2 predicate column, 4 RLE operand, 8 coverage only (mask / domain)
  int cst;        // RLE operand: index of its per-fragment value array
  int64_t kmin, stride;
  const int64_t* dir;  // rank directory of e (null: whole-list search)
  int dshift;
  int64_t dnb;
};
// A list's conjuncts on integer values folded on the host into one interval
// and at most one value set (IN lists intersected; NE values excluded), so a
// candidate tests two compares and a short set scan instead of interpreting
// every conjunct (compare_scalar's f64 semantics are exact here: every float
// literal is finite and below 2^52 in magnitude, kw_fold_conjuncts).
struct KwConj {
  int64_t lo, hi;  // lo <= v <= hi
  int nset;
  int set_in;      // 1: v must be in set; 0: v must not be
  int64_t set[XG_IN];
};
struct KwPlan {
  int nl;
  KwList l[KW_LISTS];
  int64_t start[KW_LISTS + 1];  // candidate index of each list's first run end
  int np;
  XgPred p[XG_PREDS];  // p.src = list index
  int own[KW_LISTS];   // list l has conjuncts: 1 folded (conj[l]), 2 interpreted (p[])
  KwConj conj[KW_LISTS];
};

// Rank directory of a sorted array of row positions a[0, n) over [0, total):
// dir[b] = lower_bound(a, b << shift) for b in [0, nb], so lower_bound(a, x)
// lies in [dir[x >> shift], dir[(x >> shift) + 1]] — a search over the few
// entries of one block instead of log2(n) dependent loads over the array.
// Thread i writes the blocks whose first row falls in (a[i-1], a[i]].
__global__ void k_rank_dir(const int64_t* __restrict__ a, int64_t n, int shift, int64_t nb,
                           int64_t* __restrict__ dir) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b0 = i == 0 ? 0 : (ldg64(a, i - 1) >> shift) + 1;
    const int64_t b1 = i == n ? nb : min(nb, ldg64(a, i) >> shift);
    for (int64_t b = b0; b <= b1; ++b) dir[b] = i;
  }
}

__device__ __forceinline__ int64_t kw_lower_bound_in(const int64_t* __restrict__ e, int64_t lo, int64_t hi,
                                                     int64_t x) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(e + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// lower_bound(e, x) through the directory when there is one (x >= 0)
__device__ __forceinline__ int64_t kw_lower_bound_dir(const int64_t* __restrict__ e, int64_t n,
                                                      const int64_t* __restrict__ dir, int shift, int64_t nb,
                                                      int64_t x) {
  if (!dir) return kw_lower_bound_in(e, 0, n, x);
  const int64_t b = x >> shift;
  if (b >= nb) return kw_lower_bound_in(e, ldg64(dir, nb), n, x);
  return kw_lower_bound_in(e, ldg64(dir, b), ldg64(dir, b + 1), x);
}

__device__ __forceinline__ int64_t kw_lower_bound(const int64_t* __restrict__ e, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(e + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint64_t kw_value_bits(const void* v, int dt, int64_t r) {
  return dt_is_float_dev(dt) ? static_cast<uint64_t>(__double_as_longlong(ld_f64(v, dt, r)))
                             : static_cast<uint64_t>(ld_i64(v, dt, r));
}

__device__ __forceinline__ bool kw_conj(const KwConj& C, int64_t v) {
  if (v < C.lo || v > C.hi) return false;
  // the set's own length bounds the scan (IN (3, 17, 42): three compares,
  // not XG_IN guarded ones)
  for (int t = 0; t < C.nset; ++t)
    if (C.set[t] == v) return C.set_in != 0;
  return C.set_in == 0;
}

__device__ __forceinline__ bool kw_pass(const XgPred& P, uint64_t v) {
  if (P.op >= 0) return xg_cmp1(v, P.flt, P.ki[0], P.kf[0], P.kflt[0], P.op);
  for (int t = 0; t < P.n_in; ++t)
    if (xg_cmp1(v, P.flt, P.ki[t], P.kf[t], P.kflt[t], RQ_EQ)) return true;
  return false;
}

// every conjunct of list l on value bits v
__device__ __forceinline__ bool kw_own(const KwPlan& K, int l, uint64_t v) {
  if (K.own[l] == 1) return kw_conj(K.conj[l], static_cast<int64_t>(v));
  bool keep = true;
#pragma unroll
  for (int q = 0; q < XG_PREDS; ++q)
    if (q < K.np && keep && K.p[q].src == l) keep = kw_pass(K.p[q], v);
  return keep;
}

// One thread per run end. `kept` is zeroed beforehand: a candidate that
// fails its own list's conjuncts, is not covered by some list, fails a
// conjunct of a list already located, or is not its fragment's owner
// returns early (most run ends of a selective WHERE never search the other
// lists); a kept one writes its fragment at its merged rank and adds to the
// (segments, covered rows) counters.
constexpr int KW_TILE = 2048;  // k_kway_select's tile (256 threads x 8 candidates)
// 8 resident CTAs per SM (32 registers, the per-list run indices partly in
// local memory): the pass is a set of dependent search chains, so warps in
// flight beat registers — C5 0.221 -> 0.206 ms per query against the
// compiler's 64-register / 4-CTA choice, Q6 unchanged
// (profiles/r2b_ab_kway_candidates.txt; 5 and 6 CTAs in between)
#ifndef RQ_KW_MINB
#define RQ_KW_MINB 8
#endif
__global__ void __launch_bounds__(256, RQ_KW_MINB) k_kway_candidates(const __grid_constant__ KwPlan K, uint8_t* __restrict__ kept,
                                  int64_t* __restrict__ seg_s, int64_t* __restrict__ seg_e,
                                  int64_t* __restrict__ seg_slot, uint64_t* __restrict__ seg_cst,
                                  unsigned long long* __restrict__ dims, unsigned long long* __restrict__ tagg,
                                  int64_t ntiles) {
  const int64_t N = K.start[K.nl];
  // (segments, covered rows) summed per block in shared memory, one global
  // atomic pair per block: every warp's pair on the same two addresses
  // serialised in L2
  __shared__ unsigned long long s_dims[2];
  if (threadIdx.x < 2) s_dims[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < N;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int j = 0;
    while (c >= K.start[j + 1]) ++j;
    const KwList& J = K.l[j];
    const int64_t i = c - K.start[j];
    const int64_t x = __ldg(J.e + i);
    bool keep = true;
    if (K.own[j]) keep = kw_own(K, j, kw_value_bits(J.v, J.dt, i));  // own conjuncts first: no search
    if (!keep) continue;
    int64_t rank = 0, start = __ldg(J.s + i);
    int64_t r[KW_LISTS];
#pragma unroll
    for (int l = 0; l < KW_LISTS; ++l) {  // unrolled: r[] stays in registers
      if (l >= K.nl || !keep) break;
      const KwList& L = K.l[l];
      if (l == j) {
        r[l] = i;
        rank += i;
        continue;
      }
      const int64_t rl = kw_lower_bound_dir(L.e, L.n, L.dir, L.dshift, L.dnb, x);
      if (rl >= L.n || __ldg(L.s + rl) > x) keep = false;          // x not covered by list l
      else if (l < j && __ldg(L.e + rl) == x) keep = false;        // a lower-numbered list owns this end
      if (!keep) break;
      start = max(start, __ldg(L.s + rl));
      r[l] = rl;
      rank += rl;
      if (K.own[l]) keep = kw_own(K, l, kw_value_bits(L.v, L.dt, rl));
    }
    if (!keep) continue;
    int64_t slot = 0;
#pragma unroll
    for (int l = 0; l < KW_LISTS; ++l) {
      if (l >= K.nl) break;
      const KwList& L = K.l[l];
      if (L.role & 1) slot += (ld_i64(L.v, L.dt, r[l]) - L.kmin) * L.stride;
      if (L.role & 4) seg_cst[static_cast<int64_t>(L.cst) * N + rank] = kw_value_bits(L.v, L.dt, r[l]);
    }
    kept[rank] = 1;
    seg_s[rank] = start;
    seg_e[rank] = x;
    seg_slot[rank] = slot;
    // (segments, covered rows) in total and per k_kway_select tile of ranks
    // (that kernel's tile offsets then come from a scan of these, not from a
    // look-back chain): one atomic pair per warp and per tile the warp touches
    const unsigned act = __activemask();
    const unsigned long long len = static_cast<unsigned long long>(x - start + 1);
    // len < 2^40: two 20-bit halves, each summed over <= 32 lanes without overflow
    const unsigned long long wl =
        __reduce_add_sync(act, static_cast<unsigned>(len & 0xfffffu)) +
        (static_cast<unsigned long long>(__reduce_add_sync(act, static_cast<unsigned>(len >> 20))) << 20);
    if ((threadIdx.x & 31) == __ffs(act) - 1) {
      atomicAdd(&s_dims[0], static_cast<unsigned long long>(__popc(act)));
      atomicAdd(&s_dims[1], wl);
    }
    const int64_t tile = rank / KW_TILE;
    const unsigned peers = __match_any_sync(act, static_cast<unsigned long long>(tile));
    const unsigned long long tl =
        __reduce_add_sync(peers, static_cast<unsigned>(len & 0xfffffu)) +
        (static_cast<unsigned long long>(__reduce_add_sync(peers, static_cast<unsigned>(len >> 20))) << 20);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) {
      atomicAdd(tagg + tile, static_cast<unsigned long long>(__popc(peers)));
      atomicAdd(tagg + ntiles + tile, tl);
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 && s_dims[threadIdx.x]) atomicAdd(dims + threadIdx.x, s_dims[threadIdx.x]);
}

// kept candidates → the segment table: each tile's first slot and covered-row
// offset come from the per-tile (count, rows) that k_kway_candidates
// accumulated — summed over the earlier tiles by the block itself when there
// are few tiles, else from their exclusive scan (tpre[t], tpre[ntiles + t] -
// tpre[ntiles]);
// inside the tile a block scan places every kept fragment, written there
// (s, e, slot, operand values at stride N, off). The totals stay on the
// device (dims): nothing is read back before the row kernels run.
// floor(a / b) for 0 <= a < 2^53, b > 0, without the 64-bit division
// sequence (~70 instructions): the double quotient is within one of the
// answer, one correction step each way
__device__ __forceinline__ int64_t div_floor_pos(int64_t a, int64_t b, double inv_b) {
  int64_t q = static_cast<int64_t>(static_cast<double>(a) * inv_b);
  if (q * b > a) --q;
  else if ((q + 1) * b <= a) ++q;
  return q;
}

// 5 resident CTAs per SM (<= 51 registers): the placement of a k-way table
// of up to 740 tiles runs in one wave (Q6: 684 tiles, C5: 458; at 72
// registers only 3 fitted and both ran a second, nearly empty wave)
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK, 5)
    k_kway_select(int64_t N, int ncst, const uint8_t* __restrict__ kept, const int64_t* __restrict__ cs,
                  const int64_t* __restrict__ ce, const int64_t* __restrict__ cslot, const uint64_t* __restrict__ ccst,
                  const int64_t* __restrict__ tpre, const int64_t* __restrict__ tagg, int64_t ntiles,
                  int64_t* __restrict__ s, int64_t* __restrict__ e,
                  int64_t* __restrict__ slot, uint64_t* __restrict__ cst, int64_t* __restrict__ off,
                  const int64_t* __restrict__ dims, int64_t nwarps, int64_t* __restrict__ cstart) {
  static_assert(BLOCK * ITEMS == KW_TILE, "tile of the per-tile aggregates");
  __shared__ uint64_t wn[BLOCK / 32 + 1], wr[BLOCK / 32 + 1];
  const int64_t base = (static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x) * ITEMS;
  unsigned keep = 0;  // kept items as bits (lengths re-derived from the reloaded s / e below)
  uint64_t cn = 0, cr = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t i = base + k;
    const bool kk = i < N && kept[i];
    keep |= kk ? 1u << k : 0u;
    cn += kk;
    cr += kk ? static_cast<uint64_t>(ldg64(ce, i) - ldg64(cs, i) + 1) : 0;
  }
  uint64_t tn, tr;
  uint64_t on = block_exclusive<BLOCK>(cn, tn, wn);
  uint64_t orow = block_exclusive<BLOCK>(cr, tr, wr);
  __shared__ uint64_t base_n, base_r;
  if (!tpre) {  // few tiles: this tile's prefix is the sum of the earlier tiles' aggregates
    uint64_t pn = 0, pr = 0;
    for (int64_t q = threadIdx.x; q < blockIdx.x; q += BLOCK) {
      pn += static_cast<uint64_t>(ldg64(tagg, q));
      pr += static_cast<uint64_t>(ldg64(tagg, ntiles + q));
    }
    pn = block_sum<BLOCK>(pn, wn);
    pr = block_sum<BLOCK>(pr, wr);
    if (threadIdx.x == 0) {
      base_n = pn;
      base_r = pr;
    }
  } else if (threadIdx.x == 0) {
    base_n = static_cast<uint64_t>(ldg64(tpre, blockIdx.x));
    base_r = static_cast<uint64_t>(ldg64(tpre, ntiles + blockIdx.x) - ldg64(tpre, ntiles));
  }
  __syncthreads();
  if (!cn) return;
  on += base_n;
  orow += base_r;
  const int64_t chunk = xg_chunk(ldg64(dims, 1), nwarps);  // the row kernels' chunk (same formula)
  const double inv_chunk = 1.0 / static_cast<double>(chunk);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (!((keep >> k) & 1u)) continue;
    const int64_t i = base + k, o = static_cast<int64_t>(on);
    const int64_t si = ldg64(cs, i), ei = ldg64(ce, i);
    const uint64_t len = static_cast<uint64_t>(ei - si + 1);
    s[o] = si;
    e[o] = ei;
    slot[o] = ldg64(cslot, i);
    for (int j = 0; j < ncst; ++j) cst[static_cast<int64_t>(j) * N + o] = __ldg(ccst + static_cast<int64_t>(j) * N + i);
    off[o] = static_cast<int64_t>(orow);
    // the row chunks whose first covered row falls in this segment start here
    const int64_t r0 = static_cast<int64_t>(orow), r1 = r0 + static_cast<int64_t>(len) - 1;
    const int64_t q1 = div_floor_pos(r1, chunk, inv_chunk);
    for (int64_t q = div_floor_pos(r0 + chunk - 1, chunk, inv_chunk); q <= q1; ++q) cstart[q] = o;
    ++on;
    orow += len;
  }
}

// Plain+Index operand: the outliers inside each segment, found by a binary
// search of the segment's start in the (sorted) outlier positions — the
// query touches only the outliers of selected rows — replace the base's
// decoded value (column.cpp:299-309); one add per segment (a segment has one
// slot)
__global__ void k_xg_outliers_seg(PlainSrc base, const int64_t* __restrict__ p, const void* __restrict__ v2, int v2dt,
                                  int64_t n, const int64_t* __restrict__ ss, const int64_t* __restrict__ se,
                                  const int64_t* __restrict__ seg_slot, int64_t nseg, const int64_t* __restrict__ dims,
                                  const int64_t* __restrict__ pdir, int pshift, int64_t pnb, int ne, int ei, int acc_f,
                                  unsigned long long* __restrict__ tab, double* __restrict__ part, int64_t cells) {
  if (dims) nseg = ldg64(dims, 0);
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  double* prow = part ? part + w * cells : nullptr;
  // one warp per segment (segments in order per warp): the lanes take the
  // segment's outliers 32 at a time, so a segment costs one search and a few
  // rounds of parallel loads instead of one serial walk per thread
  for (int64_t k = w; k < nseg; k += nw) {
    const int64_t a = ldg64(ss, k), b = ldg64(se, k);
    const int64_t cell = ldg64(seg_slot, k) * ne + ei;
    const int64_t i0 = kw_lower_bound_dir(p, n, pdir, pshift, pnb, a);
    double fd = 0.0;
    uint64_t id = 0;
    for (int64_t i = i0 + lane;; i += 32) {
      const int64_t pos = i < n ? ldg64(p, i) : INT64_MAX;
      const bool in = pos <= b;
      if (in) {
        if (acc_f) fd += ld_f64(v2, v2dt, i) - plain_value<double>(base, pos);
        else id += static_cast<uint64_t>(ld_i64(v2, v2dt, i)) - static_cast<uint64_t>(plain_value<int64_t>(base, pos));
      }
      if (!__all_sync(FULL, in)) break;  // the last lane passed the segment's end
    }
    if (acc_f) {
      fd = warp_sum(fd);  // a fixed butterfly: the same bits on every run
      if (lane == 0) {
        if (prow) prow[cell] += fd;
        else if (fd != 0.0) atomicAdd(reinterpret_cast<double*>(tab) + cell, fd);
      }
    } else {
      id = warp_sum(id);
      if (lane == 0 && id) atomicAdd(tab + cell, static_cast<unsigned long long>(id));
    }
  }
}
}  // namespace dev

namespace {

// 16-B aligned base and room for the 8-row vector groups past the last row
// (the generated kernel reads 8 rows per lane, the interpreted one 4)
bool xg_vec_ok(const DArr& a) {
  if (!a.buf || !a.buf->ptr) return a.n == 0;
  const size_t w = static_cast<size_t>(dt_width(a.dt));
  return (reinterpret_cast<uintptr_t>(a.buf->ptr) & 15) == 0 &&
         a.buf->cap >= static_cast<size_t>((a.n + 7) & ~int64_t(7)) * w;
}

// Several gathers in one launch, each array through its own index array (all
// of one length); each source may be of any dtype and lands as i64 / f64
// (segment-table columns). Replaces the arrays in place.
void gather_multi(const CtxPtr& ctx, const std::vector<std::pair<DArr*, const DArr*>>& items) {
  for (size_t a0 = 0; a0 < items.size(); a0 += dev::XG_GATHER) {
    dev::XgGather G{};
    std::vector<DArr> outs;
    const int64_t n = items[a0].second->n;
    for (size_t a = a0; a < items.size() && a < a0 + dev::XG_GATHER; ++a) {
      const DArr& src = *items[a].first;
      require(items[a].second->n == n, "gather_multi: index length mismatch");
      const int32_t odt = dt_float(src.dt) ? RQ_F64 : RQ_I64;
      outs.push_back(alloc_arr(ctx, odt, n));
      G.src[G.n] = src.raw();
      G.idx[G.n] = items[a].second->pos();
      G.dt[G.n] = src.dt;
      G.to_f[G.n] = odt == RQ_F64 ? 1 : 0;
      G.dst[G.n] = outs.back().raw_mut();
      ++G.n;
    }
    if (n) {
      dev::k_xg_gather<<<grid_cap(ctx, n), 256, 0, ctx->stream>>>(G, n);
      launched(ctx);
    }
    for (size_t a = a0; a < items.size() && a < a0 + dev::XG_GATHER; ++a) *items[a].first = outs[a - a0];
  }
}

void gather_many(const CtxPtr& ctx, const std::vector<DArr*>& arrs, const DArr& idx) {
  std::vector<std::pair<DArr*, const DArr*>> items;
  for (DArr* a : arrs) items.push_back({a, &idx});
  gather_multi(ctx, items);
}

// Key slot layout without building the key runs: slot = Σ (key − min)·stride
// over each key column's (cached) value range, first key most significant —
// the dense slots of build_key / build_multi_key.
bool key_layout(const CtxPtr& ctx, const std::vector<const DCol*>& keys, GroupKey& K) {
  K.G = 1;
  for (auto* k : keys) {
    if (k->enc != RQ_ENC_RLE || dt_float(k->v.dt) || k->v.n == 0) return false;
    auto mm = col_minmax(ctx, *k);
    const int64_t range = mm.second - mm.first + 1;
    if (range <= 0 || range > kFusedSlotLimit || K.G * range > kFusedSlotLimit) return false;
    K.kmin.push_back(mm.first);
    K.range.push_back(range);
    K.kdt.push_back(k->v.dt);
    K.G *= range;
  }
  K.stride.assign(keys.size(), 1);
  int64_t st = 1;
  for (size_t c = keys.size(); c-- > 0;) {
    K.stride[c] = st;
    st *= K.range[c];
  }
  return true;
}

// The rank directory of a column's sorted positions (run ends or index
// points), built on first use and kept on the column (columns are
// immutable): blocks of about four to eight elements' average span.
const DCol::RankDir& rank_dir(const CtxPtr& ctx, const DArr& a, int64_t total, DCol::RankDir& d) {
  if (d.shift >= 0 || a.n == 0 || total <= 0) return d;
  const int64_t avg = std::max<int64_t>(1, total / a.n);
  static const int extra = [] {  // RQ_DIR_SHIFT (A/B): log2 of average gaps per block
    const char* e = std::getenv("RQ_DIR_SHIFT");
    return e ? std::atoi(e) : 2;
  }();
  int sh = 0;  // floor(log2(avg)) + extra: a block spans 2^extra .. 2^(extra+1) average gaps
  while (sh < 38 && (int64_t{1} << (sh + 1)) <= avg) ++sh;
  sh = std::max(0, sh + extra);
  d.nb = ((total - 1) >> sh) + 1;
  d.dir = alloc_arr(ctx, RQ_I64, d.nb + 1);
  dev::k_rank_dir<<<grid_cap(ctx, a.n + 1), 256, 0, ctx->stream>>>(a.pos(), a.n, sh, d.nb, d.dir.as<int64_t>());
  launched(ctx);
  d.shift = sh;
  return d;
}

// Fold each list's conjuncts on integer values into KwConj (interval ∩ one
// value set); lists whose values are float, or with a float literal that is
// not finite or exceeds 2^52 in magnitude (where compare_scalar's f64
// rounding could differ from an integer compare), stay interpreted.
void kw_fold_conjuncts(dev::KwPlan& KP, const std::vector<int>& list_float) {
  constexpr double LIM = 4503599627370496.0;  // 2^52
  for (int l = 0; l < KP.nl; ++l) {
    if (!KP.own[l]) continue;
    KP.own[l] = 2;
    if (list_float[static_cast<size_t>(l)]) continue;
    int64_t lo = INT64_MIN, hi = INT64_MAX;
    bool have_in = false, ok = true;
    std::vector<int64_t> in, out;
    for (int q = 0; q < KP.np && ok; ++q) {
      const dev::XgPred& P = KP.p[q];
      if (P.src != l) continue;
      if (P.op >= 0) {
        int64_t k = P.ki[0];
        double kf = P.kf[0];
        if (P.kflt[0] && !(std::isfinite(kf) && std::fabs(kf) < LIM)) {
          ok = false;
          break;
        }
        // the integer bound equivalent to x op k (x integral)
        const bool integral = !P.kflt[0] || std::floor(kf) == kf;
        const int64_t fl = P.kflt[0] ? static_cast<int64_t>(std::floor(kf)) : k;
        const int64_t ce = P.kflt[0] ? static_cast<int64_t>(std::ceil(kf)) : k;
        switch (P.op) {
          case RQ_LT: if (ce == INT64_MIN) { lo = INT64_MAX; hi = INT64_MIN; } else hi = std::min(hi, ce - 1); break;
          case RQ_LE: hi = std::min(hi, fl); break;
          case RQ_GE: lo = std::max(lo, ce); break;
          case RQ_GT: if (fl == INT64_MAX) { lo = INT64_MAX; hi = INT64_MIN; } else lo = std::max(lo, fl + 1); break;
          case RQ_EQ:
            if (!integral) { lo = INT64_MAX; hi = INT64_MIN; }
            else { lo = std::max(lo, fl); hi = std::min(hi, fl); }
            break;
          case RQ_NE: if (integral) out.push_back(fl); break;
          default: ok = false;
        }
      } else {
        std::vector<int64_t> vals;
        for (int t = 0; t < P.n_in; ++t) {
          if (P.kflt[t]) {
            const double kf = P.kf[t];
            if (std::isnan(kf)) continue;  // never equal
            if (!(std::isfinite(kf) && std::fabs(kf) < LIM)) { ok = false; break; }
            if (std::floor(kf) != kf) continue;
            vals.push_back(static_cast<int64_t>(kf));
          } else {
            vals.push_back(P.ki[t]);
          }
        }
        if (!have_in) {
          in = vals;
          have_in = true;
        } else {
          std::vector<int64_t> keep;
          for (int64_t v : in)
            if (std::find(vals.begin(), vals.end(), v) != vals.end()) keep.push_back(v);
          in.swap(keep);
        }
      }
    }
    if (!ok) continue;
    dev::KwConj& C = KP.conj[l];
    C.lo = lo;
    C.hi = hi;
    if (have_in) {
      std::vector<int64_t> keep;
      for (int64_t v : in)
        if (v >= lo && v <= hi && std::find(out.begin(), out.end(), v) == out.end() &&
            std::find(keep.begin(), keep.end(), v) == keep.end())
          keep.push_back(v);
      if (keep.empty()) {  // nothing passes
        C.lo = 1;
        C.hi = 0;
      }
      if (keep.size() > static_cast<size_t>(dev::XG_IN)) continue;
      C.nset = static_cast<int>(keep.size());
      C.set_in = 1;
      for (size_t t = 0; t < keep.size(); ++t) C.set[t] = keep[t];
    } else {
      std::vector<int64_t> ex;
      for (int64_t v : out)
        if (v >= lo && v <= hi && std::find(ex.begin(), ex.end(), v) == ex.end()) ex.push_back(v);
      if (ex.size() > static_cast<size_t>(dev::XG_IN)) continue;
      C.nset = static_cast<int>(ex.size());
      C.set_in = 0;
      for (size_t t = 0; t < ex.size(); ++t) C.set[t] = ex[t];
    }
    KP.own[l] = 1;
  }
}

// The segment table in one pass over every run list (k_kway_candidates +
// k_kway_select): s / e / slot / per-segment RLE-operand values / covered-row
// offsets, sized by their capacity `cap` (the candidate count) with the real
// (segments, covered rows) left on the device in `dims` — no readback.
// Returns false when the lists do not fit the kernel (the pairwise path then
// builds the table).
bool kway_segments(const CtxPtr& ctx, const std::vector<const DCol*>& keys, const DMask* mask,
                   const std::vector<XPred>* preds, const std::vector<const DCol*>& rle_cols, int64_t total,
                   GroupKey& K, DArr& s, DArr& e, DArr& slot, DArr& cst_all, DArr& off, DArr& dims,
                   DArr& cstart, int64_t& cap) {
  if (total <= 0 || total >= dev::KW_MAX_ROWS) return false;
  auto host_timer = std::make_unique<KTimer>(ctx, "kw_host");  // the plan, up to the first launch
  if (!key_layout(ctx, keys, K)) return false;
  dev::KwPlan KP{};
  std::vector<const DCol*> of_list;  // the column behind each list (null: mask / domain)
  auto add = [&](const DArr& ls, const DArr& le, const DCol* col) -> int {
    for (int l = 0; l < KP.nl; ++l)  // one list per column, whatever its roles
      if (col && of_list[l] && (of_list[l] == col || (of_list[l]->v.raw() == col->v.raw() &&
                                                      of_list[l]->e.raw() == col->e.raw())))
        return l;
    if (KP.nl >= dev::KW_LISTS) return -1;
    dev::KwList& L = KP.l[KP.nl];
    L.s = ls.pos();
    L.e = le.pos();
    L.n = le.n;
    L.v = col ? col->v.raw() : nullptr;
    L.dt = col ? col->v.dt : RQ_I64;
    L.role = 0;
    L.cst = -1;
    L.dir = nullptr;
    if (col) {
      const DCol::RankDir& d = rank_dir(ctx, le, col->total, col->dir_e);
      if (d.shift >= 0) {
        L.dir = d.dir.pos();
        L.dshift = d.shift;
        L.dnb = d.nb;
      }
    }
    of_list.push_back(col);
    return KP.nl++;
  };
  for (size_t c = 0; c < keys.size(); ++c) {
    const int l = add(keys[c]->s, keys[c]->e, keys[c]);
    if (l < 0 || (KP.l[l].role & 1)) return false;  // the same column twice as a key
    KP.l[l].role |= 1;
    KP.l[l].kmin = K.kmin[c];
    KP.l[l].stride = K.stride[c];
  }
  DArr ms, me;  // the mask's true rows as runs
  if (mask) {
    if (mask->enc == RQ_MASK_RLE) {
      ms = mask->s;
      me = mask->e;
    } else if (mask->enc == RQ_MASK_PLAIN) {
      plain_mask_to_rle(ctx, mask->bits, ms, me);
    } else if (mask->enc == RQ_MASK_INDEX) {
      ms = me = mask->p;
    } else {
      return false;
    }
    if (add(ms, me, nullptr) < 0) return false;
  }
  const size_t npred = preds ? preds->size() : 0;
  for (size_t i = 0; i < npred; ++i) {
    const XPred& q = (*preds)[i];
    const int l = add(q.col->s, q.col->e, q.col);
    if (l < 0) return false;
    KP.l[l].role |= 2;
    dev::XgPred& P = KP.p[KP.np++];
    P.src = l;
    KP.own[l] = 1;
    P.flt = dt_float(q.col->v.dt) ? 1 : 0;
    P.op = q.in.empty() ? q.op : -1;
    const std::vector<Scalar> one{q.k};
    const std::vector<Scalar>& ks = q.in.empty() ? one : q.in;
    P.n_in = static_cast<int>(ks.size());
    for (size_t j = 0; j < ks.size(); ++j) {
      P.kflt[j] = ks[j].is_float ? 1 : 0;
      P.ki[j] = ks[j].i;
      P.kf[j] = ks[j].f;
    }
  }
  {
    std::vector<int> list_float(static_cast<size_t>(KP.nl), 0);
    for (int l = 0; l < KP.nl; ++l) list_float[static_cast<size_t>(l)] = dt_float(KP.l[l].dt) ? 1 : 0;
    kw_fold_conjuncts(KP, list_float);
  }
  for (size_t j = 0; j < rle_cols.size(); ++j) {
    const int l = add(rle_cols[j]->s, rle_cols[j]->e, rle_cols[j]);
    if (l < 0) return false;
    if (KP.l[l].role & 4) return false;  // two operand slots on one list: pairwise path
    KP.l[l].role |= 4;
    KP.l[l].cst = static_cast<int>(j);
  }
  DArr dom_s, dom_e;
  if (KP.nl == 0) {  // no run list at all: the whole domain is one segment
    const int64_t z = 0, t1 = total - 1;
    dom_s = upload_arr(ctx, RQ_I64, &z, 1);
    dom_e = upload_arr(ctx, RQ_I64, &t1, 1);
    add(dom_s, dom_e, nullptr);
  }
  // role bits → the kernel's roles (0 key, 1 predicate, 2 operand, 3 coverage): a
  // list may carry several; the kernel reads them as bits too
  for (int l = 0; l < KP.nl; ++l) {
    KP.l[l].role = KP.l[l].role == 0 ? 8 : KP.l[l].role;
    if (!(KP.l[l].role & 4)) KP.l[l].cst = -1;
  }
  KP.start[0] = 0;
  for (int l = 0; l < KP.nl; ++l) KP.start[l + 1] = KP.start[l] + KP.l[l].n;
  const int64_t N = KP.start[KP.nl];
  if (N + total >= dev::KW_MAX_ROWS) return false;  // the tile scan runs (counts | rows) as one 40-bit prefix
  const int ncst = static_cast<int>(rle_cols.size());
  host_timer.reset();
  dims = alloc_arr(ctx, RQ_I64, 2);
  RQ_CUDA_CHECK(cudaMemsetAsync(dims.raw_mut(), 0, 16, ctx->stream));
  // the table is sized by its capacity N (every candidate kept); the real
  // (segments, covered rows) stay in `dims` on the device
  s = alloc_arr(ctx, RQ_I64, N);
  e = alloc_arr(ctx, RQ_I64, N);
  slot = alloc_arr(ctx, RQ_I64, N);
  off = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, N));
  cst_all = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, N * ncst));
  // the row kernels' grid (xg_fused: same average-length estimate, total / capacity)
  const int64_t nwarps = static_cast<int64_t>(ctx->sm_count) * xg_row_blocks_per_sm(total / std::max<int64_t>(1, N)) * 8;
  cstart = alloc_arr(ctx, RQ_I64, nwarps + 1);
  cap = N;
  if (N == 0) return true;
  constexpr int B = 256, IT = dev::KW_TILE / 256;
  const int64_t ntiles = (N + dev::KW_TILE - 1) / dev::KW_TILE;
  // the per-tile (count, rows) aggregates, then the kept flags: one zeroing memset
  const int64_t words = 2 * ntiles + (N + 7) / 8;
  DArr zero = alloc_arr(ctx, RQ_I64, words), cs = alloc_arr(ctx, RQ_I64, N), ce = alloc_arr(ctx, RQ_I64, N),
       cslot = alloc_arr(ctx, RQ_I64, N), ccst = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, N * ncst));
  RQ_CUDA_CHECK(cudaMemsetAsync(zero.raw_mut(), 0, static_cast<size_t>(words) * 8, ctx->stream));
  auto* tagg = zero.as<unsigned long long>();
  auto* kept = reinterpret_cast<uint8_t*>(tagg + 2 * ntiles);
  dev::k_kway_candidates<<<grid_cap(ctx, N), 256, 0, ctx->stream>>>(
      KP, kept, cs.as<int64_t>(), ce.as<int64_t>(), cslot.as<int64_t>(), ccst.as<uint64_t>(),
      dims.as<unsigned long long>(), tagg, ntiles);
  launched(ctx);
  DArr tv = zero;  // the aggregates (the buffer's head), then — many tiles — their exclusive scan
  tv.n = 2 * ntiles;
  DArr tpre;
  if (ntiles > 2048) scan_exclusive_i64(ctx, tv, tpre);
  dev::k_kway_select<B, IT><<<static_cast<unsigned>(ntiles), B, 0, ctx->stream>>>(
      N, ncst, kept, cs.pos(), ce.pos(), cslot.pos(), ccst.as<uint64_t>(), tpre.n ? tpre.pos() : nullptr,
      tv.pos(), ntiles, s.as<int64_t>(),
      e.as<int64_t>(), slot.as<int64_t>(), cst_all.as<uint64_t>(), off.as<int64_t>(), dims.pos(), nwarps,
      cstart.as<int64_t>());
  launched(ctx);
  return true;
}

// ---- CUDA graphs of repeated plans ------------------------------------------------
//
// A query plan re-run on the same user handles (the C API sets ctx->graph_key
// from the handles' ids, the expressions, literals and functions) launches the
// same kernels on the same columns. The launches from the segment table to the
// row folds have no host readback when the k-way builder makes the table, so
// the second such call captures them into a CUDA graph and later calls replay
// it: one launch instead of ~10 (Q6 / C5 were host-paced). The graph keeps
// every block its kernels touch (freed blocks are held, not recycled); the
// accumulators it fills (tab, cnt) are read by the host-side tail of the call
// as before. A profiled region inside is a pair of event nodes; each replay's
// time is read before the next replay re-records them. RQ_NO_GRAPH=1
// disables graphs (A/B).
struct XgGraph : Ctx::GraphEntry {
  Ctx* ctx = nullptr;
  int seen = 0;
  bool capturable = true;
  cudaGraphExec_t exec = nullptr;
  std::vector<Ctx::CapTimer> timers;  // event nodes of the profiled regions (owned)
  std::vector<std::pair<void*, size_t>> owned;
  GroupKey K;
  void* tab = nullptr;
  void* cnt = nullptr;
  size_t tab_cap = 0, cnt_cap = 0;
  int64_t tab_n = 0, cnt_n = 0;
  int64_t nlaunch = 0;
  ~XgGraph() override {
    if (exec) cudaGraphExecDestroy(exec);
    for (auto& t : timers) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    for (auto& b : owned) ctx->free(b.first, b.second);
  }
  // one launch; the previous run's region times are read first (the replay
  // re-records the same events)
  void replay(Ctx& c) {
    for (auto& t : timers) c.read_graph_timer(t.a);
    RQ_CUDA_CHECK(cudaGraphLaunch(exec, c.stream));
    for (auto& t : timers) c.graph_timers_unread.push_back(t);
    c.count_launch(static_cast<int>(nlaunch));
  }
};

// a non-owning view of a block the graph keeps
DArr graph_view(const CtxPtr& ctx, void* p, size_t cap, int64_t n) {
  DArr a;
  a.dt = RQ_I64;
  a.n = n;
  a.buf = std::make_shared<Buffer>();
  a.buf->ctx = ctx;
  a.buf->ptr = p;
  a.buf->bytes = static_cast<size_t>(n) * 8;
  a.buf->cap = cap;
  a.buf->owned = false;
  return a;
}

// Runs `middle` (returns 0: plan not fusable) directly, by capturing it, or by
// replaying its graph; K / tab / cnt / kway are its outputs.
template <class F>
bool run_graph(const CtxPtr& ctx, bool allowed, F& middle, GroupKey& K, DArr& tab, DArr& cnt, bool& kway) {
  std::string key;
  key.swap(ctx->graph_key);  // consumed by the first fused pass of the call
  static const bool off = std::getenv("RQ_NO_GRAPH") != nullptr;
  if (key.empty() || off || !allowed) return middle() != 0;
  if (ctx->profiling) {  // graphs captured with and without event nodes are distinct
    key += "|prof";
    for (const auto& t : ctx->profile_only) key += "," + t;
  }
  auto it = ctx->graphs.find(key);
  if (it == ctx->graphs.end()) {
    if (ctx->graphs.size() >= 16) ctx->drop_graphs();  // bounded: drop them all (after a sync)
    auto fresh = std::make_shared<XgGraph>();
    fresh->ctx = ctx.get();
    it = ctx->graphs.emplace(key, fresh).first;
  }
  auto* g = static_cast<XgGraph*>(it->second.get());
  if (g->exec) {  // replay
    g->replay(*ctx);
    K = g->K;
    tab = graph_view(ctx, g->tab, g->tab_cap, g->tab_n);
    cnt = graph_view(ctx, g->cnt, g->cnt_cap, g->cnt_n);
    kway = true;
    return true;
  }
  if (g->seen == 0 || !g->capturable) {  // first call: run it, note whether it can be captured
    ++g->seen;
    const bool ok = middle() != 0;
    g->capturable = g->capturable && ok && kway;
    return ok;
  }
  // second call: capture, then replay
  ctx->capture_owned.clear();
  ctx->capture_timers.clear();
  ctx->capture_broken = false;
  RQ_CUDA_CHECK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
  ctx->capturing = true;
  const int64_t l0 = ctx->launches;
  int r = 0;
  bool threw = false;
  try {
    r = middle();
  } catch (...) {
    threw = true;
  }
  ctx->capturing = false;
  cudaGraph_t graph = nullptr;
  if (cudaStreamEndCapture(ctx->stream, &graph) != cudaSuccess) {
    cudaGetLastError();
    ctx->capture_broken = true;
  }
  cudaGraphExec_t exec = nullptr;
  const bool ok = !threw && r == 1 && kway && !ctx->capture_broken && graph &&
                  cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  auto timers = std::move(ctx->capture_timers);
  ctx->capture_timers.clear();
  if (!ok) {  // not capturable after all: release what the capture held, run it directly
    cudaGetLastError();
    if (exec) cudaGraphExecDestroy(exec);
    for (auto& t : timers) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    auto owned = std::move(ctx->capture_owned);
    ctx->capture_owned.clear();
    for (auto& b : owned) ctx->free(b.first, b.second);  // nothing ran: safe to recycle
    g->capturable = false;
    K = GroupKey();
    tab = cnt = DArr();
    return middle() != 0;
  }
  g->exec = exec;
  g->timers = std::move(timers);
  g->owned = std::move(ctx->capture_owned);
  ctx->capture_owned.clear();
  g->nlaunch = ctx->launches - l0;
  ctx->launches = l0;  // counted when the graph runs (replay)
  g->K = K;  // the layout only: no arrays held (they would keep the context alive)
  g->K.s = g->K.e = g->K.slot = DArr();
  // the accumulators now belong to the graph; this call reads them through views
  g->tab = tab.raw_mut();
  g->tab_cap = tab.buf->cap;
  g->tab_n = tab.n;
  tab.buf->owned = false;
  g->owned.push_back({g->tab, g->tab_cap});
  g->cnt = cnt.raw_mut();
  g->cnt_cap = cnt.buf->cap;
  g->cnt_n = cnt.n;
  cnt.buf->owned = false;
  g->owned.push_back({g->cnt, g->cnt_cap});
  g->replay(*ctx);
  return true;
}

bool xg_fused(const CtxPtr& ctx, const DMask* mask, const std::vector<const DCol*>& keys,
              const std::vector<XExpr>& exprs, const std::vector<int>& fns, GroupAggOut& out,
              const GroupKey* preK, const std::vector<XPred>* preds) {
  if (exprs.size() > static_cast<size_t>(dev::XG_EXPRS) || keys.size() > 8) return false;
  auto plan_timer = std::make_unique<KTimer>(ctx, "xg_plan");  // host-side planning (profiling only)
  const int64_t total = !keys.empty() ? keys[0]->total
                        : mask        ? mask->total
                                      : (exprs.empty() || exprs[0].terms.empty() ? -1 : exprs[0].terms[0].col->total);
  if (total < 0) return false;
  if (mask && (mask->total != total || mask->enc == RQ_MASK_COMPOSITE)) return false;
  const size_t npred = preds ? preds->size() : 0;
  if (npred > static_cast<size_t>(dev::XG_PREDS)) return false;
  for (size_t i = 0; i < npred; ++i) {
    const XPred& q = (*preds)[i];
    if (q.col->enc != RQ_ENC_RLE || q.col->total != total || q.in.size() > static_cast<size_t>(dev::XG_IN)) return false;
    if (q.in.empty() && (q.op < RQ_LT || q.op > RQ_GT)) return false;
  }
  for (int f : fns)
    if (f != RQ_SUM && f != RQ_AVG && f != RQ_COUNT) return false;
  for (auto* k : keys)
    if (k->enc != RQ_ENC_RLE || dt_float(k->v.dt) || k->total != total) return false;

  dev::XgPlan P{};
  std::vector<const DCol*> plain_cols, rle_cols;
  std::vector<std::pair<int, const DCol*>> pi_exprs;  // (expr, Plain+Index column)
  auto col_slot = [](std::vector<const DCol*>& v, const DCol* c, int cap) -> int {
    for (size_t i = 0; i < v.size(); ++i)  // the same column (possibly through another handle)
      if (v[i] == c || (v[i]->enc == c->enc && v[i]->v.raw() == c->v.raw() && v[i]->e.raw() == c->e.raw()))
        return static_cast<int>(i);
    if (static_cast<int>(v.size()) >= cap) return -1;
    v.push_back(c);
    return static_cast<int>(v.size()) - 1;
  };
  P.ne = static_cast<int>(exprs.size());
  for (size_t i = 0; i < exprs.size(); ++i) {
    const XExpr& x = exprs[i];
    dev::XgExpr& X = P.e[i];
    X.nt = static_cast<int>(x.terms.size());
    if (X.nt > 3 || static_cast<int>(x.ops.size()) != std::max(0, X.nt - 1)) return false;
    if (X.nt == 0 && fns[i] != RQ_COUNT) return false;
    int vf = 0;
    for (int t = 0; t < X.nt; ++t) {
      const XTerm& tm = x.terms[static_cast<size_t>(t)];
      const DCol& c = *tm.col;
      if (c.total != total) return false;
      dev::XgTerm& T = X.t[t];
      T.sop = tm.sop;
      T.rev = tm.rev ? 1 : 0;
      T.kflt = tm.k.is_float ? 1 : 0;
      T.ki = tm.k.i;
      T.kf = tm.k.f;
      if (tm.sop >= 0 && (tm.sop < RQ_ADD || tm.sop > RQ_DIV)) return false;
      if (c.enc == RQ_ENC_PLAIN || c.enc == RQ_ENC_PLAIN_INDEX) {
        if (c.enc == RQ_ENC_PLAIN_INDEX) {  // bare column SUM / AVG only
          if (X.nt != 1 || tm.sop >= 0) return false;
          pi_exprs.push_back({static_cast<int>(i), &c});
        }
        if (!xg_vec_ok(c.v)) return false;
        const int ci = col_slot(plain_cols, &c, dev::XG_COLS);
        if (ci < 0) return false;
        T.src = ci;
        T.flt = (dt_float(c.v.dt) || dt_float(c.logical)) ? 1 : 0;
        X.rows = 1;
      } else if (c.enc == RQ_ENC_RLE) {
        const int ri = col_slot(rle_cols, &c, dev::XG_CONSTS);
        if (ri < 0) return false;
        T.src = dev::XG_COLS + ri;
        T.flt = dt_float(c.v.dt) ? 1 : 0;
      } else {
        return false;  // Index / RLE+Index operands: operator chain
      }
      const int yf = T.flt || (T.sop >= 0 && T.kflt);
      if (t > 0) {
        X.op[t - 1] = x.ops[static_cast<size_t>(t - 1)];
        if (X.op[t - 1] < RQ_ADD || X.op[t - 1] > RQ_DIV) return false;
      }
      vf = vf || yf;
    }
    X.res_f = vf;
    X.acc_f = vf ? 1 : 0;  // integer results (AVG too) sum exactly in int64
  }
  // plain columns referenced by a Plain+Index expression are read as their base
  P.nc = static_cast<int>(plain_cols.size());
  for (size_t c = 0; c < plain_cols.size(); ++c) P.col[c] = plain_src(*plain_cols[c]);
  P.ncst = static_cast<int>(rle_cols.size());
  for (size_t j = 0; j < rle_cols.size(); ++j) P.cst_f[j] = dt_float(rle_cols[j]->v.dt) ? 1 : 0;

  // ---- segment table: keys ∩ mask ∩ WHERE ∩ RLE operands (align_many's joint shape) ----
  plan_timer.reset();
  KTimer timer(ctx, "group_exprs");
  GroupKey K;
  DArr tab, cnt;
  int* err = reinterpret_cast<int*>(ctx->tickets + 2);  // zero between launches (reset after the check)
  bool kway = false;
  // The plan's launches from the segment table to the row folds: no host
  // readback when the k-way builder makes the table, so a repeated call on
  // the same user handles replays them as one CUDA graph (run_graph below).
  auto middle = [&]() -> int {
    DArr s, e, slot, cst_all, off, dims, cstart;
    int64_t nseg = 0, ncov = 0;  // host-known sizes (pairwise builder); the k-way one leaves them in dims
    kway = !preK && kway_segments(ctx, keys, mask, preds, rle_cols, total, K, s, e, slot, cst_all, off, dims,
                                  cstart, nseg);
    if (!kway) {
      auto stage = std::make_unique<KTimer>(ctx, "xg_keys");  // per-stage profile tags (no-ops unless profiling)
      if (preK) {
        K = *preK;
      } else if (!keys.empty()) {
        if (!(keys.size() == 1 ? build_key(ctx, keys, K) : build_multi_key(ctx, keys, K))) return 0;
      } else {
        if (total == 0) return 0;
        // one run [0, total) in slot 0 (one device fill: no host staging)
        K.s = alloc_arr(ctx, RQ_I64, 1);
        K.e = alloc_arr(ctx, RQ_I64, 1);
        K.slot = alloc_arr(ctx, RQ_I64, 1);
        dev::k_xg_fill3<<<1, 1, 0, ctx->stream>>>(K.s.as<int64_t>(), 0, K.e.as<int64_t>(), total - 1,
                                                  K.slot.as<int64_t>(), 0);
        launched(ctx);
        K.G = 1;
      }
      stage = std::make_unique<KTimer>(ctx, "xg_where");
      s = K.s;
      e = K.e;
      slot = K.slot;
      std::vector<DArr> cst;
      if (mask) {
        // the mask's true rows as runs: RLE as is, a plain byte mask through
        // plain_mask_to_rle (primitives.cpp:349-360), index points as 1-row runs
        DArr ms = mask->s, me = mask->e;
        if (mask->enc == RQ_MASK_PLAIN) plain_mask_to_rle(ctx, mask->bits, ms, me);
        else if (mask->enc == RQ_MASK_INDEX) ms = me = mask->p;
        Intersection r = range_intersect(ctx, s, e, ms, me, true, false);
        slot = gather(ctx, slot, r.idx1);
        s = r.s;
        e = r.e;
      }
      if (npred) {
        // WHERE pushdown: the segments are intersected with each distinct
        // predicate column's runs (fewest runs first) and the passing segments
        // kept; before a column with many runs the segments are pruned by the
        // conjuncts already evaluable, so the large intersection runs on the
        // selected segments only.
        std::vector<const DCol*> pcols;  // distinct predicate columns
        std::vector<int> pcol_of(npred);
        for (size_t i = 0; i < npred; ++i) {
          const XPred& q = (*preds)[i];
          int src = -1;
          for (size_t j = 0; j < pcols.size(); ++j)
            if (pcols[j] == q.col || (pcols[j]->v.raw() == q.col->v.raw() && pcols[j]->e.raw() == q.col->e.raw()))
              src = static_cast<int>(j);
          if (src < 0) {
            pcols.push_back(q.col);
            src = static_cast<int>(pcols.size()) - 1;
          }
          pcol_of[i] = src;
        }
        std::vector<int> order(pcols.size());
        for (size_t j = 0; j < order.size(); ++j) order[j] = static_cast<int>(j);
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return pcols[x]->e.n < pcols[y]->e.n; });
        std::vector<int> slot_of(pcols.size(), -1);  // predicate column -> its value array in pv
        std::vector<DArr> pv;
        // keep the segments passing every conjunct whose column is already joined in
        auto prune = [&]() {
          dev::XgPreds W{};
          for (size_t i = 0; i < npred; ++i) {
            const int src = slot_of[pcol_of[i]];
            if (src < 0) continue;
            const XPred& q = (*preds)[i];
            dev::XgPred& P = W.p[W.n++];
            P.src = src;
            P.flt = dt_float(q.col->v.dt) ? 1 : 0;
            P.op = q.in.empty() ? q.op : -1;
            const std::vector<Scalar> one{q.k};
            const std::vector<Scalar>& ks = q.in.empty() ? one : q.in;
            P.n_in = static_cast<int>(ks.size());
            for (size_t j = 0; j < ks.size(); ++j) {
              P.kflt[j] = ks[j].is_float ? 1 : 0;
              P.ki[j] = ks[j].i;
              P.kf[j] = ks[j].f;
            }
          }
          for (size_t j = 0; j < pv.size(); ++j) W.val[j] = reinterpret_cast<const uint64_t*>(pv[j].raw());
          if (!s.n || !W.n) return;
          DArr flags = alloc_arr(ctx, RQ_I8, s.n);
          dev::k_xg_where<<<grid_cap(ctx, s.n), 256, 0, ctx->stream>>>(W, s.n, flags.as<uint8_t>());
          launched(ctx);
          DArr keep;
          flagged_indices(ctx, flags, s.n, keep);
          std::vector<DArr*> g{&s, &e, &slot};
          for (auto& v : pv) g.push_back(&v);
          gather_many(ctx, g, keep);
        };
        for (size_t oi = 0; oi < order.size(); ++oi) {
          const DCol* col = pcols[order[oi]];
          if (oi > 0 && col->e.n >= 65536 && s.n > 0 && col->e.n >= 16 * s.n) prune();
          Intersection r = range_intersect(ctx, s, e, col->s, col->e, true, true);
          DArr nv = col->v;  // segment tables through idx1, the column's values through idx2: one launch
          std::vector<std::pair<DArr*, const DArr*>> g{{&slot, &r.idx1}};
          for (auto& v : pv) g.push_back({&v, &r.idx1});
          g.push_back({&nv, &r.idx2});
          gather_multi(ctx, g);
          pv.push_back(nv);
          slot_of[order[oi]] = static_cast<int>(pv.size()) - 1;
          s = r.s;
          e = r.e;
        }
        prune();
      }
      stage = std::make_unique<KTimer>(ctx, "xg_operands");
      for (const DCol* rc : rle_cols) {
        Intersection r = range_intersect(ctx, s, e, rc->s, rc->e, true, true);
        DArr nv = rc->v;
        std::vector<std::pair<DArr*, const DArr*>> g{{&slot, &r.idx1}};
        for (auto& c : cst) g.push_back({&c, &r.idx1});
        g.push_back({&nv, &r.idx2});
        gather_multi(ctx, g);
        cst.push_back(nv);
        s = r.s;
        e = r.e;
      }
      stage = std::make_unique<KTimer>(ctx, "xg_prep");
      nseg = s.n;
      cst_all = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, nseg * static_cast<int64_t>(cst.size())));
      for (size_t j = 0; j < cst.size(); ++j)
        if (nseg)
          RQ_CUDA_CHECK(cudaMemcpyAsync(cst_all.as<int64_t>() + j * nseg, cst[j].raw(), nseg * 8,
                                        cudaMemcpyDeviceToDevice, ctx->stream));
      off = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, nseg));
      if (nseg) {
        // lengths plus a trailing 0: the exclusive scan's last entry is the covered-row total
        DArr len = alloc_arr(ctx, RQ_I64, nseg + 1);
        dev::k_xg_lengths<<<grid_cap(ctx, nseg + 1), 256, 0, ctx->stream>>>(s.pos(), e.pos(), nseg, len.as<int64_t>());
        launched(ctx);
        scan_exclusive_i64(ctx, len, off);
        ncov = *ctx->readback(off.as<int64_t>() + nseg, 8);
      }
    }
    auto stage = std::make_unique<KTimer>(ctx, "xg_prep");
    const int64_t G = K.G;
    const int64_t cells = G * P.ne;
    if (cells > (int64_t{1} << 26)) return 0;
    tab = new_table(ctx, std::max<int64_t>(1, cells), 0);
    cnt = new_table(ctx, G, 0);
    // k-way: nseg is the table's capacity, the counts are read on the device
    dev::XgSegs S{s.pos(), e.pos(), off.pos(),  slot.pos(), reinterpret_cast<const uint64_t*>(cst_all.raw()),
                  nseg,    ncov,    nullptr,    0,          kway ? dims.pos() : nullptr,
                  nseg,    kway ? cstart.pos() : nullptr};
    // average covered segment length (the row kernel's prefetch choice): the
    // k-way table's is estimated as rows per candidate
    const int64_t avg_len = kway ? total / std::max<int64_t>(1, nseg) : ncov / std::max<int64_t>(1, nseg);
    auto* tabp = reinterpret_cast<unsigned long long*>(tab.raw_mut());
    auto* cntp = reinterpret_cast<unsigned long long*>(cnt.raw_mut());
    DArr dpart;
    int64_t dchunks = 0;
    // f64 expressions over RLE operands only: per-warp partial rows + a
    // fixed-order fold (bit-identical results; atomics past the budget)
    auto f64_part = [&](int blocks, DArr& part) -> double* {
      const int64_t rows = static_cast<int64_t>(blocks) * 8;
      if (rows * cells > (int64_t{8} << 20)) return nullptr;
      part = alloc_arr(ctx, RQ_F64, rows * cells);
      RQ_CUDA_CHECK(cudaMemsetAsync(part.raw_mut(), 0, static_cast<size_t>(rows * cells) * 8, ctx->stream));
      return part.as<double>();
    };
    // keyless plans of row-evaluated SUMs read neither the per-slot row counts
    // nor any per-segment term: no segment pass (Q6: one launch less)
    static const bool always_segs = std::getenv("RQ_XG_ALWAYS_SEGS") != nullptr;  // A/B knob
    bool need_segs = always_segs || !keys.empty();
    for (int i = 0; i < P.ne; ++i)
      need_segs = need_segs || !P.e[i].rows || P.e[i].nt == 0 || fns[static_cast<size_t>(i)] != RQ_SUM;
    if (nseg && need_segs) {
      dev::XgIsF sf{};
      bool any_sf = false;
      for (int i = 0; i < P.ne; ++i) {
        sf.f[i] = !P.e[i].rows && P.e[i].nt > 0 && P.e[i].acc_f;
        any_sf = any_sf || sf.f[i];
      }
      const int gs = grid_cap(ctx, nseg);
      DArr spart;
      double* sp = any_sf ? f64_part(gs, spart) : nullptr;
      dev::k_xg_segs<<<gs, 256, 0, ctx->stream>>>(P, S, tabp, cntp, err, sp, cells);
      launched(ctx);
      if (sp) {
        dev::k_xg_dfold<<<static_cast<unsigned>(cells), dev::DFOLD_B, 0, ctx->stream>>>(sp, int64_t{gs} * 8, cells, P.ne, sf,
                                                                               tabp);
        launched(ctx);
      }
    }
    bool any_rows = false;
    for (int i = 0; i < P.ne; ++i) any_rows = any_rows || P.e[i].rows;
    stage.reset();
    if (any_rows && (kway ? nseg > 0 : ncov > 0)) {
      constexpr int B = 256;
      const int bps = xg_row_blocks_per_sm(avg_len);
      const int64_t warps = static_cast<int64_t>(ctx->sm_count) * bps * (B / 32);
      // chunk 0: the kernel derives it from the device-side row count (same formula)
      const int64_t chunk = kway ? 0 : dev::xg_chunk(ncov, warps);
      // f64 row sums: per-chunk partial tables + a fixed-order fold, so two runs
      // give bit-identical results (atomics only past the table budget)
      bool any_f = false;
      for (int i = 0; i < P.ne; ++i) any_f = any_f || (P.e[i].rows && P.e[i].acc_f);
      const int64_t nchunks = kway ? warps : (ncov + chunk - 1) / chunk;  // k-way: the bound (zeros fold exactly)
      static const bool nodet = std::getenv("RQ_XG_NODET") != nullptr;  // A/B knob: atomic f64 flushes
      if (any_f && !nodet && nchunks * cells <= (int64_t{8} << 20)) {
        dpart = alloc_arr(ctx, RQ_F64, nchunks * cells);
        RQ_CUDA_CHECK(cudaMemsetAsync(dpart.raw_mut(), 0, static_cast<size_t>(nchunks * cells) * 8, ctx->stream));
        S.dpart = dpart.as<double>();
        S.dcells = cells;
        dchunks = nchunks;
      }
      const int64_t blocks = kway ? static_cast<int64_t>(ctx->sm_count) * bps
                                  : std::min<int64_t>(static_cast<int64_t>(ctx->sm_count) * bps,
                                                      (ncov / chunk + (B / 32)) / (B / 32) + 1);
      constexpr size_t smem = dev::xg_rows_smem<B>();
      kernel_occupancy(ctx, dev::k_xg_rows<B>, B, smem);  // shared-memory opt-in on this device
      KTimer rows_timer(ctx, "xg_rows");
      const char* nojit = std::getenv("RQ_NO_JIT");
      bool folded = false;  // the generated kernel's last CTA folded dpart
      bool jit_ran = false;
      if (!(nojit && nojit[0] == '1')) {
        dev::XgSegs SJ = S;
        // few f64 cells (Q6: one): fold inside the row kernel, no k_xg_dfold
        // launch; many cells (Q1: 48) keep the one-block-per-cell fold
        static const bool no_kfold = std::getenv("RQ_XG_NO_KFOLD") != nullptr;  // A/B knob
        unsigned fmask = 0;
        int nf = 0;
        for (int i = 0; i < P.ne; ++i)
          if (P.e[i].rows && P.e[i].acc_f) fmask |= 1u << i, ++nf;
        if (S.dpart && !no_kfold && G * nf <= 4) {
          SJ.fticket = ctx->tickets + 8;
          SJ.fchunks = dchunks;
          SJ.fmask = fmask;
        }
        jit_ran = xg_jit_launch(ctx, P, SJ, chunk, tabp, G, err, static_cast<unsigned>(blocks), avg_len);
        folded = jit_ran && SJ.fticket != nullptr;
      }
      if (!jit_ran) dev::k_xg_rows<B><<<static_cast<unsigned>(blocks), B, smem, ctx->stream>>>(P, S, chunk, tabp, G, err);
      launched(ctx);
      if (S.dpart && !folded) {
        dev::XgIsF isf{};  // by value: no host staging
        for (int i = 0; i < P.ne; ++i) isf.f[i] = P.e[i].rows && P.e[i].acc_f;
        dev::k_xg_dfold<<<static_cast<unsigned>(cells), dev::DFOLD_B, 0, ctx->stream>>>(S.dpart, dchunks, cells, P.ne, isf,
                                                                               tabp);
        launched(ctx);
      }
    }
    for (auto& pe : pi_exprs) {  // Plain+Index: outliers inside segments (located by search, not materialised)
      const DCol& c = *pe.second;
      if (c.p2.n == 0 || nseg == 0) continue;
      const dev::XgExpr& X = P.e[pe.first];
      const DCol::RankDir& pd = rank_dir(ctx, c.p2, c.total, c.dir_p2);
      const int gs = grid_cap(ctx, nseg * 32);  // a warp per segment
      DArr opart;
      double* op = X.acc_f ? f64_part(gs, opart) : nullptr;
      dev::k_xg_outliers_seg<<<gs, 256, 0, ctx->stream>>>(
          P.col[X.t[0].src], c.p2.pos(), c.v2.raw(), c.v2.dt, c.p2.n, s.pos(), e.pos(), slot.pos(), nseg, S.dims,
          pd.shift >= 0 ? pd.dir.pos() : nullptr, pd.shift, pd.nb, P.ne, pe.first, X.acc_f, tabp, op, cells);
      launched(ctx);
      if (op) {  // added after the row pass's fold wrote the base sums
        dev::XgIsF of{};
        of.f[pe.first] = 1;
        dev::k_xg_dfold<<<static_cast<unsigned>(cells), dev::DFOLD_B, 0, ctx->stream>>>(op, int64_t{gs} * 8, cells, P.ne, of,
                                                                               tabp, 1);
        launched(ctx);
      }
    }
    return 1;
  };
  if (!run_graph(ctx, preK == nullptr, middle, K, tab, cnt, kway)) return false;
  const int64_t G = K.G;
  bool int_div = false;  // only integer division can raise (align.cpp:297-299)
  for (int i = 0; i < P.ne; ++i)
    for (int t = 0; t < P.e[i].nt; ++t)
      int_div = int_div || P.e[i].t[t].sop == RQ_DIV || (t > 0 && P.e[i].op[t - 1] == RQ_DIV);
  if (int_div) {
    const int64_t* h = ctx->readback(err, 8);
    const bool div0 = (h[0] & 0xffffffff) != 0;
    if (div0) {
      RQ_CUDA_CHECK(cudaMemsetAsync(err, 0, 4, ctx->stream));
      fail("integer division by zero");
    }
  }
  // ---- outputs: present slots ascending (= ascending keys) ----
  auto stage = std::make_unique<KTimer>(ctx, "xg_out");
  static const bool no_tail = std::getenv("RQ_XG_NO_TAIL") != nullptr;  // A/B knob: the multi-launch tail
  if (!keys.empty() && keys.size() <= 8 && G <= dev::XG_TAIL_MAX && !no_tail) {
    dev::XgTailKeys KT{};
    KT.nk = static_cast<int>(keys.size());
    for (size_t c = 0; c < keys.size(); ++c) {
      DArr kout = alloc_arr(ctx, K.kdt[c], G);  // capacity: every slot present
      KT.dt[c] = K.kdt[c];
      KT.kmin[c] = K.kmin[c];
      KT.stride[c] = K.stride[c];
      KT.range[c] = K.range[c];
      KT.out[c] = kout.raw_mut();
      out.keys.push_back(kout);
    }
    dev::XgFinish F{};
    F.ne = P.ne;
    for (int i = 0; i < P.ne; ++i) {
      const int fn = fns[static_cast<size_t>(i)];
      const int32_t odt = fn == RQ_COUNT ? RQ_I64 : (fn == RQ_AVG || P.e[i].res_f) ? RQ_F64 : RQ_I64;
      DArr res = alloc_arr(ctx, odt, G);
      F.fn[i] = fn;
      F.isf[i] = P.e[i].acc_f;
      F.out[i] = res.raw_mut();
      out.vals.push_back(res);
    }
    DArr ngd = alloc_arr(ctx, RQ_I64, 1);
    dev::k_xg_tail<<<1, dev::XG_TAIL_B, 0, ctx->stream>>>(F, KT, G, reinterpret_cast<const unsigned long long*>(tab.raw()),
                                                          reinterpret_cast<const unsigned long long*>(cnt.raw()),
                                                          ngd.as<int64_t>());
    launched(ctx);
    const int64_t ng = ctx->readback(ngd.raw(), 8)[0];
    out.n_groups = ng;
    for (auto& a : out.keys) {
      a.n = ng;
      if (ng == 0) a.buf.reset();
    }
    for (auto& a : out.vals) {
      a.n = ng;
      if (ng == 0) a.buf.reset();
    }
    return true;
  }
  DArr present;
  if (keys.empty()) {
    present.n = 1;  // one group (slot 0): finish reads no slot list
  } else {
    DArr flags = alloc_arr(ctx, RQ_I8, G);
    dev::k_gk_flags<<<grid_cap(ctx, G), 256, 0, ctx->stream>>>(reinterpret_cast<const unsigned long long*>(cnt.raw()),
                                                                G, flags.as<uint8_t>());
    launched(ctx);
    flagged_indices(ctx, flags, G, present);
  }
  const int64_t ng = present.n;
  out.n_groups = ng;
  for (size_t c = 0; c < keys.size(); ++c) {
    DArr kout = alloc_arr(ctx, K.kdt[c], ng);
    if (ng) {
      dev::k_gk_keys<<<grid_cap(ctx, ng), 256, 0, ctx->stream>>>(present.pos(), ng, K.kmin[c], K.stride[c],
                                                                 K.range[c], K.kdt[c], kout.raw_mut());
      launched(ctx);
    }
    out.keys.push_back(kout);
  }
  dev::XgFinish F{};  // every expression's output in one launch
  F.ne = P.ne;
  for (int i = 0; i < P.ne; ++i) {
    const int fn = fns[static_cast<size_t>(i)];
    const int32_t odt = fn == RQ_COUNT ? RQ_I64 : (fn == RQ_AVG || P.e[i].res_f) ? RQ_F64 : RQ_I64;
    DArr res = alloc_arr(ctx, odt, ng);
    F.fn[i] = fn;
    F.isf[i] = P.e[i].acc_f;
    F.out[i] = res.raw_mut();
    out.vals.push_back(res);
  }
  if (ng) {
    dev::k_xg_finish_all<<<grid_cap(ctx, ng), 256, 0, ctx->stream>>>(
        F, keys.empty() ? nullptr : present.pos(), ng, reinterpret_cast<const unsigned long long*>(tab.raw()),
        reinterpret_cast<const unsigned long long*>(cnt.raw()));
    launched(ctx);
  }
  return true;
}

// The runner's chain (runner.cpp:243-336) on the operator API: Filter every
// operand column, evaluate the expressions with arith / arith_scalar, then
// group_aggregate(normalize) — or aggregate_all per expression with no keys.
GroupAggOut xg_chain(const CtxPtr& ctx, const DMask* mask, const std::vector<const DCol*>& keys,
                     const std::vector<XExpr>& exprs, const std::vector<int>& fns) {
  std::vector<std::pair<const DCol*, DCol>> filtered;
  size_t nref = keys.size();
  for (auto& x : exprs) nref += x.terms.size();
  filtered.reserve(nref);  // references into it stay valid
  auto F = [&](const DCol* c) -> const DCol& {
    if (!mask) return *c;
    for (auto& f : filtered)
      if (f.first == c) return f.second;
    filtered.push_back({c, filter(ctx, *c, *mask)});
    return filtered.back().second;
  };
  std::vector<DCol> keep;  // stable storage for expression results
  keep.reserve(exprs.size() + 1);
  std::vector<const DCol*> kf;
  for (auto* k : keys) kf.push_back(&F(k));
  std::vector<const DCol*> data;
  for (size_t i = 0; i < exprs.size(); ++i) {
    const XExpr& x = exprs[i];
    if (x.terms.empty()) {  // COUNT(*): any column with the query's coverage
      require(!kf.empty() || !exprs.empty(), "count: no column");
      const DCol* any = !kf.empty() ? kf[0] : nullptr;
      for (size_t j = 0; !any && j < exprs.size(); ++j)
        if (!exprs[j].terms.empty()) any = &F(exprs[j].terms[0].col);
      require(any != nullptr, "count(*) needs a key or an operand column");
      data.push_back(any);
      continue;
    }
    auto term = [&](const XTerm& t) -> DCol {
      const DCol& c = F(t.col);
      return t.sop >= 0 ? arith_scalar(ctx, c, t.k, t.sop, t.rev) : c;
    };
    DCol v = term(x.terms[0]);
    for (size_t t = 1; t < x.terms.size(); ++t) v = arith(ctx, v, term(x.terms[t]), x.ops[t - 1]);
    keep.push_back(v);
    data.push_back(&keep.back());
  }
  if (!keys.empty()) return group_aggregate(ctx, kf, data, fns, true);
  GroupAggOut out;
  out.n_groups = 1;
  for (size_t i = 0; i < data.size(); ++i) {
    AggOut a = aggregate_column(ctx, normalize_basic(ctx, *data[i]), fns[i]);
    DArr r = a.dtype == RQ_F64 ? upload_arr(ctx, RQ_F64, &a.f, 1) : upload_arr(ctx, RQ_I64, &a.i, 1);
    out.vals.push_back(r);
  }
  return out;
}

}  // namespace

bool col_full_coverage(const CtxPtr& ctx, const DCol& c) {
  switch (c.enc) {
    case RQ_ENC_PLAIN:
    case RQ_ENC_PLAIN_INDEX: return true;
    case RQ_ENC_RLE: return col_gapless(ctx, c);
    case RQ_ENC_INDEX: return c.p.n == c.total;
    default: return false;
  }
}

GroupAggOut group_aggregate_exprs(const CtxPtr& ctx, const DMask* mask, const std::vector<const DCol*>& keys,
                                  const std::vector<XExpr>& exprs, const std::vector<int>& fns, bool* fused,
                                  const std::vector<XPred>* preds, bool fused_only) {
  require(exprs.size() == fns.size(), "group_aggregate_exprs: one function per expression");
  for (auto& x : exprs) {
    require(x.terms.size() <= 3 && x.ops.size() + 1 == std::max<size_t>(1, x.terms.size()),
            "group_aggregate_exprs: expressions are left-deep chains of at most 3 terms");
    for (auto& t : x.terms) require(t.col != nullptr, "group_aggregate_exprs: null operand");
  }
  GroupAggOut out;
  const bool has_preds = preds && !preds->empty();
  // Without keys the runner aggregates each expression over its own coverage
  // (aggregate_all per column, runner.cpp:325-333); the fused pass shares one
  // segment table across expressions, which is the same thing only when the
  // operands' coverages cannot differ.
  bool fusable = true;
  if (keys.empty() && exprs.size() > 1)
    for (auto& x : exprs)
      for (auto& t : x.terms) fusable = fusable && col_full_coverage(ctx, *t.col);
  bool ok = fusable && xg_fused(ctx, mask, keys, exprs, fns, out, nullptr, has_preds ? preds : nullptr);
  // the CUDA-graph key names this call's user handles: the passes below run on
  // per-call arrays (a built mask) and must never replay a graph
  ctx->graph_key.clear();
  if (ok) {
    if (fused) *fused = true;
    return out;
  }
  // the WHERE list as the runner builds it: compare_scalar per conjunct
  // (IN = OR of equalities), and_mask across conjuncts and with `mask`
  std::unique_ptr<DMask> built;
  if (has_preds) {
    for (const XPred& q : *preds) {
      DMask m;
      if (q.in.empty()) {
        m = compare_scalar(ctx, *q.col, q.k, q.op, false);
      } else {
        m = compare_scalar(ctx, *q.col, q.in[0], RQ_EQ, false);
        for (size_t j = 1; j < q.in.size(); ++j) m = mask_or(ctx, m, compare_scalar(ctx, *q.col, q.in[j], RQ_EQ, false));
      }
      built.reset(new DMask(built ? mask_and(ctx, *built, m) : m));
    }
    if (mask) built.reset(new DMask(mask_and(ctx, *built, *mask)));
    ok = fusable && xg_fused(ctx, built.get(), keys, exprs, fns, out);
    if (ok) {
      if (fused) *fused = true;
      return out;
    }
  }
  if (fused) *fused = false;
  // probe-only callers (the plan executor) run their own generic path next:
  // do not run the chain here too
  if (fused_only) return GroupAggOut{};
  return xg_chain(ctx, built ? built.get() : mask, keys, exprs, fns);
}

}  // namespace rqb
