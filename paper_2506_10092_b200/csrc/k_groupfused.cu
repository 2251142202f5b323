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
#include <cmath>
#include <limits>

#include "merge_walk.cuh"
#include "rq_internal.hpp"

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
};

constexpr int kSmemSlots = 4096;

template <int KIND>
__device__ __forceinline__ unsigned long long* g_table_begin(unsigned long long* smem, const GTable& t) {
  if (t.G > kSmemSlots) return t.g;
  for (int64_t s = threadIdx.x; s < t.G; s += blockDim.x) smem[s] = g_identity<KIND>();
  __syncthreads();
  return smem;
}

template <int KIND>
__device__ __forceinline__ void g_table_end(unsigned long long* smem, const GTable& t) {
  if (t.G > kSmemSlots) return;
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

struct PlainSrc {  // bit-width-reduced plain column (decode inline)
  const void* v;
  int dt, logical, has_center, flt;
  int64_t center;
};

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
  tl.walk(sk, [&](int64_t i, int64_t j, bool takeA, int64_t key) {
    if (i >= m.na || j >= m.nb) return;
    // key run i starts after key run i-1's end; data run j starts at ds[j]
    const int64_t ks = ldg64(kst, i);
    const int64_t lo = max(ks, ldg64(ds, j));
    const int64_t len = key - lo + 1;
    if (len <= 0) return;
    const int64_t slot = ld_i64(kv, kdt, i) - t.kmin;
    if (slot != cur) {
      if (cur >= 0) g_atomic<KIND>(tab, cur, acc);
      acc = g_zero<KIND>();
      cur = slot;
      if (KIND == G_SQ) mu = mean[slot];
    }
    g_fold<KIND>(acc, ld_as<T>(dv, ddt, j), len, mu);
  });
  if (cur >= 0) g_atomic<KIND>(tab, cur, acc);
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
        if (lane == 0 && slot >= 0) g_atomic<KIND>(tab, slot, r);
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
    if (lane == 0 && slot >= 0) g_atomic<KIND>(tab, slot, r);
  }
  g_table_end<KIND>(smem, t);
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
  constexpr int B = 256, IT = 8, TILE = B * IT;
  const int64_t na = K.e.n, nb = de.n;
  if (na == 0 || nb == 0) return;
  const int64_t ntiles = (na + nb + TILE - 1) / TILE;
  DArr part = alloc_arr(ctx, RQ_I64, ntiles + 1);
  dev::k_merge_partition<<<static_cast<unsigned>(((ntiles + 1) * 32 + 255) / 256), 256, 0, ctx->stream>>>(
      K.e.pos(), na, de.pos(), nb, TILE, ntiles + 1, part.as<int64_t>());
  launched(ctx);
  dev::MergeArgs m{K.e.pos(), na, de.pos(), nb, part.as<int64_t>()};
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
  if (POINTS) {
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
  fold_column<KIND>(ctx, K, d, t, mean);
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
  auto mm = minmax(ctx, vals[0]);
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
    auto mm = minmax(ctx, vals[c]);
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
  KTimer timer(ctx, "group_fused");
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
  select_points(ctx, flags, iota(ctx, K.G), present, nullptr);
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

}  // namespace rqb
