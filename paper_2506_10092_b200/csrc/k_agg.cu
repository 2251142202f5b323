// k_agg.cu — run-length-weighted aggregation (K2/K5 reductions).
//
// agg::aggregate_array (groupby.cpp:67-135) multiplies each slot's value by
// its weight (run length for run shapes, 1 otherwise) and scatter-reduces.
// Here the weight is computed inline from (s, e) and the product is folded
// into per-thread accumulators; each CTA writes one partial record and a
// single-CTA pass combines the partials in a fixed order (deterministic f64).
// The fused RLE×RLE kernel (K2) runs the merge-path walk of range_intersect
// and folds (va op vb)·len per fragment without materialising fragments —
// the whole compute::arith → agg::aggregate_all chain (align.cpp:495-508,
// groupby.cpp:164-172) in one pass over the compressed bytes.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <type_traits>

#include "merge_walk.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

struct AggPart {
  unsigned long long isum;  // Σ int64(v)·w, wrapping
  double fsum;              // Σ f64(v)·f64(w)  (pass 2: Σ (v-mean)²·w)
  long long cnt;            // Σ w
  long long imin, imax;
  double fmin, fmax;
  double pad;
};

struct Acc {
  uint64_t isum = 0;
  double fsum = 0.0;
  int64_t cnt = 0;
  int64_t imin = INT64_MAX, imax = INT64_MIN;
  double fmin = INFINITY, fmax = -INFINITY;

  template <class T>
  __device__ __forceinline__ void add(T x, int64_t w, bool pass2, double mean) {
    if (pass2) {
      const double d = static_cast<double>(x) - mean;
      fsum += d * d * static_cast<double>(w);
      return;
    }
    isum += static_cast<uint64_t>(static_cast<int64_t>(x)) * static_cast<uint64_t>(w);
    fsum += static_cast<double>(x) * static_cast<double>(w);
    cnt += w;
    const int64_t xi = static_cast<int64_t>(x);
    imin = xi < imin ? xi : imin;
    imax = xi > imax ? xi : imax;
    const double xf = static_cast<double>(x);
    fmin = xf < fmin ? xf : fmin;
    fmax = xf > fmax ? xf : fmax;
  }
};

template <>
__device__ __forceinline__ void Acc::add<double>(double x, int64_t w, bool pass2, double mean) {
  if (pass2) {
    const double d = x - mean;
    fsum += d * d * static_cast<double>(w);
    return;
  }
  fsum += x * static_cast<double>(w);
  cnt += w;
  fmin = x < fmin ? x : fmin;
  fmax = x > fmax ? x : fmax;
}

template <int BLOCK>
__device__ __forceinline__ void block_store_acc(Acc a, AggPart* out) {
  __shared__ uint64_t ru[BLOCK / 32 + 1];
  __shared__ double rf[BLOCK / 32 + 1];
  __shared__ int64_t ri[BLOCK / 32 + 1];
  constexpr int NW = BLOCK / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t isum = block_sum<BLOCK>(a.isum, ru);
  const double fsum = block_sum<BLOCK>(a.fsum, rf);
  const uint64_t cnt = block_sum<BLOCK>(static_cast<uint64_t>(a.cnt), ru);
  // min / max via warp reductions
  int64_t imin = warp_min(a.imin), imax = warp_max(a.imax);
  double fmin = warp_min(a.fmin), fmax = warp_max(a.fmax);
  __shared__ int64_t smin[NW], smax[NW];
  __shared__ double sfmin[NW], sfmax[NW];
  if (lane == 0) {
    smin[wid] = imin;
    smax[wid] = imax;
    sfmin[wid] = fmin;
    sfmax[wid] = fmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NW; ++w) {
      imin = smin[w] < imin ? smin[w] : imin;
      imax = smax[w] > imax ? smax[w] : imax;
      fmin = sfmin[w] < fmin ? sfmin[w] : fmin;
      fmax = sfmax[w] > fmax ? sfmax[w] : fmax;
    }
    AggPart p;
    p.isum = isum;
    p.fsum = fsum;
    p.cnt = static_cast<long long>(cnt);
    p.imin = imin;
    p.imax = imax;
    p.fmin = fmin;
    p.fmax = fmax;
    p.pad = 0;
    *out = p;
  }
  (void)ri;
}

// Generic slot reduction. Weighted by run length when s != nullptr, unit
// weight otherwise. Optional inline decode (bit-width-reduced plain storage:
// wrap to logical width, add centre) — K9 fused into the reduction.
struct SlotSpec {
  const void* v;
  int dt;
  const int64_t* s;
  const int64_t* e;
  int64_t n;
  int decode;  // 1: integer decode with logical/centre
  int logical;
  int has_center;
  int64_t center;
};

template <class T, int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_reduce_slots(SlotSpec sp, int pass2, double mean, AggPart* __restrict__ parts) {
  Acc acc;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < sp.n;
       i += static_cast<int64_t>(gridDim.x) * BLOCK) {
    T x;
    if (sp.decode) {
      int64_t r = wrap_to(sp.logical, ld_i64(sp.v, sp.dt, i));
      if (sp.has_center)
        r = wrap_to(sp.logical, static_cast<int64_t>(static_cast<uint64_t>(r) + static_cast<uint64_t>(sp.center)));
      x = static_cast<T>(r);
    } else {
      x = ld_as<T>(sp.v, sp.dt, i);
    }
    const int64_t w = sp.s ? ldg64(sp.e, i) - ldg64(sp.s, i) + 1 : 1;
    acc.add<T>(x, w, pass2 != 0, mean);
  }
  block_store_acc<BLOCK>(acc, parts + blockIdx.x);
}

// Combines `n` partials in a fixed order into parts_out[0].
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_combine(const AggPart* __restrict__ parts, int64_t n,
                                                   AggPart* __restrict__ out) {
  Acc acc;
  for (int64_t i = threadIdx.x; i < n; i += BLOCK) {
    const AggPart p = parts[i];
    acc.isum += p.isum;
    acc.fsum += p.fsum;
    acc.cnt += p.cnt;
    acc.imin = p.imin < acc.imin ? p.imin : acc.imin;
    acc.imax = p.imax > acc.imax ? p.imax : acc.imax;
    acc.fmin = p.fmin < acc.fmin ? p.fmin : acc.fmin;
    acc.fmax = p.fmax > acc.fmax ? p.fmax : acc.fmax;
  }
  block_store_acc<BLOCK>(acc, out);
}

// K2: fused RLE×RLE intersection + (va op vb)·len reduction.
template <int BLOCK, int ITEMS, bool GAPLESS, class T>
__global__ void __launch_bounds__(BLOCK)
    k_pair_reduce(MergeArgs m, const int64_t* __restrict__ s1, const int64_t* __restrict__ s2,
                  const void* __restrict__ v1, int dt1, const void* __restrict__ v2, int dt2, int op,
                  int pass2, double mean, AggPart* __restrict__ parts, int* __restrict__ err) {
  using Tile = MergeTile<BLOCK, ITEMS>;
  __shared__ int64_t sk[Tile::TILE];
  Tile t;
  t.load(m, blockIdx.x, sk);
  Acc acc;
  int lerr = 0;
  int64_t prev = GAPLESS ? t.prev_key(sk, m) : 0;
  t.walk(sk, [&](int64_t i, int64_t j, bool takeA, int64_t key) {
    // the walk reports (A index, B index); one of them is the consumed key
    const int64_t ia = i, jb = j;
    const bool valid = takeA ? (jb < m.nb) : (ia < m.na);
    int64_t len;
    if (GAPLESS) {
      len = key - prev;
      prev = key;
    } else {
      const int64_t lo = valid ? max(ldg64(s1, ia), ldg64(s2, jb)) : key + 1;
      len = key - lo + 1;
    }
    if (valid && len > 0) {
      const T a = ld_as<T>(v1, dt1, ia);
      const T b = ld_as<T>(v2, dt2, jb);
      acc.add<T>(arith_t<T>(a, b, op, &lerr), len, pass2 != 0, mean);
    }
  });
  if (lerr) atomicExch(err, 1);
  __syncthreads();
  block_store_acc<BLOCK>(acc, parts + blockIdx.x);
}

// K2 fast path for two GAPLESS run lists (every merged end closes one
// fragment of length key − previous key): keys and values of the tile's two
// segments are staged in shared memory (values converted to T once, plus the
// run just past each segment, which can be the other list's cursor); each
// step reloads only the consumed side. KIND: 0 = Σ r·len as int64 (SUM int),
// 1 = Σ r·len as f64 + Σ len (SUM float / AVG), 2 = Σ len (COUNT).
template <int BLOCK, int ITEMS, class T, int OP, int KIND>
__global__ void __launch_bounds__(BLOCK)
    k_pair_reduce_gapless(MergeArgs m, const void* __restrict__ v1, int dt1, const void* __restrict__ v2,
                          int dt2, AggPart* __restrict__ parts, int* __restrict__ err) {
  constexpr int TILE = BLOCK * ITEMS;
  __shared__ int64_t sk[TILE];
  __shared__ T sv[TILE + 2];
  const int tile = blockIdx.x;
  const int64_t d0 = static_cast<int64_t>(tile) * TILE;
  const int64_t d1 = min(d0 + TILE, m.na + m.nb);
  const int64_t i0 = m.part[tile], i1 = m.part[tile + 1];
  const int64_t j0 = d0 - i0, j1 = d1 - i1;
  const int a = static_cast<int>(i1 - i0), b = static_cast<int>(j1 - j0);
  // keys: A ends [0, a), B ends [a, a + b); values: A [0, a], B [a + 1, a + b + 1]
  // (all loads of a thread issued before the stores; typed fast path when
  // both value arrays already hold T)
  {
    const int64_t* pa = m.A + i0;
    const int64_t* pb = m.B + j0 - a;
    constexpr int DT = sizeof(T) == 8 && T(0.5) != T(0) ? RQ_F64 : RQ_I64;
    const bool typed = dt1 == DT && dt2 == DT;
    const T* tv1 = static_cast<const T*>(v1) + i0;
    const T* tv2 = static_cast<const T*>(v2) + j0 - (a + 1);
    int64_t tk[ITEMS];
    T tvv[ITEMS + 1];
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int k = u * BLOCK + threadIdx.x;
      tk[u] = k < a + b ? __ldg(reinterpret_cast<const long long*>(k < a ? pa : pb) + k) : 0;
    }
    // valid value slots: A k in [0, a_lim], B k in [a + 1, b_lim] (tile-uniform)
    const int a_lim = static_cast<int>(min(static_cast<int64_t>(a), m.na - 1 - i0));
    const int b_lim = static_cast<int>(min(static_cast<int64_t>(a + b + 1), a + m.nb - j0));
    if (typed) {
#pragma unroll
      for (int u = 0; u <= ITEMS; ++u) {
        const int k = u * BLOCK + threadIdx.x;
        const bool in_a = k <= a;
        const bool ok = in_a ? k <= a_lim : k <= b_lim;
        tvv[u] = ok ? (in_a ? tv1 : tv2)[k] : T(0);
      }
    } else {
#pragma unroll
      for (int u = 0; u <= ITEMS; ++u) {
        const int k = u * BLOCK + threadIdx.x;
        const bool in_a = k <= a;
        const bool ok = in_a ? k <= a_lim : k <= b_lim;
        tvv[u] = !ok ? T(0) : in_a ? ld_as<T>(v1, dt1, i0 + k) : ld_as<T>(v2, dt2, j0 + (k - a - 1));
      }
    }
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int k = u * BLOCK + threadIdx.x;
      if (k < a + b) sk[k] = tk[u];
    }
#pragma unroll
    for (int u = 0; u <= ITEMS; ++u) {
      const int k = u * BLOCK + threadIdx.x;
      if (k < a + b + 2) sv[k] = tvv[u];
    }
  }
  __syncthreads();
  int diag = threadIdx.x * ITEMS;
  if (diag > a + b) diag = a + b;
  int x = smem_merge_path(sk, a, b, diag);
  int y = diag - x;
  // previous merged key (-1 before the first run of the column)
  int64_t prev;
  {
    int64_t pa = -1, pb = -1;
    if (x > 0) pa = sk[x - 1];
    else if (i0 > 0) pa = ldg64(m.A, i0 - 1);
    if (y > 0) pb = sk[a + y - 1];
    else if (j0 > 0) pb = ldg64(m.B, j0 - 1);
    prev = pa > pb ? pa : pb;
  }
  int64_t ka = x < a ? sk[x] : KEY_MAX;
  int64_t kb = y < b ? sk[a + y] : KEY_MAX;
  T va = sv[x], vb = sv[a + 1 + y];
  uint64_t isum = 0;
  double fsum = 0.0;
  int64_t cnt = 0;
  int lerr = 0;
  const int steps = min(ITEMS, a + b - diag);
  for (int it = 0; it < steps; ++it) {
    const bool takeA = ka <= kb;
    const int64_t key = takeA ? ka : kb;
    const int64_t len = key - prev;  // 0 on a shared end (tie)
    prev = key;
    if (KIND == 0) {
      if (len > 0) {  // a tie closes no fragment (and must not divide)
        const T r = arith_t<T>(va, vb, OP, &lerr);
        isum += static_cast<uint64_t>(static_cast<int64_t>(r)) * static_cast<uint64_t>(len);
      }
    } else if (KIND == 1) {
      if (len > 0) {
        const T r = arith_t<T>(va, vb, OP, &lerr);
        fsum += static_cast<double>(r) * static_cast<double>(len);
      }
      cnt += len;
    } else {
      cnt += len;
    }
    if (takeA) {
      ++x;
      ka = x < a ? sk[x] : KEY_MAX;
      va = sv[x];
    } else {
      ++y;
      kb = y < b ? sk[a + y] : KEY_MAX;
      vb = sv[a + 1 + y];
    }
  }
  if (lerr) atomicExch(err, 1);
  __shared__ uint64_t ru[BLOCK / 32 + 1];
  __shared__ double rf[BLOCK / 32 + 1];
  isum = block_sum<BLOCK>(isum, ru);
  fsum = block_sum<BLOCK>(fsum, rf);
  const uint64_t c = block_sum<BLOCK>(static_cast<uint64_t>(cnt), ru);
  if (threadIdx.x == 0) {
    AggPart p{};
    p.isum = isum;
    p.fsum = fsum;
    p.cnt = static_cast<long long>(c);
    p.imin = INT64_MAX;
    p.imax = INT64_MIN;
    p.fmin = INFINITY;
    p.fmax = -INFINITY;
    parts[tile] = p;
  }
}

// ---------------------------------------------------------------------------
// K2 persistent TMA form (gapless RLE × gapless RLE, 8-byte values).
// The list with more runs drives: tile t = its runs [t·TA, (t+1)·TA) (the
// row range (r_lo, r_hi]); the other list's window = its runs whose ends
// fall after r_lo, chained from tile to tile by the producer warp (rank of
// r_hi + 1 in the landed window, a warp search only past it) and staged with
// 1-D bulk copies into two mbarrier stages, as in the C2 kernel. Every
// fragment of the union of boundaries ends at a driver end or at an other-
// list end; consumers take the driver ends (ITEMS per lane: one shared-
// memory lower_bound, forward steps) and then the other list's ends inside
// the tile (ties belong to the driver), each closing
//   (va op vb) · (end − max(prev driver end, prev other end)).
// Per-CTA partials are folded by the last CTA (ticket counter).
// ---------------------------------------------------------------------------

template <int TA, int BW>
struct PairStage {
  static constexpr int AE = TA + 2 + 16;  // ends: 2 previous + tile (+ rounding)
  static constexpr int AV = TA + 16;
  static constexpr int BE = BW + 16;      // window padded to BW (+8 for the forward steps)
  static constexpr size_t AE_OFF = 0;
  static constexpr size_t AV_OFF = AE_OFF + AE * 8;
  static constexpr size_t BE_OFF = AV_OFF + AV * 8;
  static constexpr size_t BV_OFF = BE_OFF + BE * 8;
  static constexpr size_t BYTES = BV_OFF + BE * 8;
};

template <int BLOCK, int IA, int BW, class T, int OP, int KIND>
__global__ void __launch_bounds__(BLOCK, 1024 / BLOCK)
    k_pair_reduce_tma(const int64_t* __restrict__ Ae, const T* __restrict__ Av, int64_t na,
                      const int64_t* __restrict__ Be, const T* __restrict__ Bv, int64_t nb, int swap,
                      int ta, int64_t ntiles, AggPart* __restrict__ parts, unsigned* __restrict__ ticket,
                      AggPart* __restrict__ out, int* __restrict__ err) {
  constexpr int NCW = BLOCK / 32 - 1;
  constexpr int NL = NCW * 32;  // consumer lanes
  constexpr int TA = NL * IA;
  using S = PairStage<TA, BW>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[2], empty[2];
  __shared__ int64_t s_lo[2];
  __shared__ int s_nb[2], s_jf[2];

  const int64_t t_begin = static_cast<int64_t>(blockIdx.x) * ntiles / gridDim.x;
  const int64_t t_end = static_cast<int64_t>(blockIdx.x + 1) * ntiles / gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto sAe = [&](int st) { return reinterpret_cast<int64_t*>(smem + st * S::BYTES + S::AE_OFF); };
  auto sAv = [&](int st) { return reinterpret_cast<T*>(smem + st * S::BYTES + S::AV_OFF); };
  auto sBe = [&](int st) { return reinterpret_cast<int64_t*>(smem + st * S::BYTES + S::BE_OFF); };
  auto sBv = [&](int st) { return reinterpret_cast<T*>(smem + st * S::BYTES + S::BV_OFF); };

  if (threadIdx.x == 0) {
    mbar_init(&full[0], 32);
    mbar_init(&full[1], 32);
    mbar_init(&empty[0], NCW);
    mbar_init(&empty[1], NCW);
  }
  __syncthreads();

  uint64_t isum = 0;
  double fsum = 0.0;
  int64_t cnt = 0;
  int lerr = 0;
  if (wid == 0) {
    // ---- producer ----
    int64_t jb = 0, b_lo = 0;
    int b_est = BW, b_n = 0;
    int hw0 = BW + 8, hw1 = BW + 8;  // per stage: entries [hw, BW + 8) still hold the pad
    // start-up search inputs loaded together: the end before the CTA's first
    // A run and B's last end (interpolation round of warp_lower_bound_pair)
    const int64_t a_first = t_begin * static_cast<int64_t>(ta);
    const int64_t r_lo0 = t_begin < t_end && a_first > 0 ? ldg64(Ae, a_first - 1) : -1;
    const int64_t b_last = nb > 0 ? ldg64(Be, nb - 1) : -1;
    for (int64_t t = t_begin; t < t_end; ++t) {
      const int st = static_cast<int>((t - t_begin) & 1);
      const uint32_t use = static_cast<uint32_t>((t - t_begin) >> 1);
      const int64_t a0 = t * ta;
      const int na_t = static_cast<int>(min(static_cast<int64_t>(ta), na - a0));
      if (t - t_begin >= 2) mbar_wait(&empty[st], (use - 1) & 1);
      int64_t* wAe = sAe(st);
      T* wAv = sAv(st);
      int64_t* wBe = sBe(st);
      T* wBv = sBv(st);
      // (1) the driver part does not depend on the window chain: issue it
      // first, as soon as the stage is free (ends from a0 - 2: two previous
      // ends, -1 before the column; values from a0). Its bytes are expected
      // on the stage barrier without arriving; the lanes arrive in (2).
      const bool first = a0 == 0;
      const int ae_n = na_t + (first ? 0 : 2);
      const int ae_bulk = ae_n & ~1, av_bulk = na_t & ~1;
      int64_t* ae_dst = first ? wAe + 2 : wAe;
      const int64_t* ae_src = first ? Ae : Ae + (a0 - 2);
      if (first && lane < 2) wAe[lane] = -1;
      if (lane == 0 && ae_bulk < ae_n) ae_dst[ae_bulk] = ldg64(ae_src, ae_bulk);
      if (lane == 1 && av_bulk < na_t) wAv[av_bulk] = Av[a0 + av_bulk];
      if (lane == 0) {
        fence_proxy_async_smem();
        mbar_expect_tx(&full[st], static_cast<uint32_t>(ae_bulk + av_bulk) * 8u);
        if (ae_bulk) bulk_g2s(ae_dst, ae_src, ae_bulk * 8u, &full[st]);
        if (av_bulk) bulk_g2s(wAv, Av + a0, av_bulk * 8u, &full[st]);
      }
      // (2) the other list's window: chained from tile t-1's landed window
      if (t == t_begin) {
        int64_t unused;
        warp_lower_bound_pair(Be, nb, b_last, r_lo0 + 1, nullptr, 0, -1, 0, jb, unused);
      } else {
        mbar_wait(&full[st ^ 1], ((t - 1 - t_begin) >> 1) & 1);  // tile t-1 landed
        const int pst = st ^ 1;
        const int pna = static_cast<int>(min(static_cast<int64_t>(ta), na - (a0 - ta)));
        const int64_t r_prev_hi = sAe(pst)[2 + pna - 1];
        const int rb = warp_smem_lower_bound(sBe(pst), BW, r_prev_hi + 1);
        int64_t jn = b_lo + rb;
        if (rb >= b_n && jn < nb) jn += warp_lower_bound(Be + jn, nb - jn, r_prev_hi + 1);
        const int64_t used = jn - jb;
        b_est = static_cast<int>(min(static_cast<int64_t>(BW), used + (used >> 2) + 32));
        jb = jn;
      }
      // window [b_lo, b_lo + b_n): even start, < BW - 8 entries, clipped at nb
      b_lo = jb & ~int64_t(1);
      int64_t n = static_cast<int64_t>(b_est) + (jb - b_lo);
      if (n > BW - 16) n = BW - 16;
      n = (n + 1) & ~int64_t(1);  // whole 16-byte chunks: the tail path runs only at the column end
      if (n > nb - b_lo) n = nb - b_lo;
      b_n = n > 0 ? static_cast<int>(n) : 0;
      const int b_bulk = b_n & ~1;
      if (lane == 2 && b_bulk < b_n) {
        wBe[b_bulk] = ldg64(Be, b_lo + b_bulk);
        wBv[b_bulk] = Bv[b_lo + b_bulk];
      }
      {  // re-pad only what earlier copies into this stage overwrote
        int& hw = st == 0 ? hw0 : hw1;
        for (int i = b_n + lane; i < hw; i += 32) wBe[i] = INT64_MAX;
        hw = b_n;
      }
      if (lane != 0) mbar_arrive(&full[st]);
      if (lane == 0) {
        s_lo[st] = b_lo;
        s_nb[st] = b_n;
        s_jf[st] = static_cast<int>(jb - b_lo);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(2 * b_bulk) * 8u);
        if (b_bulk) {
          bulk_g2s(wBe, Be + b_lo, b_bulk * 8u, &full[st]);
          bulk_g2s(wBv, Bv + b_lo, b_bulk * 8u, &full[st]);
        }
      }
      __syncwarp();
    }
  } else {
    // ---- consumers ----
    const int cl = (wid - 1) * 32 + lane;  // consumer lane
    auto fold = [&](T va, T vb, int64_t len) {
      if (len <= 0) return;
      if (KIND == 2) {
        cnt += len;
        return;
      }
      const T r = swap ? arith_t<T>(vb, va, OP, &lerr) : arith_t<T>(va, vb, OP, &lerr);
      if (KIND == 0) {
        isum += static_cast<uint64_t>(static_cast<int64_t>(r)) * static_cast<uint64_t>(len);
      } else {
        fsum += static_cast<double>(r) * static_cast<double>(len);
        cnt += len;
      }
    };
    for (int64_t t = t_begin; t < t_end; ++t) {
      const int st = static_cast<int>((t - t_begin) & 1);
      const uint32_t use = static_cast<uint32_t>((t - t_begin) >> 1);
      const int64_t a0 = t * ta;
      const int na_t = static_cast<int>(min(static_cast<int64_t>(ta), na - a0));
      mbar_wait(&full[st], use & 1u);
      const int64_t b_lo = s_lo[st];
      const int b_n = s_nb[st];
      const int64_t* wAe = sAe(st) + 2;  // wAe[-1] = previous driver end
      const T* wAv = sAv(st);
      const int64_t* wBe = sBe(st);
      const T* wBv = sBv(st);
      const int64_t r_lo = wAe[-1], r_hi = wAe[na_t - 1];
      // other-list window entries: [jf, jl) end inside (r_lo, r_hi); entry jl
      // is the run covering r_hi (uniform searches)
      const int jf = s_jf[st];  // = jb - window start (the producer's search)
      const int jl = warp_smem_lower_bound(wBe, BW, r_hi);
      if (jl < b_n) {
        // fast path: merge path over the tile's driver ends and the window's
        // ends, ITEMS-free even split of the merged sequence over the lanes;
        // ties take the driver end first (the other end then closes 0 rows)
        const int nbi = jl - jf;
        const int tot = na_t + nbi;
        const int per = (tot + NL - 1) / NL;
        const int d = min(cl * per, tot), dend = min(d + per, tot);
        if (d < dend) {
          const int64_t* wB = wBe + jf;
          const T* vB = wBv + jf;
          int lo = d > nbi ? d - nbi : 0, hi = d < na_t ? d : na_t;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (wAe[mid] <= wB[d - mid - 1]) lo = mid + 1;
            else hi = mid;
          }
          int x = lo, y = d - lo;
          const int64_t pa0 = wAe[x - 1];
          const int64_t pb0 = jf + y > 0 ? wB[y - 1] : INT64_MIN;
          int64_t prev = pa0 > pb0 ? pa0 : pb0;
          // branch-free steps (no divergence between lanes taking A or B):
          // both cursors' keys and values are reloaded every step; reads at
          // x = na_t / y = nbi stay inside the stage (slack entries / run jl)
          int64_t ka = x < na_t ? wAe[x] : INT64_MAX;
          int64_t kb = y < nbi ? wB[y] : INT64_MAX;
          T va = wAv[x], vb = vB[y];
          // a tile spanning < 2^32 rows has fragment lengths that fit 32 bits:
          // the integer sum then multiplies 64 x 32 bits (one IMAD fewer per
          // fragment) and takes the length from the keys' low words
          auto walk = [&](auto narrow) {
            constexpr bool N32 = decltype(narrow)::value;
            for (int it = d; it < dend; ++it) {
              const bool takeA = ka <= kb;
              const int64_t key = takeA ? ka : kb;
              if (KIND == 0 && OP != RQ_DIV && N32) {
                const uint32_t len32 = static_cast<uint32_t>(key) - static_cast<uint32_t>(prev);
                const T r = swap ? arith_t<T>(vb, va, OP, &lerr) : arith_t<T>(va, vb, OP, &lerr);
                isum += static_cast<uint64_t>(static_cast<int64_t>(r)) * len32;
              } else {
                const int64_t len = key - prev;  // 0 on a tie: no fragment
                if (KIND == 2) {
                  cnt += len;
                } else if (KIND == 0 && OP != RQ_DIV) {
                  const T r = swap ? arith_t<T>(vb, va, OP, &lerr) : arith_t<T>(va, vb, OP, &lerr);
                  isum += static_cast<uint64_t>(static_cast<int64_t>(r)) * static_cast<uint64_t>(len);
                } else {
                  fold(va, vb, len);
                }
              }
              prev = key;
              x += takeA ? 1 : 0;
              y += takeA ? 0 : 1;
              ka = x < na_t ? wAe[x] : INT64_MAX;
              kb = y < nbi ? wB[y] : INT64_MAX;
              va = wAv[x];
              vb = vB[y];
            }
          };
          if (r_hi - r_lo < (int64_t{1} << 32)) walk(std::true_type{});
          else walk(std::false_type{});
        }
      } else {
        // slow path (the covering run is past the staged window): driver
        // ends ranked in the window with global fall-backs, then the other
        // list's ends inside the tile
        // (a) fragments ending at driver ends
        const int i0 = cl * IA;
        if (i0 < na_t) {
          int j = smem_lower_bound(wBe, BW, wAe[i0]);
  #pragma unroll
          for (int k = 0; k < IA; ++k) {
            const int i = i0 + k;
            if (i >= na_t) break;
            const int64_t e = wAe[i];
            if (k > 0) {
              j = wBe[j + 1] < e ? j + 2 : j;
              j = wBe[j] < e ? j + 1 : j;
              while (wBe[j] < e) ++j;
            }
            int64_t gj = b_lo + j, pb;
            T vb;
            if (j < b_n) {
              vb = wBv[j];
              pb = j > 0 ? wBe[j - 1] : INT64_MIN;
            } else {  // past the staged window
              gj += lower_bound_g(Be + gj, nb - gj, e);
              vb = gj < nb ? Bv[gj] : T(0);
              pb = gj > 0 ? ldg64(Be, gj - 1) : INT64_MIN;
            }
            const int64_t pa = wAe[i - 1];
            fold(wAv[i], vb, e - (pa > pb ? pa : pb));
          }
        }
        // (b) fragments ending at other-list ends strictly inside (r_lo, r_hi)
        // that are not driver ends; ends past the staged window come from
        // global memory (rare)
        const int jf = smem_lower_bound(wBe, BW, r_lo + 1);  // first window end > r_lo (uniform)
        const int64_t last_in = wBe[b_n > 0 ? b_n - 1 : 0];
        const bool spill = b_n == 0 || (last_in < r_hi && b_lo + b_n < nb);
        const int64_t jcount = (b_n > jf ? b_n - jf : 0);
        const int per = static_cast<int>((jcount + NL - 1) / NL);
        int i = 0;
        bool have_i = false;
        for (int k = 0; k < per; ++k) {
          const int j = jf + cl * per + k;
          if (j >= b_n) break;
          const int64_t e = wBe[j];
          if (e >= r_hi) break;
          if (!have_i) {
            i = smem_lower_bound(wAe, na_t, e);
            have_i = true;
          } else {
            while (wAe[i] < e) ++i;
          }
          if (wAe[i] == e) continue;  // tie: closed by the driver end
          const int64_t pa = wAe[i - 1];
          const int64_t pb = j > 0 ? wBe[j - 1] : INT64_MIN;
          fold(wAv[i], wBv[j], e - (pa > pb ? pa : pb));
        }
        if (spill) {  // other-list ends past the window: strided over consumer lanes
          for (int64_t gj = b_lo + b_n + cl; gj < nb; gj += NL) {
            const int64_t e = ldg64(Be, gj);
            if (e >= r_hi) break;
            if (e <= r_lo) continue;
            const int ii = smem_lower_bound(wAe, na_t, e);
            if (wAe[ii] == e) continue;
            const int64_t pa = wAe[ii - 1];
            const int64_t pb = ldg64(Be, gj - 1);
            fold(wAv[ii], Bv[gj], e - (pa > pb ? pa : pb));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
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
    last = atomicInc(ticket, gridDim.x - 1) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
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
    pp.imin = INT64_MAX;
    pp.imax = INT64_MIN;
    pp.fmin = INFINITY;
    pp.fmax = -INFINITY;
    pp.pad = __longlong_as_double(static_cast<long long>(atomicExch(err, 0)));
    *out = pp;
  }
}

}  // namespace dev

namespace {

constexpr int RB = 256;

struct AggHost {
  uint64_t isum = 0;
  double fsum = 0.0;
  int64_t cnt = 0;
  int64_t imin = INT64_MAX, imax = INT64_MIN;
  double fmin = std::numeric_limits<double>::infinity();
  double fmax = -std::numeric_limits<double>::infinity();
};

int grid_for(const CtxPtr& ctx, int64_t n) {
  int64_t g = (n + RB * 4 - 1) / (RB * 4);
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

AggHost combine(const CtxPtr& ctx, const DArr& parts, int64_t nparts) {
  DArr out = alloc_arr(ctx, RQ_I64, sizeof(dev::AggPart) / 8);
  dev::k_combine<RB><<<1, RB, 0, ctx->stream>>>(parts.as<dev::AggPart>(), nparts,
                                                out.as<dev::AggPart>());
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  const auto* p = reinterpret_cast<const dev::AggPart*>(ctx->readback(out.raw(), sizeof(dev::AggPart)));
  AggHost h;
  h.isum = p->isum;
  h.fsum = p->fsum;
  h.cnt = p->cnt;
  h.imin = p->imin;
  h.imax = p->imax;
  h.fmin = p->fmin;
  h.fmax = p->fmax;
  return h;
}

// runs the slot reduction over several parts (e.g. RLE+Index runs + points)
AggHost reduce_specs(const CtxPtr& ctx, const std::vector<dev::SlotSpec>& specs, bool flt,
                     bool pass2, double mean) {
  int64_t total_blocks = 0;
  std::vector<int> grids;
  for (const auto& sp : specs) {
    grids.push_back(grid_for(ctx, sp.n));
    total_blocks += grids.back();
  }
  DArr parts = alloc_arr(ctx, RQ_I64, total_blocks * (sizeof(dev::AggPart) / 8));
  int64_t off = 0;
  for (size_t k = 0; k < specs.size(); ++k) {
    auto* dst = parts.as<dev::AggPart>() + off;
    if (flt)
      dev::k_reduce_slots<double, RB><<<grids[k], RB, 0, ctx->stream>>>(specs[k], pass2, mean, dst);
    else
      dev::k_reduce_slots<int64_t, RB><<<grids[k], RB, 0, ctx->stream>>>(specs[k], pass2, mean, dst);
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
    off += grids[k];
  }
  return combine(ctx, parts, total_blocks);
}

// Final scalar per AggFn (groupby.cpp:67-135, kernels.cpp:97-125 sentinels).
AggOut finish(int fn, bool flt, const AggHost& h, const AggHost* sq) {
  AggOut o;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  switch (fn) {
    case RQ_SUM:
      if (flt) {
        o.dtype = RQ_F64;
        o.f = h.fsum;
      } else {
        o.dtype = RQ_I64;
        o.i = static_cast<int64_t>(h.isum);
      }
      break;
    case RQ_COUNT:
      o.dtype = RQ_I64;
      o.i = h.cnt;
      break;
    case RQ_MIN:
      if (flt) {
        o.dtype = RQ_F64;
        o.f = h.fmin;
      } else {
        o.dtype = RQ_I64;
        o.i = h.imin;
      }
      break;
    case RQ_MAX:
      if (flt) {
        o.dtype = RQ_F64;
        o.f = h.fmax;
      } else {
        o.dtype = RQ_I64;
        o.i = h.imax;
      }
      break;
    case RQ_AVG:
      o.dtype = RQ_F64;
      o.f = h.cnt > 0 ? h.fsum / static_cast<double>(h.cnt) : nan;
      break;
    case RQ_VAR:
    case RQ_STD: {
      o.dtype = RQ_F64;
      if (h.cnt == 0 || !sq) {
        o.f = nan;
        break;
      }
      const double var = sq->fsum / static_cast<double>(h.cnt);
      o.f = fn == RQ_VAR ? var : std::sqrt(var);
      break;
    }
    default:
      fail("aggregate: unknown function");
  }
  return o;
}

dev::SlotSpec spec_of(const DArr& v, const DArr* s, const DArr* e) {
  dev::SlotSpec sp{};
  sp.v = v.raw();
  sp.dt = v.dt;
  sp.s = s ? s->pos() : nullptr;
  sp.e = e ? e->pos() : nullptr;
  sp.n = v.n;
  return sp;
}

AggOut reduce_with_specs(const CtxPtr& ctx, const std::vector<dev::SlotSpec>& specs, bool flt,
                         int fn) {
  AggHost h = reduce_specs(ctx, specs, flt, false, 0.0);
  if ((fn == RQ_VAR || fn == RQ_STD) && h.cnt > 0) {
    const double mean = h.fsum / static_cast<double>(h.cnt);
    AggHost sq = reduce_specs(ctx, specs, flt, true, mean);
    return finish(fn, flt, h, &sq);
  }
  return finish(fn, flt, h, nullptr);
}

}  // namespace

AggOut reduce_slots(const CtxPtr& ctx, const DArr& v, const DArr* s, const DArr* e, int fn) {
  return reduce_with_specs(ctx, {spec_of(v, s, e)}, dt_float(v.dt), fn);
}

// agg::aggregate_all (groupby.cpp:164-172): normalize_basic then one group.
// Composite parts are reduced in place (no expansion of RLE+Index to rows):
// every aggregate is a fold over covered rows, so runs (weighted) and points
// (unit) contribute to the same accumulators.
AggOut aggregate_column(const CtxPtr& ctx, const DCol& c, int fn) {
  require(fn >= RQ_SUM && fn <= RQ_VAR, "aggregate: unknown function");
  switch (c.enc) {
    case RQ_ENC_PLAIN: {
      dev::SlotSpec sp = spec_of(c.v, nullptr, nullptr);
      const bool flt = dt_float(c.logical) || dt_float(c.v.dt);
      if (!flt && (c.has_center || c.v.dt != c.logical)) {
        sp.decode = 1;
        sp.logical = c.logical;
        sp.has_center = c.has_center ? 1 : 0;
        sp.center = c.center;
        return reduce_with_specs(ctx, {sp}, false, fn);
      }
      if (flt && c.v.dt != c.logical) {
        DArr dec = decode_plain(ctx, c);
        return reduce_with_specs(ctx, {spec_of(dec, nullptr, nullptr)}, true, fn);
      }
      return reduce_with_specs(ctx, {sp}, flt, fn);
    }
    case RQ_ENC_RLE:
      return reduce_with_specs(ctx, {spec_of(c.v, &c.s, &c.e)}, dt_float(c.v.dt), fn);
    case RQ_ENC_INDEX:
      return reduce_with_specs(ctx, {spec_of(c.v, nullptr, nullptr)}, dt_float(c.v.dt), fn);
    case RQ_ENC_PLAIN_INDEX: {
      DArr dec = decode_plain_index(ctx, c);
      return reduce_with_specs(ctx, {spec_of(dec, nullptr, nullptr)}, dt_float(dec.dt), fn);
    }
    case RQ_ENC_RLE_INDEX: {
      require(c.v.dt == c.v2.dt, "array dtype mismatch");  // to_rows merge (column.cpp:353-370)
      std::vector<dev::SlotSpec> specs;
      if (c.s.n) specs.push_back(spec_of(c.v, &c.s, &c.e));
      if (c.p2.n) specs.push_back(spec_of(c.v2, nullptr, nullptr));
      if (specs.empty()) specs.push_back(spec_of(c.v, &c.s, &c.e));
      return reduce_with_specs(ctx, specs, dt_float(c.v.dt), fn);
    }
  }
  fail("aggregate: unknown encoding");
}

namespace {

constexpr int PB = 256, PI = 8;

template <class T, int OP>
void launch_gapless_t(const CtxPtr& ctx, unsigned g, const dev::MergeArgs& m, const DCol& a, const DCol& b,
                      int kind, dev::AggPart* P, int* err) {
  switch (kind) {
    case 0: dev::k_pair_reduce_gapless<PB, PI, T, OP, 0><<<g, PB, 0, ctx->stream>>>(m, a.v.raw(), a.v.dt, b.v.raw(), b.v.dt, P, err); break;
    case 1: dev::k_pair_reduce_gapless<PB, PI, T, OP, 1><<<g, PB, 0, ctx->stream>>>(m, a.v.raw(), a.v.dt, b.v.raw(), b.v.dt, P, err); break;
    default: dev::k_pair_reduce_gapless<PB, PI, T, OP, 2><<<g, PB, 0, ctx->stream>>>(m, a.v.raw(), a.v.dt, b.v.raw(), b.v.dt, P, err); break;
  }
}

void launch_gapless(const CtxPtr& ctx, unsigned g, const dev::MergeArgs& m, const DCol& a, const DCol& b,
                    int op, int kind, bool flt, dev::AggPart* P, int* err) {
  if (flt) {
    switch (op) {
      case RQ_ADD: launch_gapless_t<double, RQ_ADD>(ctx, g, m, a, b, kind, P, err); break;
      case RQ_SUB: launch_gapless_t<double, RQ_SUB>(ctx, g, m, a, b, kind, P, err); break;
      case RQ_MUL: launch_gapless_t<double, RQ_MUL>(ctx, g, m, a, b, kind, P, err); break;
      default: launch_gapless_t<double, RQ_DIV>(ctx, g, m, a, b, kind, P, err); break;
    }
  } else {
    switch (op) {
      case RQ_ADD: launch_gapless_t<int64_t, RQ_ADD>(ctx, g, m, a, b, kind, P, err); break;
      case RQ_SUB: launch_gapless_t<int64_t, RQ_SUB>(ctx, g, m, a, b, kind, P, err); break;
      case RQ_MUL: launch_gapless_t<int64_t, RQ_MUL>(ctx, g, m, a, b, kind, P, err); break;
      default: launch_gapless_t<int64_t, RQ_DIV>(ctx, g, m, a, b, kind, P, err); break;
    }
  }
}

// ---- persistent TMA form (K2) ----
// CTA shape: BLOCK threads (one producer warp), IA driver runs per consumer
// lane, BW-entry window of the other list. TpCfg<128, 10, 768> measured
// best on C1 (sweep of 5..14 runs per lane, 128..256 threads, 384..1024
// window entries: every other shape 3-15% slower).
template <int B_, int I_, int W_>
struct TpCfg {
  static constexpr int BLOCK = B_, IA = I_, BW = W_;
  static constexpr int TA = (B_ - 32) * I_;
  static constexpr size_t SMEM = 2 * dev::PairStage<TA, W_>::BYTES;
};
using TpBase = TpCfg<128, 10, 768>;

template <class C, class T, int OP, int KIND>
void launch_pair_tma3(const CtxPtr& ctx, const DCol& A, const DCol& B, int swap, dev::AggPart* parts,
                      dev::AggPart* out, int ta, int64_t ntiles, int64_t& grid_out, bool dry) {
  auto k = dev::k_pair_reduce_tma<C::BLOCK, C::IA, C::BW, T, OP, KIND>;
  const int occ = kernel_occupancy(ctx, k, C::BLOCK, C::SMEM);
  int64_t grid = static_cast<int64_t>(ctx->sm_count) * occ;
  if (grid > ntiles) grid = ntiles;
  grid_out = grid;
  if (dry) return;
  k<<<static_cast<unsigned>(grid), C::BLOCK, C::SMEM, ctx->stream>>>(
      A.e.pos(), static_cast<const T*>(A.v.raw()), A.e.n, B.e.pos(), static_cast<const T*>(B.v.raw()), B.e.n, swap,
      ta, ntiles, parts, ctx->tickets, out, reinterpret_cast<int*>(ctx->tickets + 3));
}

template <class T, int OP>
void launch_pair_tma2(int kind, const CtxPtr& ctx, const DCol& A, const DCol& B, int swap, dev::AggPart* parts,
                      dev::AggPart* out, int ta, int64_t ntiles, int64_t& grid, bool dry) {
  switch (kind) {
    case 0: launch_pair_tma3<TpBase, T, OP, 0>(ctx, A, B, swap, parts, out, ta, ntiles, grid, dry); break;
    case 1: launch_pair_tma3<TpBase, T, OP, 1>(ctx, A, B, swap, parts, out, ta, ntiles, grid, dry); break;
    default: launch_pair_tma3<TpBase, T, OP, 2>(ctx, A, B, swap, parts, out, ta, ntiles, grid, dry); break;
  }
}

template <class T>
void launch_pair_tma1(int op, int kind, const CtxPtr& ctx, const DCol& A, const DCol& B, int swap,
                      dev::AggPart* parts, dev::AggPart* out, int ta, int64_t ntiles, int64_t& grid, bool dry) {
  switch (op) {
    case RQ_ADD: launch_pair_tma2<T, RQ_ADD>(kind, ctx, A, B, swap, parts, out, ta, ntiles, grid, dry); break;
    case RQ_SUB: launch_pair_tma2<T, RQ_SUB>(kind, ctx, A, B, swap, parts, out, ta, ntiles, grid, dry); break;
    case RQ_MUL: launch_pair_tma2<T, RQ_MUL>(kind, ctx, A, B, swap, parts, out, ta, ntiles, grid, dry); break;
    default: launch_pair_tma2<T, RQ_DIV>(kind, ctx, A, B, swap, parts, out, ta, ntiles, grid, dry); break;
  }
}

// driver runs per tile: the full capacity unless the other list is dense
// enough that its window would overflow (expected window ≈ ta · nb / na)
template <class C>
int tile_runs(const DCol& A, const DCol& B) {
  int ta = C::TA;
  const double ratio = static_cast<double>(B.e.n) / static_cast<double>(A.e.n);
  const int fit = static_cast<int>((C::BW - 16 - 64) / std::max(ratio, 1e-9) * 0.9);
  if (fit < ta) ta = std::max(64, fit & ~1);
  return ta;
}

// gapless RLE × gapless RLE with 8-byte values of the arithmetic type, every
// array bulk-copyable: the persistent kernel (one launch). false otherwise.
bool pair_reduce_tma(const CtxPtr& ctx, const DCol& a, const DCol& b, int op, bool flt, int kind, AggHost& h) {
  const int32_t tdt = flt ? RQ_F64 : RQ_I64;
  if (a.v.dt != tdt || b.v.dt != tdt) return false;
  if (!tma_ok(a.e) || !tma_ok(a.v) || !tma_ok(b.e) || !tma_ok(b.v)) return false;
  const bool a_drives = a.e.n >= b.e.n;  // the list with more runs drives
  const DCol& A = a_drives ? a : b;
  const DCol& B = a_drives ? b : a;
  const int swap = a_drives ? 0 : 1;
  auto launch = [&](dev::AggPart* parts, dev::AggPart* out, int64_t& grid, bool dry) {
    const int ta = tile_runs<TpBase>(A, B);
    const int64_t ntiles = (A.e.n + ta - 1) / ta;
    if (flt) launch_pair_tma1<double>(op, kind, ctx, A, B, swap, parts, out, ta, ntiles, grid, dry);
    else launch_pair_tma1<int64_t>(op, kind, ctx, A, B, swap, parts, out, ta, ntiles, grid, dry);
  };
  int64_t grid = 0;
  launch(nullptr, nullptr, grid, true);
  // partials in the context's scratch; the folded result lands in mapped pinned host memory
  auto* parts = static_cast<dev::AggPart*>(ctx->get_scratch(static_cast<size_t>(grid) * sizeof(dev::AggPart)));
  auto* out = static_cast<dev::AggPart*>(ctx->result_dev);
  {
    KTimer timer(ctx, "pair_reduce");
    launch(parts, out, grid, false);
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  ctx->sync();
  const auto* p = static_cast<const dev::AggPart*>(ctx->result_host);
  h.isum = p->isum;
  h.fsum = p->fsum;
  h.cnt = p->cnt;
  long long e;
  std::memcpy(&e, &p->pad, 8);
  if (!flt && op == RQ_DIV && e) fail("integer division by zero");
  return true;
}

// fast_kind: gapless fast-path accumulator (0 SUM int, 1 SUM f64/AVG, 2
// COUNT) or -1 for the general walk (VAR/STD passes, gapped inputs).
AggHost pair_reduce(const CtxPtr& ctx, const DCol& a, const DCol& b, int op, bool gapless,
                    bool flt, bool pass2, double mean, int fast_kind = -1) {
  if (gapless && fast_kind >= 0 && !pass2) {
    AggHost h;
    const char* off = std::getenv("RQ_NO_TMA");
    if (!(off && off[0] == '1') && pair_reduce_tma(ctx, a, b, op, flt, fast_kind, h)) return h;
  }
  constexpr int TILE = PB * PI;
  const int64_t na = a.e.n, nb = b.e.n;
  const int64_t ntiles = (na + nb + TILE - 1) / TILE;
  DArr part = alloc_arr(ctx, RQ_I64, ntiles + 2);
  auto timer = std::make_unique<KTimer>(ctx, "pair_reduce");
  {
    const int64_t nparts = ntiles + 1;
    const int blocks = static_cast<int>((nparts * 32 + 255) / 256);
    dev::k_merge_partition<<<blocks, 256, 0, ctx->stream>>>(a.e.pos(), na, b.e.pos(), nb, TILE,
                                                            nparts, part.as<int64_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  DArr parts = alloc_arr(ctx, RQ_I64, ntiles * (sizeof(dev::AggPart) / 8));
  DArr err = alloc_arr(ctx, RQ_I32, 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(err.raw_mut(), 0, 4, ctx->stream));
  dev::MergeArgs m{a.e.pos(), na, b.e.pos(), nb, part.as<int64_t>()};
  auto* P = parts.as<dev::AggPart>();
  const unsigned g = static_cast<unsigned>(ntiles);
  if (gapless && fast_kind >= 0) {
    launch_gapless(ctx, g, m, a, b, op, fast_kind, flt, P, err.as<int>());
  } else if (gapless) {
    if (flt) dev::k_pair_reduce<PB, PI, true, double><<<g, PB, 0, ctx->stream>>>(m, a.s.pos(), b.s.pos(), a.v.raw(), a.v.dt, b.v.raw(), b.v.dt, op, pass2, mean, P, err.as<int>());
    else dev::k_pair_reduce<PB, PI, true, int64_t><<<g, PB, 0, ctx->stream>>>(m, a.s.pos(), b.s.pos(), a.v.raw(), a.v.dt, b.v.raw(), b.v.dt, op, pass2, mean, P, err.as<int>());
  } else {
    if (flt) dev::k_pair_reduce<PB, PI, false, double><<<g, PB, 0, ctx->stream>>>(m, a.s.pos(), b.s.pos(), a.v.raw(), a.v.dt, b.v.raw(), b.v.dt, op, pass2, mean, P, err.as<int>());
    else dev::k_pair_reduce<PB, PI, false, int64_t><<<g, PB, 0, ctx->stream>>>(m, a.s.pos(), b.s.pos(), a.v.raw(), a.v.dt, b.v.raw(), b.v.dt, op, pass2, mean, P, err.as<int>());
  }
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  timer.reset();
  AggHost h = combine(ctx, parts, ntiles);
  if (!flt && op == RQ_DIV) {
    const int64_t* e = ctx->readback(err.raw(), 8);
    if (static_cast<int32_t>(e[0] & 0xffffffff)) fail("integer division by zero");
  }
  return h;
}

}  // namespace

// aggregate_all(arith(a, b, op), fn) fused for RLE×RLE (K2); other encoding
// pairs run the materialising operator chain on the device.
AggOut aggregate_binop(const CtxPtr& ctx, const DCol& a, const DCol& b, int op, int fn) {
  require(op >= RQ_ADD && op <= RQ_DIV, "aggregate_binop: arithmetic operator required");
  require(a.total == b.total, "align: total_size mismatch");
  if (a.enc == RQ_ENC_RLE && b.enc == RQ_ENC_RLE && fn != RQ_MIN && fn != RQ_MAX) {
    const bool flt = dt_float(a.v.dt) || dt_float(b.v.dt);
    if (a.e.n == 0 || b.e.n == 0) {
      AggHost h;
      return finish(fn, flt, h, nullptr);
    }
    const bool gapless = col_gapless(ctx, a) && col_gapless(ctx, b);
    int fast_kind = -1;
    if (fn == RQ_SUM) fast_kind = flt ? 1 : 0;
    else if (fn == RQ_AVG) fast_kind = 1;
    else if (fn == RQ_COUNT) fast_kind = 2;
    AggHost h = pair_reduce(ctx, a, b, op, gapless, flt, false, 0.0, fast_kind);
    if ((fn == RQ_VAR || fn == RQ_STD) && h.cnt > 0) {
      AggHost sq = pair_reduce(ctx, a, b, op, gapless, flt, true, h.fsum / static_cast<double>(h.cnt));
      return finish(fn, flt, h, &sq);
    }
    return finish(fn, flt, h, nullptr);
  }
  DCol r = arith(ctx, a, b, op);
  return aggregate_column(ctx, r, fn);
}

}  // namespace rqb
