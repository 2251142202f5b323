// merge_walk.cuh — merge-path tile machinery over two sorted int64 key lists.
//
// The reference aligns two position-sorted structures with a searchsorted +
// repeat_interleave + range_arange pipeline (primitives.cpp:15-46 over
// kernels.cpp:10-60), i.e. one binary search per run plus materialised
// per-fragment index arrays. Here the merged order of the two key lists
// (run ends, point positions) is split into equal diagonal tiles (merge
// path): a partition kernel locates each tile's start with a warp-cooperative
// 32-ary search, each CTA stages its tile's keys in shared memory with
// coalesced loads, and every thread walks ITEMS consecutive merge steps.
// A step consumes one key from A or B (ties take A first) and knows the
// cursor of the other list, which is exactly the pair (i, j) of the
// reference's overlap formula.
#pragma once

#include "device_common.cuh"

namespace rqb {
namespace dev {

struct MergeArgs {
  const int64_t* A;
  int64_t na;
  const int64_t* B;
  int64_t nb;
  const int64_t* part;  // A-count at each tile boundary (ntiles + 1)
};

// one warp per tile boundary
__global__ void k_merge_partition(const int64_t* __restrict__ A, int64_t na,
                                  const int64_t* __restrict__ B, int64_t nb, int64_t tile,
                                  int64_t nparts, int64_t* __restrict__ part);

// merge-path search inside shared memory: A = sk[0, a), B = sk[a, a + b)
__device__ __forceinline__ int smem_merge_path(const int64_t* sk, int a, int b, int diag) {
  int lo = diag > b ? diag - b : 0;
  int hi = diag < a ? diag : a;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sk[mid] <= sk[a + diag - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int BLOCK, int ITEMS>
struct MergeTile {
  static constexpr int TILE = BLOCK * ITEMS;
  int64_t i0, j0;  // global start of the A / B segments
  int a, b;        // segment lengths
  int ti, tj;      // this thread's start inside the segments

  // Loads the tile's keys into sk (TILE entries) and positions the thread.
  __device__ __forceinline__ void load(const MergeArgs& m, int tile, int64_t* sk) {
    const int64_t d0 = static_cast<int64_t>(tile) * TILE;
    int64_t d1 = d0 + TILE;
    if (d1 > m.na + m.nb) d1 = m.na + m.nb;
    i0 = m.part[tile];
    const int64_t i1 = m.part[tile + 1];
    j0 = d0 - i0;
    const int64_t j1 = d1 - i1;
    a = static_cast<int>(i1 - i0);
    b = static_cast<int>(j1 - j0);
    // a + b <= TILE: ITEMS unrolled, independent coalesced loads per thread
    const int64_t* pa = m.A + i0;
    const int64_t* pb = m.B + j0 - a;
    int64_t t[ITEMS];
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int k = u * BLOCK + threadIdx.x;
      t[u] = k < a + b ? __ldg(reinterpret_cast<const long long*>(k < a ? pa : pb) + k) : 0;
    }
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int k = u * BLOCK + threadIdx.x;
      if (k < a + b) sk[k] = t[u];
    }
    __syncthreads();
    int diag = threadIdx.x * ITEMS;
    if (diag > a + b) diag = a + b;
    ti = smem_merge_path(sk, a, b, diag);
    tj = diag - ti;
  }

  // f(i_global, j_global, takeA, key): i/j are the consumed element's index
  // in its list and the other list's cursor.
  template <class F>
  __device__ __forceinline__ void walk(const int64_t* sk, F&& f) const {
    int x = ti, y = tj;
#pragma unroll 4
    for (int it = 0; it < ITEMS; ++it) {
      if (x + y >= a + b) break;
      const int64_t ka = x < a ? sk[x] : KEY_MAX;
      const int64_t kb = y < b ? sk[a + y] : KEY_MAX;
      const bool takeA = (y >= b) || (x < a && ka <= kb);
      f(i0 + x, j0 + y, takeA, takeA ? ka : kb);
      if (takeA) ++x;
      else ++y;
    }
  }

  // Merged key immediately before this thread's first step (-1 if none).
  __device__ __forceinline__ int64_t prev_key(const int64_t* sk, const MergeArgs& m) const {
    int64_t pa = -1, pb = -1;
    if (ti > 0) pa = sk[ti - 1];
    else if (i0 > 0) pa = ldg64(m.A, i0 - 1);
    if (tj > 0) pb = sk[a + tj - 1];
    else if (j0 > 0) pb = ldg64(m.B, j0 - 1);
    return pa > pb ? pa : pb;
  }
};

// Materialising select over the merge: Policy::test(i, j, takeA, key) -> 0/1
// and Policy::emit(out, i, j, takeA, key). Output order = merge order
// (position order). Two walks per tile (count, then write) around one
// block scan + decoupled look-back, so the input is read once.
template <int BLOCK, int ITEMS, class Policy>
__global__ void __launch_bounds__(BLOCK)
    k_merge_select(MergeArgs m, Policy pol, LookBack lb, int64_t* __restrict__ count_out) {
  using Tile = MergeTile<BLOCK, ITEMS>;
  __shared__ int64_t sk[Tile::TILE];
  __shared__ uint32_t wt[BLOCK / 32 + 1];
  __shared__ uint64_t tile_base;
  Tile t;
  const int tile = blockIdx.x;
  t.load(m, tile, sk);
  uint32_t cnt = 0;
  t.walk(sk, [&](int64_t i, int64_t j, bool takeA, int64_t key) {
    cnt += pol.test(i, j, takeA, key) ? 1u : 0u;
  });
  uint32_t total;
  const uint32_t off = block_exclusive<BLOCK>(cnt, total, wt);
  if (threadIdx.x < 32) {
    const uint64_t base = lb.exclusive(tile, total);
    if (threadIdx.x == 0) {
      tile_base = base;
      if (tile == static_cast<int>(gridDim.x) - 1) *count_out = static_cast<int64_t>(base + total);
    }
  }
  __syncthreads();
  if (cnt == 0) return;
  int64_t o = static_cast<int64_t>(tile_base + off);
  t.walk(sk, [&](int64_t i, int64_t j, bool takeA, int64_t key) {
    if (pol.test(i, j, takeA, key)) pol.emit(o++, i, j, takeA, key);
  });
}

// ---- policies ---------------------------------------------------------------------

// enc::range_intersect (primitives.cpp:15-46): A = e1, B = e2. The fragment
// of runs (i, j) is [max(s1_i, s2_j), min(e1_i, e2_j)]; it is produced at the
// merge step of its smaller end (ties: at A's step), so every overlapping
// pair appears exactly once and fragments come out in position order —
// the same list the reference produces (primitives.hpp:24-27).
struct IntersectPolicy {
  const int64_t *s1, *e1, *s2, *e2;
  int64_t n1, n2;
  int64_t *s, *e, *idx1, *idx2;

  __device__ __forceinline__ bool test(int64_t i, int64_t j, bool takeA, int64_t key) const {
    if (takeA) {
      if (j >= n2) return false;
      const int64_t lo = max(ldg64(s1, i), ldg64(s2, j));
      return lo <= key;
    }
    if (i >= n1) return false;
    const int64_t lo = max(ldg64(s1, i), ldg64(s2, j));
    return lo <= key;
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i, int64_t j, bool, int64_t key) const {
    const int64_t lo = max(ldg64(s1, i), ldg64(s2, j));
    s[o] = lo;
    e[o] = key;
    if (idx1) idx1[o] = i;
    if (idx2) idx2[o] = j;
  }
};

// enc::idx_in_rle / rle_contain_idx (primitives.cpp:48-86): A = points p,
// B = run ends e. A point step with run cursor j (= #ends < p) is inside run
// j iff s_j <= p.
struct PointsInRunsPolicy {
  const int64_t* s;
  int64_t nr;
  int64_t *p_out, *run_of, *idx_of;

  __device__ __forceinline__ bool test(int64_t, int64_t j, bool takeA, int64_t key) const {
    return takeA && j < nr && ldg64(s, j) <= key;
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i, int64_t j, bool, int64_t key) const {
    if (p_out) p_out[o] = key;
    if (run_of) run_of[o] = j;
    if (idx_of) idx_of[o] = i;
  }
};

// enc::idx_in_idx (primitives.cpp:88-100): A = p1, B = p2; a p1 step with
// cursor j (= #p2 < p1_i) matches iff p2_j == p1_i.
struct PointsEqPolicy {
  const int64_t* p2;
  int64_t n2;
  int64_t *p_out, *idx1, *idx2;

  __device__ __forceinline__ bool test(int64_t, int64_t j, bool takeA, int64_t key) const {
    return takeA && j < n2 && ldg64(p2, j) == key;
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i, int64_t j, bool, int64_t key) const {
    if (p_out) p_out[o] = key;
    if (idx1) idx1[o] = i;
    if (idx2) idx2[o] = j;
  }
};

// Merge of two DISJOINT sorted position lists carrying values (and an
// optional second position array, run ends): every step emits its element.
// align.cpp merge_disjoint_points / merge_disjoint_runs (:384-439) and the
// RLE+Index to_rows merge (column.cpp:349-372).
struct MergeEmitPolicy {
  const int64_t *eA, *eB;  // optional run ends travelling with the keys
  const void *vA, *vB;     // values (same byte width)
  int width;
  int64_t *k_out, *e_out;
  void* v_out;
  __device__ __forceinline__ bool test(int64_t, int64_t, bool, int64_t) const { return true; }
  __device__ __forceinline__ void emit(int64_t o, int64_t i, int64_t j, bool takeA, int64_t key) const {
    k_out[o] = key;
    const int64_t src = takeA ? i : j;
    if (e_out) e_out[o] = ldg64(takeA ? eA : eB, src);
    if (v_out) {
      const char* vs = static_cast<const char*>(takeA ? vA : vB);
      switch (width) {
        case 1: static_cast<uint8_t*>(v_out)[o] = reinterpret_cast<const uint8_t*>(vs)[src]; break;
        case 2: static_cast<uint16_t*>(v_out)[o] = reinterpret_cast<const uint16_t*>(vs)[src]; break;
        case 4: static_cast<uint32_t*>(v_out)[o] = reinterpret_cast<const uint32_t*>(vs)[src]; break;
        default: static_cast<uint64_t*>(v_out)[o] = reinterpret_cast<const uint64_t*>(vs)[src]; break;
      }
    }
  }
};

// Points NOT inside any run (subtract_runs, mask_ops.cpp:94-108): A = points,
// B = run ends; complement of PointsInRunsPolicy's test.
struct PointsNotInRunsPolicy {
  const int64_t* s;
  int64_t nr;
  int64_t* p_out;
  __device__ __forceinline__ bool test(int64_t, int64_t j, bool takeA, int64_t key) const {
    return takeA && !(j < nr && ldg64(s, j) <= key);
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t, int64_t, bool, int64_t key) const {
    p_out[o] = key;
  }
};

// Merge of two sorted lists keeping duplicates (range_union's std::merge of
// the start lists and of the end lists, primitives.cpp:107-110).
struct MergeKeysPolicy {
  int64_t* out;
  __device__ __forceinline__ bool test(int64_t, int64_t, bool, int64_t) const { return true; }
  __device__ __forceinline__ void emit(int64_t o, int64_t, int64_t, bool, int64_t key) const {
    out[o] = key;
  }
};

// Sorted de-duplicated union of two strictly increasing position lists
// (merge_sorted_idx / concat_sort_idx, primitives.cpp:125-139 — both give the
// same list). Ties take A first, so a B step equal to the last A key is a
// duplicate.
struct UnionPolicy {
  const int64_t* A;
  int64_t* out;
  __device__ __forceinline__ bool test(int64_t i, int64_t, bool takeA, int64_t key) const {
    return takeA || i == 0 || ldg64(A, i - 1) != key;
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t, int64_t, bool, int64_t key) const {
    out[o] = key;
  }
};

}  // namespace dev
}  // namespace rqb
