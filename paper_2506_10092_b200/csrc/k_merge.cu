// k_merge.cu — K1 range_intersect, K3 points_in_runs, K4 points_intersect,
// bucketize. Materialising merge-path kernels with single-pass compaction.
#include "merge_walk.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

__global__ void k_merge_partition(const int64_t* __restrict__ A, int64_t na,
                                  const int64_t* __restrict__ B, int64_t nb, int64_t tile,
                                  int64_t nparts, int64_t* __restrict__ part) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= nparts) return;  // warp-uniform
  int64_t diag = w * tile;
  if (diag > na + nb) diag = na + nb;
  const int64_t i = warp_merge_path(A, na, B, nb, diag);
  if ((threadIdx.x & 31) == 0) part[w] = i;
}

// kernels::bucketize (kernels.cpp:10-19): independent binary search per probe.
__global__ void k_bucketize(const int64_t* __restrict__ x, int64_t nx,
                            const int64_t* __restrict__ b, int64_t nb, int right,
                            int64_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nx) return;
  const int64_t v = ldg64(x, i);
  out[i] = right ? upper_bound_g(b, nb, v) : lower_bound_g(b, nb, v);
}

// Points located by independent binary search (used when the point list is
// much shorter than the run list; same outputs as the merge version).
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK)
    k_points_in_runs_search(const int64_t* __restrict__ p, int64_t np, const int64_t* __restrict__ s,
                            const int64_t* __restrict__ e, int64_t nr, LookBack lb,
                            int64_t* __restrict__ p_out, int64_t* __restrict__ run_of,
                            int64_t* __restrict__ idx_of, int64_t* __restrict__ count_out) {
  __shared__ uint32_t wt[BLOCK / 32 + 1];
  __shared__ uint64_t tile_base;
  const int tile = blockIdx.x;
  const int64_t base = static_cast<int64_t>(tile) * BLOCK * ITEMS + threadIdx.x * ITEMS;
  int64_t runs[ITEMS];
  uint32_t cnt = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    runs[k] = -1;
    const int64_t q = base + k;
    if (q < np) {
      const int64_t pos = ldg64(p, q);
      const int64_t r = lower_bound_g(e, nr, pos);  // first run with e >= pos
      if (r < nr && ldg64(s, r) <= pos) {
        runs[k] = r;
        ++cnt;
      }
    }
  }
  uint32_t total;
  const uint32_t off = block_exclusive<BLOCK>(cnt, total, wt);
  if (threadIdx.x < 32) {
    const uint64_t b0 = lb.exclusive(tile, total);
    if (threadIdx.x == 0) {
      tile_base = b0;
      if (tile == static_cast<int>(gridDim.x) - 1) *count_out = static_cast<int64_t>(b0 + total);
    }
  }
  __syncthreads();
  int64_t o = static_cast<int64_t>(tile_base + off);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (runs[k] >= 0) {
      const int64_t q = base + k;
      if (p_out) p_out[o] = ldg64(p, q);
      if (run_of) run_of[o] = runs[k];
      if (idx_of) idx_of[o] = q;
      ++o;
    }
  }
}

}  // namespace dev

namespace {

constexpr int MB = 256;  // merge block
constexpr int MI = 8;    // merge items per thread
constexpr int MTILE = MB * MI;

// Runs the partition kernel for (A, B); returns the partition array.
DArr merge_partition(const CtxPtr& ctx, const int64_t* A, int64_t na, const int64_t* B, int64_t nb,
                     int64_t tile, int64_t& ntiles) {
  ntiles = (na + nb + tile - 1) / tile;
  DArr part = alloc_arr(ctx, RQ_I64, ntiles + 2);
  const int64_t nparts = ntiles + 1;
  const int64_t threads = nparts * 32;
  const int blocks = static_cast<int>((threads + 255) / 256);
  dev::k_merge_partition<<<blocks, 256, 0, ctx->stream>>>(A, na, B, nb, tile, nparts,
                                                          part.as<int64_t>());
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  return part;
}

template <class Policy>
int64_t merge_select(const CtxPtr& ctx, const int64_t* A, int64_t na, const int64_t* B,
                     int64_t nb, const Policy& pol, const char* tag) {
  if (na + nb == 0) return 0;
  int64_t ntiles = (na + nb + MTILE - 1) / MTILE;
  dev::LookBack lb{nullptr, 0};
  lb.status = ctx->lookback_status(ntiles, &lb.epoch);
  DArr part;
  int64_t* count;
  {
    KTimer timer(ctx, tag);
    part = merge_partition(ctx, A, na, B, nb, MTILE, ntiles);
    dev::MergeArgs m{A, na, B, nb, part.as<int64_t>()};
    count = ctx->count_slot_dev();
    dev::k_merge_select<MB, MI, Policy>
        <<<static_cast<unsigned>(ntiles), MB, 0, ctx->stream>>>(m, pol, lb, count);
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  return ctx->read_count_slot();
}

// Shrink an over-allocated output array's logical length (buffer kept).
void set_len(DArr& a, int64_t n) {
  if (n == 0) a.buf.reset();
  a.n = n;
}

}  // namespace

Intersection range_intersect(const CtxPtr& ctx, const DArr& s1, const DArr& e1, const DArr& s2,
                             const DArr& e2, bool want_idx1, bool want_idx2) {
  require(s1.n == e1.n && s2.n == e2.n, "range_intersect: start/end length mismatch");
  require(s1.dt == RQ_I64 && e1.dt == RQ_I64 && s2.dt == RQ_I64 && e2.dt == RQ_I64,
          "range_intersect: positions must be i64");
  Intersection out;
  const int64_t cap = s1.n + s2.n;
  out.s = alloc_arr(ctx, RQ_I64, cap);
  out.e = alloc_arr(ctx, RQ_I64, cap);
  if (want_idx1) out.idx1 = alloc_arr(ctx, RQ_I64, cap);
  if (want_idx2) out.idx2 = alloc_arr(ctx, RQ_I64, cap);
  dev::IntersectPolicy pol{s1.pos(), e1.pos(), s2.pos(), e2.pos(), s1.n, s2.n,
                           out.s.as<int64_t>(), out.e.as<int64_t>(),
                           want_idx1 ? out.idx1.as<int64_t>() : nullptr,
                           want_idx2 ? out.idx2.as<int64_t>() : nullptr};
  const int64_t n = (s1.n == 0 || s2.n == 0) ? 0 : merge_select(ctx, e1.pos(), e1.n, e2.pos(), e2.n, pol, "range_intersect");
  set_len(out.s, n);
  set_len(out.e, n);
  if (want_idx1) set_len(out.idx1, n);
  if (want_idx2) set_len(out.idx2, n);
  return out;
}

PointsInRuns points_in_runs(const CtxPtr& ctx, const DArr& p, const DArr& s, const DArr& e,
                            bool want_run_of, bool want_idx_of) {
  require(s.n == e.n, "points_in_runs: start/end length mismatch");
  PointsInRuns out;
  const int64_t cap = p.n;
  out.p_out = alloc_arr(ctx, RQ_I64, cap);
  if (want_run_of) out.run_of = alloc_arr(ctx, RQ_I64, cap);
  if (want_idx_of) out.idx_of = alloc_arr(ctx, RQ_I64, cap);
  int64_t n = 0;
  if (p.n > 0 && s.n > 0) {
    int64_t* po = out.p_out.as<int64_t>();
    int64_t* ro = want_run_of ? out.run_of.as<int64_t>() : nullptr;
    int64_t* io = want_idx_of ? out.idx_of.as<int64_t>() : nullptr;
    if (p.n * 24 < s.n) {
      // few points: independent binary searches beat streaming all runs
      constexpr int B = 256, IT = 4;
      const int64_t ntiles = (p.n + B * IT - 1) / (B * IT);
      dev::LookBack lb{nullptr, 0};
      lb.status = ctx->lookback_status(ntiles, &lb.epoch);
      dev::k_points_in_runs_search<B, IT><<<static_cast<unsigned>(ntiles), B, 0, ctx->stream>>>(
          p.pos(), p.n, s.pos(), e.pos(), s.n, lb, po, ro, io, ctx->count_slot_dev());
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
      n = ctx->read_count_slot();
    } else {
      dev::PointsInRunsPolicy pol{s.pos(), s.n, po, ro, io};
      n = merge_select(ctx, p.pos(), p.n, e.pos(), e.n, pol, "points_in_runs");
    }
  }
  set_len(out.p_out, n);
  if (want_run_of) set_len(out.run_of, n);
  if (want_idx_of) set_len(out.idx_of, n);
  return out;
}

PointsIntersect points_intersect(const CtxPtr& ctx, const DArr& p1, const DArr& p2,
                                 bool want_idx1, bool want_idx2) {
  PointsIntersect out;
  const int64_t cap = p1.n < p2.n ? p1.n : p2.n;
  out.p_out = alloc_arr(ctx, RQ_I64, cap);
  if (want_idx1) out.idx1 = alloc_arr(ctx, RQ_I64, cap);
  if (want_idx2) out.idx2 = alloc_arr(ctx, RQ_I64, cap);
  int64_t n = 0;
  if (p1.n > 0 && p2.n > 0) {
    dev::PointsEqPolicy pol{p2.pos(), p2.n, out.p_out.as<int64_t>(),
                            want_idx1 ? out.idx1.as<int64_t>() : nullptr,
                            want_idx2 ? out.idx2.as<int64_t>() : nullptr};
    n = merge_select(ctx, p1.pos(), p1.n, p2.pos(), p2.n, pol, "points_intersect");
  }
  set_len(out.p_out, n);
  if (want_idx1) set_len(out.idx1, n);
  if (want_idx2) set_len(out.idx2, n);
  return out;
}

void merge_disjoint(const CtxPtr& ctx, const DArr& kA, const DArr* eA, const DArr* vA,
                    const DArr& kB, const DArr* eB, const DArr* vB, DArr& k_out, DArr* e_out,
                    DArr* v_out) {
  const int64_t n = kA.n + kB.n;
  k_out = alloc_arr(ctx, RQ_I64, n);
  if (e_out) *e_out = alloc_arr(ctx, RQ_I64, n);
  if (v_out) {
    require(vA && vB && dt_width(vA->dt) == dt_width(vB->dt), "merge_disjoint: value width mismatch");
    *v_out = alloc_arr(ctx, vA->dt, n);
  }
  if (n == 0) return;
  dev::MergeEmitPolicy pol{eA ? eA->pos() : nullptr, eB ? eB->pos() : nullptr,
                           vA ? vA->raw() : nullptr, vB ? vB->raw() : nullptr,
                           vA ? dt_width(vA->dt) : 8, k_out.as<int64_t>(),
                           e_out ? e_out->as<int64_t>() : nullptr,
                           v_out ? v_out->raw_mut() : nullptr};
  const int64_t got = merge_select(ctx, kA.pos(), kA.n, kB.pos(), kB.n, pol, "merge_disjoint");
  require(got == n, "merge_disjoint: count mismatch");
}

DArr union_points(const CtxPtr& ctx, const DArr& p1, const DArr& p2) {
  DArr out = alloc_arr(ctx, RQ_I64, p1.n + p2.n);
  if (p1.n + p2.n == 0) return out;
  dev::UnionPolicy pol{p1.pos(), out.as<int64_t>()};
  const int64_t n = merge_select(ctx, p1.pos(), p1.n, p2.pos(), p2.n, pol, "union_points");
  set_len(out, n);
  return out;
}

DArr points_not_in_runs(const CtxPtr& ctx, const DArr& p, const DArr& s, const DArr& e) {
  DArr out = alloc_arr(ctx, RQ_I64, p.n);
  if (p.n == 0) return out;
  if (s.n == 0) return copy_prefix(ctx, p, p.n);
  dev::PointsNotInRunsPolicy pol{s.pos(), s.n, out.as<int64_t>()};
  const int64_t n = merge_select(ctx, p.pos(), p.n, e.pos(), e.n, pol, "points_not_in_runs");
  set_len(out, n);
  return out;
}

DArr merge_keys(const CtxPtr& ctx, const DArr& a, const DArr& b) {
  DArr out = alloc_arr(ctx, RQ_I64, a.n + b.n);
  if (a.n + b.n == 0) return out;
  dev::MergeKeysPolicy pol{out.as<int64_t>()};
  merge_select(ctx, a.pos(), a.n, b.pos(), b.n, pol, "merge_keys");
  return out;
}

DArr bucketize(const CtxPtr& ctx, const DArr& x, const DArr& b, bool right) {
  require(x.dt == RQ_I64 && b.dt == RQ_I64, "bucketize: i64 inputs required");
  DArr out = alloc_arr(ctx, RQ_I64, x.n);
  if (x.n > 0) {
    const int blocks = static_cast<int>((x.n + 255) / 256);
    dev::k_bucketize<<<blocks, 256, 0, ctx->stream>>>(x.pos(), x.n, b.pos(), b.n, right ? 1 : 0,
                                                      out.as<int64_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  return out;
}

}  // namespace rqb
