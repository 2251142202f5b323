// k_select.cu — K6 predicate→mask with run compaction, mask conversions,
// run expansion and small reductions over positional structures.
//
// Compaction is order-preserving and single-pass: each warp owns 32×ITEMS
// consecutive items, evaluates the predicate with coalesced loads
// (item = base + k·32 + lane), keeps one __ballot_sync word per round,
// ranks survivors with __popc(ballot & lanemask_lt), and CTAs chain their
// offsets with decoupled look-back. Replaces the reference's push_back loops
// (align.cpp:607-619, primitives.cpp:349-368).
#include "device_common.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

template <int BLOCK, int ITEMS, class Policy>
__global__ void __launch_bounds__(BLOCK)
    k_select(int64_t n, Policy pol, LookBack lb, int64_t* __restrict__ count_out) {
  constexpr int NW = BLOCK / 32;
  constexpr int TILE = BLOCK * ITEMS;
  __shared__ uint32_t wt[NW];
  __shared__ uint64_t tile_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t wbase = static_cast<int64_t>(blockIdx.x) * TILE + static_cast<int64_t>(wid) * 32 * ITEMS;
  uint32_t bal[ITEMS];
  uint32_t wcnt = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    const bool f = i < n && pol.flag(i);
    bal[k] = __ballot_sync(FULL, f);
    wcnt += __popc(bal[k]);
  }
  if (lane == 0) wt[wid] = wcnt;
  __syncthreads();
  if (wid == 0) {
    const uint32_t x = lane < NW ? wt[lane] : 0u;
    const uint32_t inc = warp_inclusive(x);
    const uint32_t tot = __shfl_sync(FULL, inc, NW - 1);
    __syncwarp();
    if (lane < NW) wt[lane] = inc - x;
    const uint64_t b = lb.exclusive(blockIdx.x, tot);
    if (lane == 0) {
      tile_base = b;
      if (blockIdx.x == gridDim.x - 1) *count_out = static_cast<int64_t>(b + tot);
    }
  }
  __syncthreads();
  int64_t o = static_cast<int64_t>(tile_base + wt[wid]);
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if ((bal[k] >> lane) & 1u) pol.emit(o + __popc(bal[k] & lt), wbase + k * 32 + lane);
    o += __popc(bal[k]);
  }
}

// ---- policies ---------------------------------------------------------------------

struct RunsByFlags {
  const uint8_t* flags;
  const int64_t *s, *e;
  int64_t *s_out, *e_out;
  __device__ __forceinline__ bool flag(int64_t i) const { return flags[i] != 0; }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const {
    s_out[o] = ldg64(s, i);
    e_out[o] = ldg64(e, i);
  }
};

struct PointsByFlags {
  const uint8_t* flags;
  const int64_t* p;
  int64_t *p_out, *idx_out;
  __device__ __forceinline__ bool flag(int64_t i) const { return flags[i] != 0; }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const {
    p_out[o] = p ? ldg64(p, i) : i;  // no p: the flagged indices themselves
    if (idx_out) idx_out[o] = i;
  }
};

// compare_scalar on an RLE column (align.cpp compare_scalar `case Rle`):
// per-run flag in the promoted type, passing runs kept unmerged.
template <class T>
struct RleCmp {
  const void* v;
  int dt;
  const int64_t *s, *e;
  T k;
  int op;
  bool reversed;
  int64_t *s_out, *e_out;
  __device__ __forceinline__ bool flag(int64_t i) const {
    const T x = ld_as<T>(v, dt, i);
    return reversed ? cmp_t<T>(k, x, op) : cmp_t<T>(x, k, op);
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const {
    s_out[o] = ldg64(s, i);
    e_out[o] = ldg64(e, i);
  }
};

template <class T>
struct IndexCmp {
  const void* v;
  int dt;
  const int64_t* p;
  T k;
  int op;
  bool reversed;
  int64_t* p_out;
  __device__ __forceinline__ bool flag(int64_t i) const {
    const T x = ld_as<T>(v, dt, i);
    return reversed ? cmp_t<T>(k, x, op) : cmp_t<T>(x, k, op);
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const { p_out[o] = ldg64(p, i); }
};

struct MaskTrue {  // plain_mask_to_index (primitives.cpp:362-368)
  const uint8_t* bits;
  int64_t* p_out;
  __device__ __forceinline__ bool flag(int64_t i) const { return bits[i] != 0; }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const { p_out[o] = i; }
};

// plain_mask_to_rle (primitives.cpp:349-360): a run starts where the bit
// rises and ends where it falls; starts and ends are compacted separately
// and pair up by rank.
struct MaskRise {
  const uint8_t* bits;
  int64_t* out;
  __device__ __forceinline__ bool flag(int64_t i) const {
    return bits[i] != 0 && (i == 0 || bits[i - 1] == 0);
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const { out[o] = i; }
};
struct MaskFall {
  const uint8_t* bits;
  int64_t n;
  int64_t* out;
  __device__ __forceinline__ bool flag(int64_t i) const {
    return bits[i] != 0 && (i == n - 1 || bits[i + 1] == 0);
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const { out[o] = i; }
};

// complement_rle / complement_index (primitives.cpp:141-167): candidate gap i
// in [0, n] spans [e_{i-1} + 1, s_i - 1] (with e_{-1} = -1, s_n = total);
// kept when non-empty and inside [0, total).
struct ComplementGaps {
  const int64_t *s, *e;
  int64_t n, total;
  int64_t *s_out, *e_out;
  __device__ __forceinline__ int64_t cs(int64_t i) const { return i == 0 ? 0 : ldg64(e, i - 1) + 1; }
  __device__ __forceinline__ int64_t ce(int64_t i) const { return i == n ? total - 1 : ldg64(s, i) - 1; }
  __device__ __forceinline__ bool flag(int64_t i) const {
    const int64_t a = cs(i), b = ce(i);
    return a <= b && a < total && b >= 0;
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const {
    s_out[o] = cs(i);
    e_out[o] = ce(i);
  }
};

// range_union (primitives.cpp:102-123) over the independently merged start
// list S and end list E: the reference pairs the k-th start with the k-th
// end and breaks where S[i] > running max end + 1; E is sorted, so the
// running max of E[0..i-1] is E[i-1].
struct UnionStart {
  const int64_t *S, *E;
  int64_t* out;
  __device__ __forceinline__ bool flag(int64_t i) const {
    return i == 0 || ldg64(S, i) > ldg64(E, i - 1) + 1;
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const { out[o] = ldg64(S, i); }
};
struct UnionEnd {
  const int64_t *S, *E;
  int64_t n;
  int64_t* out;
  __device__ __forceinline__ bool flag(int64_t i) const {
    return i == n - 1 || ldg64(S, i + 1) > ldg64(E, i) + 1;
  }
  __device__ __forceinline__ void emit(int64_t o, int64_t i) const { out[o] = ldg64(E, i); }
};

// ---- reductions over runs / bytes ----------------------------------------------------

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_sum_lengths(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t n,
                  unsigned long long* __restrict__ out) {
  __shared__ uint64_t red[BLOCK / 32 + 1];
  uint64_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * BLOCK)
    acc += static_cast<uint64_t>(ldg64(e, i) - ldg64(s, i) + 1);
  acc = block_sum<BLOCK>(acc, red);
  if (threadIdx.x == 0) atomicAdd(out, static_cast<unsigned long long>(acc));
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_count_nonzero(const uint8_t* __restrict__ bits, int64_t n, unsigned long long* __restrict__ out) {
  __shared__ uint64_t red[BLOCK / 32 + 1];
  uint64_t acc = 0;
  const int64_t n16 = n / 16;
  const uint4* b16 = reinterpret_cast<const uint4*>(bits);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * BLOCK) {
    const uint4 w = __ldg(b16 + i);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // count nonzero bytes
      const uint32_t x = ws[q];
      const uint32_t nz = ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu | x) & 0x80808080u;
      acc += __popc(nz);
    }
  }
  for (int64_t i = n16 * 16 + static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * BLOCK)
    acc += bits[i] != 0;
  acc = block_sum<BLOCK>(acc, red);
  if (threadIdx.x == 0) atomicAdd(out, static_cast<unsigned long long>(acc));
}

// violations of the gapless tiling s0 = 0, s_i = e_{i-1} + 1, e_last = total - 1
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_gap_check(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t n,
                int64_t total, unsigned long long* __restrict__ out) {
  __shared__ uint64_t red[BLOCK / 32 + 1];
  uint64_t bad = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * BLOCK) {
    const int64_t si = ldg64(s, i);
    const int64_t prev = i == 0 ? -1 : ldg64(e, i - 1);
    bad += si != prev + 1;
    if (i == n - 1) bad += ldg64(e, i) != total - 1;
  }
  bad = block_sum<BLOCK>(bad, red);
  if (threadIdx.x == 0 && bad) atomicAdd(out, static_cast<unsigned long long>(bad));
}

// exclusive scan of run lengths (range_arange / compact_rle offsets) with
// decoupled look-back; blocked ITEMS per thread.
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK)
    k_scan_lengths(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t n,
                   LookBack lb, int64_t* __restrict__ offs, int64_t* __restrict__ total_out) {
  __shared__ uint64_t wt[BLOCK / 32 + 1];
  __shared__ uint64_t tile_base;
  const int64_t base = (static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x) * ITEMS;
  uint64_t len[ITEMS];
  uint64_t sum = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t i = base + k;
    len[k] = i < n ? static_cast<uint64_t>(ldg64(e, i) - ldg64(s, i) + 1) : 0;
    sum += len[k];
  }
  uint64_t total;
  uint64_t off = block_exclusive<BLOCK>(sum, total, wt);
  if (threadIdx.x < 32) {
    const uint64_t b = lb.exclusive(blockIdx.x, total);
    if (threadIdx.x == 0) {
      tile_base = b;
      if (blockIdx.x == gridDim.x - 1) *total_out = static_cast<int64_t>(b + total);
    }
  }
  __syncthreads();
  off += tile_base;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t i = base + k;
    if (i < n) offs[i] = static_cast<int64_t>(off);
    off += len[k];
  }
}

// range_arange (kernels.cpp:47-60) over runs: output row k belongs to run
// r = upper_bound(offs, k) - 1 and sits at s_r + (k - offs_r).
template <int ITEMS>
__global__ void k_expand_runs(const int64_t* __restrict__ s, const int64_t* __restrict__ offs,
                              int64_t nr, int64_t rows, int64_t* __restrict__ positions,
                              int64_t* __restrict__ run_idx) {
  const int64_t base = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * ITEMS;
  if (base >= rows) return;
  int64_t r = upper_bound_g(offs, nr, base) - 1;
  int64_t next = r + 1 < nr ? ldg64(offs, r + 1) : INT64_MAX;
  int64_t start = ldg64(offs, r);
  int64_t sr = ldg64(s, r);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t row = base + k;
    if (row >= rows) break;
    while (row >= next) {
      ++r;
      start = next;
      next = r + 1 < nr ? ldg64(offs, r + 1) : INT64_MAX;
      sr = ldg64(s, r);
    }
    if (positions) positions[row] = sr + (row - start);
    if (run_idx) run_idx[row] = r;
  }
}

__global__ void k_compact_ends(const int64_t* __restrict__ offs, const int64_t* __restrict__ s,
                               const int64_t* __restrict__ e, int64_t n, int64_t* __restrict__ e_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) e_out[i] = ldg64(offs, i) + (ldg64(e, i) - ldg64(s, i));
}

}  // namespace dev

namespace {

constexpr int SB = 256;
constexpr int SI = 8;
constexpr int STILE = SB * SI;

template <class Policy>
int64_t run_select(const CtxPtr& ctx, int64_t n, const Policy& pol) {
  if (n == 0) return 0;
  const int64_t ntiles = (n + STILE - 1) / STILE;
  dev::LookBack lb{nullptr, 0};
  lb.status = ctx->lookback_status(ntiles, &lb.epoch);
  dev::k_select<SB, SI, Policy><<<static_cast<unsigned>(ntiles), SB, 0, ctx->stream>>>(
      n, pol, lb, ctx->count_slot_dev());
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  return ctx->read_count_slot();
}

void set_len(DArr& a, int64_t n) {
  if (n == 0) a.buf.reset();
  a.n = n;
}

int grid_for(const CtxPtr& ctx, int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace

void select_runs(const CtxPtr& ctx, const DArr& flags, const DArr& s, const DArr& e, DArr& s_out,
                 DArr& e_out) {
  s_out = alloc_arr(ctx, RQ_I64, s.n);
  e_out = alloc_arr(ctx, RQ_I64, s.n);
  dev::RunsByFlags pol{flags.as<uint8_t>(), s.pos(), e.pos(), s_out.as<int64_t>(),
                       e_out.as<int64_t>()};
  const int64_t n = run_select(ctx, s.n, pol);
  set_len(s_out, n);
  set_len(e_out, n);
}

void select_points(const CtxPtr& ctx, const DArr& flags, const DArr& p, DArr& p_out,
                   DArr* idx_out) {
  p_out = alloc_arr(ctx, RQ_I64, p.n);
  if (idx_out) *idx_out = alloc_arr(ctx, RQ_I64, p.n);
  dev::PointsByFlags pol{flags.as<uint8_t>(), p.pos(), p_out.as<int64_t>(),
                         idx_out ? idx_out->as<int64_t>() : nullptr};
  const int64_t n = run_select(ctx, p.n, pol);
  set_len(p_out, n);
  if (idx_out) set_len(*idx_out, n);
}

// indices of the set flags (select_points over iota without materialising it)
void flagged_indices(const CtxPtr& ctx, const DArr& flags, int64_t n, DArr& out) {
  out = alloc_arr(ctx, RQ_I64, n);
  dev::PointsByFlags pol{flags.as<uint8_t>(), nullptr, out.as<int64_t>(), nullptr};
  set_len(out, run_select(ctx, n, pol));
}

void rle_cmp_scalar_select(const CtxPtr& ctx, const DArr& v, const DArr& s, const DArr& e,
                           Scalar k, int op, bool reversed, DArr& s_out, DArr& e_out) {
  s_out = alloc_arr(ctx, RQ_I64, s.n);
  e_out = alloc_arr(ctx, RQ_I64, s.n);
  int64_t n;
  if (dt_float(v.dt) || k.is_float) {
    const double kd = k.is_float ? k.f : static_cast<double>(k.i);
    dev::RleCmp<double> pol{v.raw(), v.dt, s.pos(), e.pos(), kd, op, reversed,
                            s_out.as<int64_t>(), e_out.as<int64_t>()};
    n = run_select(ctx, s.n, pol);
  } else {
    dev::RleCmp<int64_t> pol{v.raw(), v.dt, s.pos(), e.pos(), k.i, op, reversed,
                             s_out.as<int64_t>(), e_out.as<int64_t>()};
    n = run_select(ctx, s.n, pol);
  }
  set_len(s_out, n);
  set_len(e_out, n);
}

void index_cmp_scalar_select(const CtxPtr& ctx, const DArr& v, const DArr& p, Scalar k, int op,
                             bool reversed, DArr& p_out) {
  p_out = alloc_arr(ctx, RQ_I64, p.n);
  int64_t n;
  if (dt_float(v.dt) || k.is_float) {
    const double kd = k.is_float ? k.f : static_cast<double>(k.i);
    dev::IndexCmp<double> pol{v.raw(), v.dt, p.pos(), kd, op, reversed, p_out.as<int64_t>()};
    n = run_select(ctx, p.n, pol);
  } else {
    dev::IndexCmp<int64_t> pol{v.raw(), v.dt, p.pos(), k.i, op, reversed, p_out.as<int64_t>()};
    n = run_select(ctx, p.n, pol);
  }
  set_len(p_out, n);
}

void plain_mask_to_rle(const CtxPtr& ctx, const DArr& bits, DArr& s, DArr& e) {
  const int64_t cap = bits.n / 2 + 1;
  s = alloc_arr(ctx, RQ_I64, cap);
  e = alloc_arr(ctx, RQ_I64, cap);
  dev::MaskRise rise{bits.as<uint8_t>(), s.as<int64_t>()};
  dev::MaskFall fall{bits.as<uint8_t>(), bits.n, e.as<int64_t>()};
  const int64_t ns = run_select(ctx, bits.n, rise);
  const int64_t ne = run_select(ctx, bits.n, fall);
  require(ns == ne, "plain_mask_to_rle: start/end count mismatch");
  set_len(s, ns);
  set_len(e, ne);
}

void complement_runs(const CtxPtr& ctx, const DArr& s, const DArr& e, int64_t total, DArr& s_out,
                     DArr& e_out) {
  s_out = alloc_arr(ctx, RQ_I64, s.n + 1);
  e_out = alloc_arr(ctx, RQ_I64, s.n + 1);
  dev::ComplementGaps pol{s.pos(), e.pos(), s.n, total, s_out.as<int64_t>(), e_out.as<int64_t>()};
  const int64_t n = run_select(ctx, s.n + 1, pol);
  set_len(s_out, n);
  set_len(e_out, n);
}

void union_from_merged(const CtxPtr& ctx, const DArr& S, const DArr& E, DArr& s_out, DArr& e_out) {
  s_out = alloc_arr(ctx, RQ_I64, S.n);
  e_out = alloc_arr(ctx, RQ_I64, S.n);
  dev::UnionStart us{S.pos(), E.pos(), s_out.as<int64_t>()};
  dev::UnionEnd ue{S.pos(), E.pos(), S.n, e_out.as<int64_t>()};
  const int64_t ns = run_select(ctx, S.n, us);
  const int64_t ne = run_select(ctx, S.n, ue);
  require(ns == ne, "range_union: start/end count mismatch");
  set_len(s_out, ns);
  set_len(e_out, ne);
}

DArr plain_mask_to_index(const CtxPtr& ctx, const DArr& bits) {
  const int64_t cnt = count_nonzero(ctx, bits);
  DArr p = alloc_arr(ctx, RQ_I64, cnt);
  if (cnt == 0) return p;
  dev::MaskTrue pol{bits.as<uint8_t>(), p.as<int64_t>()};
  const int64_t n = run_select(ctx, bits.n, pol);
  require(n == cnt, "plain_mask_to_index: count mismatch");
  return p;
}

int64_t covered_rows(const CtxPtr& ctx, const DArr& s, const DArr& e) {
  if (s.n == 0) return 0;
  DArr acc = alloc_arr(ctx, RQ_I64, 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(acc.raw_mut(), 0, 8, ctx->stream));
  dev::k_sum_lengths<256><<<grid_for(ctx, s.n, 256), 256, 0, ctx->stream>>>(
      s.pos(), e.pos(), s.n, reinterpret_cast<unsigned long long*>(acc.raw_mut()));
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  return *ctx->readback(acc.raw(), 8);
}

int64_t count_nonzero(const CtxPtr& ctx, const DArr& bits) {
  if (bits.n == 0) return 0;
  DArr acc = alloc_arr(ctx, RQ_I64, 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(acc.raw_mut(), 0, 8, ctx->stream));
  dev::k_count_nonzero<256><<<grid_for(ctx, bits.n / 16 + 1, 256), 256, 0, ctx->stream>>>(
      bits.as<uint8_t>(), bits.n, reinterpret_cast<unsigned long long*>(acc.raw_mut()));
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  return *ctx->readback(acc.raw(), 8);
}

bool runs_gapless(const CtxPtr& ctx, const DArr& s, const DArr& e, int64_t total) {
  if (s.n == 0) return total == 0;
  DArr acc = alloc_arr(ctx, RQ_I64, 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(acc.raw_mut(), 0, 8, ctx->stream));
  dev::k_gap_check<256><<<grid_for(ctx, s.n, 256), 256, 0, ctx->stream>>>(
      s.pos(), e.pos(), s.n, total, reinterpret_cast<unsigned long long*>(acc.raw_mut()));
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  return *ctx->readback(acc.raw(), 8) == 0;
}

namespace {
// offsets = exclusive scan of run lengths; returns total covered rows
DArr scan_lengths(const CtxPtr& ctx, const DArr& s, const DArr& e, int64_t& total) {
  constexpr int B = 256, IT = 8;
  DArr offs = alloc_arr(ctx, RQ_I64, s.n + 1);
  const int64_t ntiles = (s.n + B * IT - 1) / (B * IT);
  dev::LookBack lb{nullptr, 0};
  lb.status = ctx->lookback_status(ntiles, &lb.epoch);
  int64_t* tot = offs.as<int64_t>() + s.n;
  dev::k_scan_lengths<B, IT><<<static_cast<unsigned>(ntiles), B, 0, ctx->stream>>>(
      s.pos(), e.pos(), s.n, lb, offs.as<int64_t>(), tot);
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  total = *ctx->readback(tot, 8);
  return offs;
}
}  // namespace

void expand_runs(const CtxPtr& ctx, const DArr& s, const DArr& e, DArr* positions,
                 DArr* run_idx) {
  int64_t rows = 0;
  DArr offs;
  if (s.n > 0) offs = scan_lengths(ctx, s, e, rows);
  if (positions) *positions = alloc_arr(ctx, RQ_I64, rows);
  if (run_idx) *run_idx = alloc_arr(ctx, RQ_I64, rows);
  if (rows == 0) return;
  constexpr int IT = 8;
  const int64_t threads = (rows + IT - 1) / IT;
  dev::k_expand_runs<IT><<<static_cast<unsigned>((threads + 255) / 256), 256, 0, ctx->stream>>>(
      s.pos(), offs.pos(), s.n, rows, positions ? positions->as<int64_t>() : nullptr,
      run_idx ? run_idx->as<int64_t>() : nullptr);
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
}

// compact_rle (primitives.cpp:370-379): s' = exclusive cumsum(l), e' = s' + l - 1
DArr compact_positions(const CtxPtr& ctx, const DArr& s, const DArr& e, DArr& e_out,
                       int64_t* covered) {
  int64_t rows = 0;
  if (covered) *covered = 0;
  if (s.n == 0) {
    e_out = alloc_arr(ctx, RQ_I64, 0);
    return alloc_arr(ctx, RQ_I64, 0);
  }
  DArr offs = scan_lengths(ctx, s, e, rows);
  if (covered) *covered = rows;
  e_out = alloc_arr(ctx, RQ_I64, s.n);
  dev::k_compact_ends<<<static_cast<unsigned>((s.n + 255) / 256), 256, 0, ctx->stream>>>(
      offs.pos(), s.pos(), e.pos(), s.n, e_out.as<int64_t>());
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
  offs.n = s.n;  // drop the total slot
  return offs;
}

}  // namespace rqb
