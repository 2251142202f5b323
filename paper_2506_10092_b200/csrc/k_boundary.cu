// k_boundary.cu — the rest of the reference operator API surface (SURVEY.md
// §8b): the runq::kernels helpers (cumsum / checked_sum / repeat_interleave /
// range_arange / scatter_reduce / unique_with_inverse / gather / sort_with_perm /
// adjacent_ne, kernels.cpp), the shape weights and aggregate_array of the
// grouping API (align.cpp:57-70, groupby.cpp:67-135), the RLE expansions
// (rle_to_index / rle_to_plain, primitives.cpp:172-220), compact_rle_index
// (primitives.cpp:381-420) and decode_full / to_rows (column.cpp:311-376).
// These are the entry points the reference's own tests and the drop-in
// adapter call; the fused query kernels do not go through them.
//
// Exactness: integer prefix sums are carried in 128 bits so the first
// element whose running int64 sum overflows is found exactly (the reference
// checks every addition with __builtin_add_overflow); scatter_reduce folds
// each group's values in input order (stable sort by group, one sequential
// fold per group), so f64 sums are bit-identical to the reference's loop.
#include <cmath>
#include <cstring>

#include "device_common.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

constexpr int BT = 256, BI = 8, BTILE = BT * BI;

using i128 = __int128;

__device__ __forceinline__ bool fits_i64(i128 x) {
  return x >= static_cast<i128>(INT64_MIN) && x <= static_cast<i128>(INT64_MAX);
}

__global__ void __launch_bounds__(BT) k_tile_sums(const int64_t* __restrict__ x, int64_t n, i128* __restrict__ sums) {
  __shared__ i128 sm[BT];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * BTILE;
  i128 acc = 0;
  for (int k = 0; k < BI; ++k) {
    const int64_t i = base + static_cast<int64_t>(threadIdx.x) * BI + k;
    if (i < n) acc += x[i];
  }
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int w = BT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = sm[0];
}

// exclusive prefix of the tile sums (one thread: tiles = n / 2048)
__global__ void k_tile_prefix(i128* __restrict__ sums, int64_t tiles) {
  i128 acc = 0;
  for (int64_t t = 0; t < tiles; ++t) {
    const i128 v = sums[t];
    sums[t] = acc;
    acc += v;
  }
}

// out = (exclusive or inclusive) prefix; bad = first element whose inclusive
// prefix leaves int64 (the reference's overflow point)
__global__ void __launch_bounds__(BT) k_tile_apply(const int64_t* __restrict__ x, int64_t n, const i128* __restrict__ offs,
                                                   int exclusive, int64_t* __restrict__ out,
                                                   unsigned long long* __restrict__ bad) {
  __shared__ i128 sm[BT];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * BTILE + static_cast<int64_t>(threadIdx.x) * BI;
  i128 mine = 0;
  for (int k = 0; k < BI; ++k)
    if (base + k < n) mine += x[base + k];
  sm[threadIdx.x] = mine;
  __syncthreads();
  for (int w = 1; w < BT; w <<= 1) {  // Hillis-Steele inclusive scan
    const i128 add = threadIdx.x >= w ? sm[threadIdx.x - w] : 0;
    __syncthreads();
    sm[threadIdx.x] += add;
    __syncthreads();
  }
  i128 acc = offs[blockIdx.x] + sm[threadIdx.x] - mine;
  for (int k = 0; k < BI; ++k) {
    const int64_t i = base + k;
    if (i >= n) break;
    const i128 next = acc + x[i];
    if (!fits_i64(next)) atomicMin(bad, static_cast<unsigned long long>(i));
    if (out) out[i] = static_cast<int64_t>(exclusive ? acc : next);
    acc = next;
  }
}

// first index i with x[i] < lo or x[i] >= hi (hi < 0: no upper bound)
__global__ void k_first_outside(const int64_t* __restrict__ x, int64_t n, int64_t lo, int64_t hi,
                                unsigned long long* __restrict__ bad) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = x[i];
    if (v < lo || (hi >= 0 && v >= hi)) atomicMin(bad, static_cast<unsigned long long>(i));
  }
}

// expansion of segments of `counts` (exclusive offsets `off`) to `total`
// elements: mode 0 copies values[j] (w bytes), mode 1 writes start[j] + (i - off[j])
__global__ void k_expand(const int64_t* __restrict__ off, int64_t nseg, int64_t total, int mode,
                         const void* __restrict__ src, int w, void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = nseg;  // upper_bound(off, i) - 1
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid] <= i) lo = mid + 1;
      else hi = mid;
    }
    const int64_t j = lo - 1;
    if (mode == 1) {
      static_cast<int64_t*>(out)[i] = static_cast<const int64_t*>(src)[j] + (i - off[j]);
      continue;
    }
    switch (w) {
      case 1: static_cast<uint8_t*>(out)[i] = static_cast<const uint8_t*>(src)[j]; break;
      case 2: static_cast<uint16_t*>(out)[i] = static_cast<const uint16_t*>(src)[j]; break;
      case 4: static_cast<uint32_t*>(out)[i] = static_cast<const uint32_t*>(src)[j]; break;
      default: static_cast<uint64_t*>(out)[i] = static_cast<const uint64_t*>(src)[j]; break;
    }
  }
}

// Large groups (many elements per group, few groups): each warp folds a
// contiguous range of the input in order into its own row of a partial table
// (lanes of one group combined in lane order, then one plain add by the
// leader); integer folds go straight to the output with atomics (exact in
// any order). Row init: 0 / +inf / -inf for sum / min / max.
__global__ void k_group_fold_warp(const void* __restrict__ v, int dt, const int64_t* __restrict__ idx, int64_t n,
                                  int64_t G, int op, int flt, int64_t per_warp, double* __restrict__ fpart,
                                  unsigned long long* __restrict__ iout) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  double* row = flt ? fpart + w * G : nullptr;
  if (flt) {
    const double init = op == 1 ? INFINITY : op == 2 ? -INFINITY : 0.0;
    for (int64_t g = lane; g < G; g += 32) row[g] = init;
    __syncwarp();
  }
  const int64_t a = w * per_warp, b = min(n, a + per_warp);
  for (int64_t base = a; base < b; base += 32) {
    const int64_t j = base + lane;
    const bool ok = j < b;
    const int64_t g = ok ? idx[j] : -1;
    const unsigned same = __match_any_sync(FULL, static_cast<unsigned long long>(g));
    const int leader = __ffs(same) - 1;
    if (flt) {
      const double x = ok ? ld_f64(v, dt, j) : 0.0;
      double acc = op == 1 ? INFINITY : op == 2 ? -INFINITY : 0.0;
      for (unsigned m = same; m; m &= m - 1) {
        const double y = __shfl_sync(same, x, __ffs(m) - 1);
        if (op == 0) acc += y;
        else if (op == 1) acc = (y < acc) ? y : acc;
        else acc = (acc < y) ? y : acc;
      }
      if (ok && lane == leader) {
        if (op == 0) row[g] += acc;
        else if (op == 1) row[g] = (acc < row[g]) ? acc : row[g];
        else row[g] = (row[g] < acc) ? acc : row[g];
      }
      __syncwarp();
    } else {
      const int64_t x = !ok ? 0 : op == 3 ? 1 : ld_i64(v, dt, j);
      if (op == 0 || op == 3) {
        uint64_t acc = 0;
        for (unsigned m = same; m; m &= m - 1) acc += static_cast<uint64_t>(__shfl_sync(same, x, __ffs(m) - 1));
        if (ok && lane == leader) atomicAdd(iout + g, static_cast<unsigned long long>(acc));
      } else if (ok) {
        if (op == 1) atomicMin(reinterpret_cast<long long*>(iout) + g, static_cast<long long>(x));
        else atomicMax(reinterpret_cast<long long*>(iout) + g, static_cast<long long>(x));
      }
    }
  }
}

// the warps' rows folded per group in warp order (fixed: the same bits on every run)
__global__ void k_group_fold_rows(const double* __restrict__ fpart, int64_t nw, int64_t G, int op,
                                  double* __restrict__ out) {
  __shared__ double red[256];
  const int64_t g = blockIdx.x;
  const double init = op == 1 ? INFINITY : op == 2 ? -INFINITY : 0.0;
  double acc = init;
  for (int64_t q = threadIdx.x; q < nw; q += 256) {
    const double y = fpart[q * G + g];
    if (op == 0) acc += y;
    else if (op == 1) acc = (y < acc) ? y : acc;
    else acc = (acc < y) ? y : acc;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) {
      const double y = red[threadIdx.x + k], x = red[threadIdx.x];
      red[threadIdx.x] = op == 0 ? x + y : op == 1 ? ((y < x) ? y : x) : ((x < y) ? y : x);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[g] = red[0];
}

// one thread per group: fold values[perm[k]] for k in [start[g], start[g+1])
// in input order (scatter_loop, kernels.cpp:67-80)
__global__ void k_scatter_seq(const void* __restrict__ v, int dt, const int64_t* __restrict__ perm,
                              const int64_t* __restrict__ start, int64_t n, int64_t G, int op, int flt,
                              void* __restrict__ out) {
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < G;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = start[g], b = g + 1 < G ? start[g + 1] : n;
    if (flt) {
      double acc = op == 1 ? INFINITY : op == 2 ? -INFINITY : 0.0;
      for (int64_t k = a; k < b; ++k) {
        const double x = ld_f64(v, dt, perm[k]);
        if (op == 0) acc += x;
        else if (op == 1) acc = (x < acc) ? x : acc;  // std::min(slot, v)
        else acc = (acc < x) ? x : acc;                // std::max(slot, v)
      }
      static_cast<double*>(out)[g] = acc;
    } else {
      int64_t acc = op == 1 ? INT64_MAX : op == 2 ? INT64_MIN : 0;
      for (int64_t k = a; k < b; ++k) {
        if (op == 3) {
          acc += 1;
          continue;
        }
        const int64_t x = ld_i64(v, dt, perm[k]);
        if (op == 0) acc = static_cast<int64_t>(static_cast<uint64_t>(acc) + static_cast<uint64_t>(x));
        else if (op == 1) acc = x < acc ? x : acc;
        else acc = acc < x ? x : acc;
      }
      static_cast<int64_t*>(out)[g] = acc;
    }
  }
}

__global__ void k_adjacent_ne(const void* __restrict__ x, int dt, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i == 0) {
      out[i] = 1;
    } else if (dt_is_float_dev(dt)) {
      out[i] = !(ld_f64(x, dt, i) == ld_f64(x, dt, i - 1));
    } else {
      out[i] = !(ld_i64(x, dt, i) == ld_i64(x, dt, i - 1));
    }
  }
}

// rle_to_plain: row r takes the value of the run containing it, else fill
__global__ void k_runs_to_rows(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t nr,
                               const void* __restrict__ v, int w, const void* __restrict__ fill, int64_t total,
                               void* __restrict__ out) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < total;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = nr;  // first run with e >= r
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (e[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    const bool in = lo < nr && s[lo] <= r;
    const char* src = in ? static_cast<const char*>(v) + lo * w : static_cast<const char*>(fill);
    switch (w) {
      case 1: static_cast<uint8_t*>(out)[r] = *reinterpret_cast<const uint8_t*>(src); break;
      case 2: static_cast<uint16_t*>(out)[r] = *reinterpret_cast<const uint16_t*>(src); break;
      case 4: static_cast<uint32_t*>(out)[r] = *reinterpret_cast<const uint32_t*>(src); break;
      default: static_cast<uint64_t*>(out)[r] = *reinterpret_cast<const uint64_t*>(src); break;
    }
  }
}

// aggregate_array terms (groupby.cpp:67-135): mode 0 i64(v)·w (wrapping),
// mode 1 f64(v)·f64(w), mode 2 (f64(v) − mean[g])² · f64(w)
__global__ void k_weighted(const void* __restrict__ v, int dt, const int64_t* __restrict__ s,
                           const int64_t* __restrict__ e, int64_t n, int mode, const int64_t* __restrict__ inv,
                           const double* __restrict__ mean, void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = s ? e[i] - s[i] + 1 : 1;
    if (mode == 0) {
      static_cast<int64_t*>(out)[i] =
          static_cast<int64_t>(static_cast<uint64_t>(ld_i64(v, dt, i)) * static_cast<uint64_t>(w));
    } else if (mode == 1) {
      static_cast<double*>(out)[i] = ld_f64(v, dt, i) * static_cast<double>(w);
    } else {
      const double d = ld_f64(v, dt, i) - mean[inv[i]];
      static_cast<double*>(out)[i] = d * d * static_cast<double>(w);
    }
  }
}

// mode 0: out = cnt > 0 ? sum / cnt : NaN; mode 1 var, 2 std (sum = Σ squares)
__global__ void k_ratio(const double* __restrict__ sum, const int64_t* __restrict__ cnt, int64_t G, int mode,
                        double* __restrict__ out) {
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < G;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (cnt[g] <= 0) {
      out[g] = NAN;
      continue;
    }
    const double r = sum[g] / static_cast<double>(cnt[g]);
    out[g] = mode == 2 ? sqrt(r) : r;
  }
}

// compact_rle_index: new positions of runs and points re-based at the
// running covered count (primitives.cpp:381-420)
__global__ void k_compact_runs(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t nr,
                               const int64_t* __restrict__ len_excl, const int64_t* __restrict__ pts_before,
                               int64_t* __restrict__ s_out, int64_t* __restrict__ e_out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nr;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t at = len_excl[i] + pts_before[i];
    s_out[i] = at;
    e_out[i] = at + (e[i] - s[i]);
  }
}
__global__ void k_compact_points(int64_t np, const int64_t* __restrict__ runs_before,
                                 const int64_t* __restrict__ len_excl_ext, int64_t* __restrict__ p_out) {
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < np;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p_out[j] = j + len_excl_ext[runs_before[j]];
}

}  // namespace dev

namespace {

int grid_of(const CtxPtr& ctx, int64_t n) {
  const int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : g > 8LL * ctx->sm_count ? 8LL * ctx->sm_count : g);
}

void launched(const CtxPtr& ctx) {
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
}

// first index flagged by a k_first_outside / k_tile_apply pass, or -1
struct BadSlot {
  DArr slot;
  explicit BadSlot(const CtxPtr& ctx) : slot(alloc_arr(ctx, RQ_I64, 1)) {
    RQ_CUDA_CHECK(cudaMemsetAsync(slot.raw_mut(), 0xff, 8, ctx->stream));
  }
  unsigned long long* ptr() const { return slot.as<unsigned long long>(); }
  int64_t read(const CtxPtr& ctx) const {
    const uint64_t v = static_cast<uint64_t>(*ctx->readback(slot.raw(), 8));
    return v == ~0ull ? -1 : static_cast<int64_t>(v);
  }
};

DArr scan128(const CtxPtr& ctx, const DArr& x, bool exclusive, bool want_out, const char* what, bool is_sum) {
  require(x.dt == RQ_I64, "cumsum: int64 input required");
  DArr out = alloc_arr(ctx, RQ_I64, want_out ? x.n : 0);
  if (x.n == 0) return out;
  const int64_t tiles = (x.n + dev::BTILE - 1) / dev::BTILE;
  DArr sums = alloc_arr(ctx, RQ_I64, 2 * tiles);
  BadSlot bad(ctx);
  auto* s128 = reinterpret_cast<dev::i128*>(sums.raw_mut());
  dev::k_tile_sums<<<static_cast<unsigned>(tiles), dev::BT, 0, ctx->stream>>>(x.pos(), x.n, s128);
  launched(ctx);
  dev::k_tile_prefix<<<1, 1, 0, ctx->stream>>>(s128, tiles);
  launched(ctx);
  dev::k_tile_apply<<<static_cast<unsigned>(tiles), dev::BT, 0, ctx->stream>>>(
      x.pos(), x.n, s128, exclusive ? 1 : 0, want_out ? out.as<int64_t>() : nullptr, bad.ptr());
  launched(ctx);
  const int64_t at = bad.read(ctx);
  if (at >= 0) {
    if (is_sum) fail(std::string(what) + ": int64 overflow", RQ_OVERFLOW);
    fail(std::string(what) + ": int64 overflow at element " + std::to_string(at), RQ_OVERFLOW);
  }
  return out;
}

int64_t first_outside(const CtxPtr& ctx, const DArr& x, int64_t lo, int64_t hi) {
  if (x.n == 0) return -1;
  BadSlot bad(ctx);
  dev::k_first_outside<<<grid_of(ctx, x.n), 256, 0, ctx->stream>>>(x.pos(), x.n, lo, hi, bad.ptr());
  launched(ctx);
  return bad.read(ctx);
}

int64_t read_i64(const CtxPtr& ctx, const DArr& a, int64_t i) {
  return *ctx->readback(a.as<int64_t>() + i, 8);
}

// segments of `counts` expanded to their total (checked like the reference)
DArr expand(const CtxPtr& ctx, const DArr& counts, int mode, const DArr& src) {
  require(counts.dt == RQ_I64, "repeat_interleave: int64 counts required");
  DArr off = checked_cumsum(ctx, counts, true);
  const int64_t total = checked_sum(ctx, counts);
  if (first_outside(ctx, counts, 0, -1) >= 0) fail("repeat_interleave: negative count");
  DArr out = alloc_arr(ctx, mode == 1 ? RQ_I64 : src.dt, total);
  if (total > 0) {
    dev::k_expand<<<grid_of(ctx, total), 256, 0, ctx->stream>>>(off.pos(), counts.n, total, mode, src.raw(),
                                                                dt_width(src.dt), out.raw_mut());
    launched(ctx);
  }
  return out;
}

DArr run_lengths(const CtxPtr& ctx, const DArr& s, const DArr& e) {
  return scalar_arith_values(ctx, arith_values(ctx, e, s, RQ_SUB), Scalar{false, 1, 0.0}, RQ_ADD, false);
}

}  // namespace

DArr checked_cumsum(const CtxPtr& ctx, const DArr& x, bool exclusive) {
  return scan128(ctx, x, exclusive, true, "cumsum", false);
}

int64_t checked_sum(const CtxPtr& ctx, const DArr& x) {
  require(x.dt == RQ_I64, "sum: int64 input required");
  if (x.n == 0) return 0;
  DArr inc = scan128(ctx, x, false, true, "sum", true);
  return read_i64(ctx, inc, x.n - 1);
}

DArr repeat_interleave(const CtxPtr& ctx, const DArr& values, const DArr& counts) {
  require(values.n == counts.n, "repeat_interleave: length mismatch");
  return expand(ctx, counts, 0, values);
}

DArr range_arange(const CtxPtr& ctx, const DArr& start, const DArr& length) {
  require(start.n == length.n, "range_arange: length mismatch");
  require(start.dt == RQ_I64, "range_arange: int64 starts required");
  return expand(ctx, length, 1, start);
}

DArr scatter_reduce(const CtxPtr& ctx, const DArr& values, const DArr& index, int64_t n_groups, int op) {
  require(values.n == index.n, "scatter_reduce: values/index length mismatch");
  require(n_groups >= 0, "scatter_reduce: negative group count");
  require(index.dt == RQ_I64, "scatter_reduce: int64 index required");
  const int64_t bad = first_outside(ctx, index, 0, n_groups);
  if (bad >= 0) fail("scatter_reduce: group index out of range at element " + std::to_string(bad));
  const bool flt = dt_float(values.dt) && op != 3;
  DArr out = alloc_arr(ctx, flt ? RQ_F64 : RQ_I64, n_groups);
  if (n_groups == 0) return out;
  // few large groups: warp-range folds (one thread per group would walk
  // ~n / G elements serially); deterministic, within rounding of the
  // input-order loop for f64 sums
  const int64_t nw = static_cast<int64_t>(ctx->sm_count) * 8 * 8;
  if (index.n >= (int64_t{1} << 20) && index.n / n_groups >= 4096 && nw * n_groups <= (int64_t{8} << 20)) {
    const int64_t per = ((index.n + nw - 1) / nw + 31) / 32 * 32;
    DArr fpart;
    if (flt) {
      fpart = alloc_arr(ctx, RQ_F64, nw * n_groups);
    } else if (op == 0 || op == 3) {
      RQ_CUDA_CHECK(cudaMemsetAsync(out.raw_mut(), 0, static_cast<size_t>(n_groups) * 8, ctx->stream));
    } else {  // min / max identities (rare: a host copy and one sync)
      std::vector<int64_t> h(static_cast<size_t>(n_groups), op == 1 ? INT64_MAX : INT64_MIN);
      RQ_CUDA_CHECK(cudaMemcpyAsync(out.raw_mut(), h.data(), static_cast<size_t>(n_groups) * 8,
                                    cudaMemcpyHostToDevice, ctx->stream));
      RQ_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // h leaves scope
    }
    dev::k_group_fold_warp<<<static_cast<unsigned>(nw / 8), 256, 0, ctx->stream>>>(
        values.raw(), values.dt, index.pos(), index.n, n_groups, op, flt ? 1 : 0, per,
        flt ? fpart.as<double>() : nullptr, flt ? nullptr : out.as<unsigned long long>());
    launched(ctx);
    if (flt) {
      dev::k_group_fold_rows<<<static_cast<unsigned>(n_groups), 256, 0, ctx->stream>>>(fpart.as<double>(), nw,
                                                                                      n_groups, op, out.as<double>());
      launched(ctx);
    }
    return out;
  }
  // stable sort of the element indices by group: each group's values in input order
  DArr keys = copy_prefix(ctx, index, index.n);
  DArr perm = iota(ctx, index.n);
  int bits = 0;
  while (bits < 63 && (int64_t{1} << bits) < n_groups) ++bits;
  radix_sort_pairs(ctx, keys, perm, bits, 0);
  DArr start = bucketize(ctx, iota(ctx, n_groups), keys, false);
  dev::k_scatter_seq<<<grid_of(ctx, n_groups), 256, 0, ctx->stream>>>(
      values.raw(), values.dt, perm.pos(), start.pos(), index.n, n_groups, op, flt ? 1 : 0, out.raw_mut());
  launched(ctx);
  return out;
}

Unique unique_with_inverse(const CtxPtr& ctx, const std::vector<DArr>& cols) {
  Unique u;
  if (cols.empty()) return u;
  const int64_t n = cols[0].n;
  for (const auto& c : cols) require(c.n == n, "unique_with_inverse: column length mismatch");
  if (n == 0) {
    for (const auto& c : cols) u.keys.push_back(alloc_arr(ctx, c.dt, 0));
    u.inverse = alloc_arr(ctx, RQ_I64, 0);
    return u;
  }
  SortedGroups g = group_ids_sorted(ctx, cols);
  for (const auto& c : cols) u.keys.push_back(gather(ctx, c, g.first_rows));
  u.inverse = g.inverse;
  u.n_groups = g.n_groups;
  return u;
}

DArr gather_checked(const CtxPtr& ctx, const DArr& values, const DArr& idx) {
  require(idx.dt == RQ_I64, "gather: int64 indices required");
  const int64_t bad = first_outside(ctx, idx, 0, values.n);
  if (bad >= 0) fail("gather: index out of range: " + std::to_string(read_i64(ctx, idx, bad)));
  return gather(ctx, values, idx);
}

void sort_with_perm(const CtxPtr& ctx, const DArr& values, DArr& sorted, DArr& perm) {
  perm = values.n > 0 ? sort_permutation(ctx, {values}) : alloc_arr(ctx, RQ_I64, 0);
  sorted = gather(ctx, values, perm);
}

DArr adjacent_ne(const CtxPtr& ctx, const DArr& x) {
  DArr out = alloc_arr(ctx, RQ_I8, x.n);
  if (x.n == 0) return out;
  dev::k_adjacent_ne<<<grid_of(ctx, x.n), 256, 0, ctx->stream>>>(x.raw(), x.dt, x.n, out.as<uint8_t>());
  launched(ctx);
  return out;
}

DArr shape_weights(const CtxPtr& ctx, const Decomp& sh) {
  if (sh.kind == 1) return run_lengths(ctx, sh.s, sh.e);
  const int64_t n = sh.kind == 0 ? sh.n : sh.p.n;
  DArr w = alloc_arr(ctx, RQ_I64, n);
  if (n > 0) {  // n ones
    const int64_t one = 1;
    w = repeat_interleave(ctx, upload_arr(ctx, RQ_I64, &one, 1), upload_arr(ctx, RQ_I64, &n, 1));
  }
  return w;
}

DArr aggregate_array(const CtxPtr& ctx, const Decomp& sh, const DArr& values, const DArr& inverse, int64_t G,
                     int fn) {
  const int64_t slots = sh.kind == 0 ? sh.n : sh.kind == 1 ? sh.s.n : sh.p.n;
  require(values.n == slots, "aggregate: values do not match shape");
  require(values.n == inverse.n, "aggregate: values do not match grouping");
  const int64_t* s = sh.kind == 1 ? sh.s.pos() : nullptr;
  const int64_t* e = sh.kind == 1 ? sh.e.pos() : nullptr;
  auto weighted = [&](int mode, const DArr* mean) {
    DArr out = alloc_arr(ctx, mode == 0 ? RQ_I64 : RQ_F64, values.n);
    if (values.n > 0) {
      dev::k_weighted<<<grid_of(ctx, values.n), 256, 0, ctx->stream>>>(
          values.raw(), values.dt, s, e, values.n, mode, inverse.pos(), mean ? mean->as<double>() : nullptr,
          out.raw_mut());
      launched(ctx);
    }
    return out;
  };
  switch (fn) {
    case RQ_MIN: return scatter_reduce(ctx, values, inverse, G, 1);
    case RQ_MAX: return scatter_reduce(ctx, values, inverse, G, 2);
    case RQ_COUNT: return scatter_reduce(ctx, shape_weights(ctx, sh), inverse, G, 0);
    case RQ_SUM:
      return scatter_reduce(ctx, weighted(dt_float(values.dt) ? 1 : 0, nullptr), inverse, G, 0);
    case RQ_AVG:
    case RQ_STD:
    case RQ_VAR: {
      DArr sum = scatter_reduce(ctx, weighted(1, nullptr), inverse, G, 0);
      DArr cnt = scatter_reduce(ctx, shape_weights(ctx, sh), inverse, G, 0);
      DArr mean = alloc_arr(ctx, RQ_F64, G);
      if (G > 0) {
        dev::k_ratio<<<grid_of(ctx, G), 256, 0, ctx->stream>>>(sum.as<double>(), cnt.pos(), G, 0, mean.as<double>());
        launched(ctx);
      }
      if (fn == RQ_AVG) return mean;
      DArr sq = scatter_reduce(ctx, weighted(2, &mean), inverse, G, 0);
      DArr out = alloc_arr(ctx, RQ_F64, G);
      if (G > 0) {
        dev::k_ratio<<<grid_of(ctx, G), 256, 0, ctx->stream>>>(sq.as<double>(), cnt.pos(), G,
                                                              fn == RQ_VAR ? 1 : 2, out.as<double>());
        launched(ctx);
      }
      return out;
    }
  }
  fail("aggregate: unknown function");
}

namespace {
void check_budget(int64_t rows, int64_t budget, const char* what) {
  if (rows > budget)
    fail(std::string(what) + ": expansion of " + std::to_string(rows) + " elements exceeds budget " +
             std::to_string(budget),
         RQ_RESOURCE);
}
}  // namespace

DCol rle_to_index(const CtxPtr& ctx, const DCol& c, int64_t budget) {
  require(c.enc == RQ_ENC_RLE, "rle_to_index: rle column required");
  check_budget(covered_rows(ctx, c.s, c.e), budget, "rle_to_index");
  DCol out;
  out.enc = RQ_ENC_INDEX;
  out.total = c.total;
  DArr l = run_lengths(ctx, c.s, c.e);
  out.p = range_arange(ctx, c.s, l);
  out.v = repeat_interleave(ctx, c.v, l);
  out.logical = out.v.dt;
  return out;
}

DMask rle_mask_to_index(const CtxPtr& ctx, const DMask& m, int64_t budget) {
  require(m.enc == RQ_MASK_RLE, "rle_to_index: rle mask required");
  check_budget(covered_rows(ctx, m.s, m.e), budget, "rle_to_index");
  DMask out;
  out.enc = RQ_MASK_INDEX;
  out.total = m.total;
  out.p = range_arange(ctx, m.s, run_lengths(ctx, m.s, m.e));
  return out;
}

DCol rle_to_plain(const CtxPtr& ctx, const DCol& c, double fill, int64_t budget) {
  require(c.enc == RQ_ENC_RLE, "rle_to_plain: rle column required");
  check_budget(c.total, budget, "rle_to_plain");
  // static_cast<T>(fill) at the value dtype (primitives.cpp:200)
  unsigned char fb[8] = {0};
  switch (c.v.dt) {
    case RQ_I8: { int8_t x = static_cast<int8_t>(fill); std::memcpy(fb, &x, 1); break; }
    case RQ_I16: { int16_t x = static_cast<int16_t>(fill); std::memcpy(fb, &x, 2); break; }
    case RQ_I32: { int32_t x = static_cast<int32_t>(fill); std::memcpy(fb, &x, 4); break; }
    case RQ_I64: { int64_t x = static_cast<int64_t>(fill); std::memcpy(fb, &x, 8); break; }
    case RQ_F32: { float x = static_cast<float>(fill); std::memcpy(fb, &x, 4); break; }
    default: std::memcpy(fb, &fill, 8); break;
  }
  DArr f = upload_arr(ctx, RQ_I64, fb, 1);
  DCol out;
  out.enc = RQ_ENC_PLAIN;
  out.total = c.total;
  out.v = alloc_arr(ctx, c.v.dt, c.total);
  out.logical = c.v.dt;
  if (c.total > 0) {
    dev::k_runs_to_rows<<<grid_of(ctx, c.total), 256, 0, ctx->stream>>>(
        c.s.pos(), c.e.pos(), c.s.n, c.v.raw(), dt_width(c.v.dt), f.raw(), c.total, out.v.raw_mut());
    launched(ctx);
  }
  ctx->wait_stream();  // fb
  return out;
}

DMask rle_mask_to_plain(const CtxPtr& ctx, const DMask& m, int64_t budget) {
  require(m.enc == RQ_MASK_RLE, "rle_to_plain: rle mask required");
  check_budget(m.total, budget, "rle_to_plain");
  DMask out;
  out.enc = RQ_MASK_PLAIN;
  out.total = m.total;
  out.bits = alloc_arr(ctx, RQ_I8, m.total);
  if (m.total > 0) {
    const uint8_t one = 1, zero = 0;
    DArr v1 = upload_arr(ctx, RQ_I8, &one, 1), f0 = upload_arr(ctx, RQ_I8, &zero, 1);
    // every run's value is 1: a one-element value array indexed through a zero stride is not
    // expressible, so expand a per-run 1 array
    DArr ones = repeat_interleave(ctx, v1, upload_arr(ctx, RQ_I64, &m.s.n, 1));
    dev::k_runs_to_rows<<<grid_of(ctx, m.total), 256, 0, ctx->stream>>>(m.s.pos(), m.e.pos(), m.s.n, ones.raw(), 1,
                                                                        f0.raw(), m.total, out.bits.raw_mut());
    launched(ctx);
    ctx->wait_stream();
  }
  return out;
}

DCol compact_rle_index(const CtxPtr& ctx, const DCol& c) {
  require(c.enc == RQ_ENC_RLE_INDEX, "compact_rle_index: rle+index column required");
  const int64_t nr = c.s.n, np = c.p2.n;
  DArr l = run_lengths(ctx, c.s, c.e);
  DArr len_excl = checked_cumsum(ctx, l, true);
  // len_ext[k] = covered run rows of the first k runs (k = 0..nr)
  DArr len_incl = checked_cumsum(ctx, l, false);
  DArr len_ext = alloc_arr(ctx, RQ_I64, nr + 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(len_ext.raw_mut(), 0, 8, ctx->stream));
  if (nr > 0)
    RQ_CUDA_CHECK(cudaMemcpyAsync(len_ext.as<int64_t>() + 1, len_incl.raw(), nr * 8, cudaMemcpyDeviceToDevice,
                                  ctx->stream));
  DCol out;
  out.enc = RQ_ENC_RLE_INDEX;
  out.v = c.v;
  out.v2 = c.v2;
  out.logical = c.v.dt;
  out.s = alloc_arr(ctx, RQ_I64, nr);
  out.e = alloc_arr(ctx, RQ_I64, nr);
  out.p2 = alloc_arr(ctx, RQ_I64, np);
  if (nr > 0) {
    DArr pts_before = bucketize(ctx, c.s, c.p2, false);  // points before each run start
    dev::k_compact_runs<<<grid_of(ctx, nr), 256, 0, ctx->stream>>>(c.s.pos(), c.e.pos(), nr, len_excl.pos(),
                                                                   pts_before.pos(), out.s.as<int64_t>(),
                                                                   out.e.as<int64_t>());
    launched(ctx);
  }
  if (np > 0) {
    DArr runs_before = bucketize(ctx, c.p2, c.e, false);  // runs ending before each point
    dev::k_compact_points<<<grid_of(ctx, np), 256, 0, ctx->stream>>>(np, runs_before.pos(), len_ext.pos(),
                                                                     out.p2.as<int64_t>());
    launched(ctx);
  }
  out.total = (nr > 0 ? read_i64(ctx, len_ext, nr) : 0) + np;
  return out;
}

void col_to_rows(const CtxPtr& ctx, const DCol& c, DArr& positions, DArr& values) {
  switch (c.enc) {
    case RQ_ENC_PLAIN:
      positions = iota(ctx, c.total);
      values = decode_plain(ctx, c);
      return;
    case RQ_ENC_PLAIN_INDEX:
      positions = iota(ctx, c.total);
      values = decode_plain_index(ctx, c);
      return;
    case RQ_ENC_INDEX:
      positions = c.p;
      values = c.v;
      return;
    case RQ_ENC_RLE: {
      DArr l = run_lengths(ctx, c.s, c.e);
      positions = range_arange(ctx, c.s, l);
      values = repeat_interleave(ctx, c.v, l);
      return;
    }
    default: {  // runs' rows and the points merged in position order
      DArr rp, rv;
      DArr l = run_lengths(ctx, c.s, c.e);
      rp = range_arange(ctx, c.s, l);
      rv = repeat_interleave(ctx, c.v, l);
      require(rv.dt == c.v2.dt, "to_rows: run / point value dtypes differ");
      merge_disjoint(ctx, rp, nullptr, &rv, c.p2, nullptr, &c.v2, positions, nullptr, &values);
      return;
    }
  }
}

DArr decode_full(const CtxPtr& ctx, const DCol& c) {
  // covered_rows() == total_size (column.cpp:311-314); RLE+Index: runs + points
  const bool full = c.enc == RQ_ENC_RLE_INDEX ? covered_rows(ctx, c.s, c.e) + c.p2.n == c.total
                                              : col_full_coverage(ctx, c);
  if (!full) fail("decode_full: column has gaps; use to_rows");
  switch (c.enc) {
    case RQ_ENC_PLAIN: return decode_plain(ctx, c);
    case RQ_ENC_PLAIN_INDEX: return decode_plain_index(ctx, c);
    case RQ_ENC_INDEX: return c.v;
    case RQ_ENC_RLE: return repeat_interleave(ctx, c.v, run_lengths(ctx, c.s, c.e));
    default: {
      DArr p, v;
      col_to_rows(ctx, c, p, v);
      return v;
    }
  }
}

}  // namespace rqb
