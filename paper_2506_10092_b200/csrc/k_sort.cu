// k_sort.cu — K11: sort-based grouping for keys the dense-slot path cannot
// take (floating-point keys, or integer keys whose joint range exceeds the
// slot table). Restates kernels::unique_with_inverse (kernels.cpp:127-187):
// group ids in ascending lexicographic key order, the group's key taken from
// its FIRST row in a stable sort (the smallest slot index among equal keys),
// floats compared with `<` after f32→f64 widening (so −0.0 and +0.0 group
// together; the reference's NaN ordering is not a strict weak order and NaN
// keys are left undefined there as here).
//
// Keys are mapped to order-preserving unsigned 64-bit words (ints: x − min;
// floats: sign-flipped IEEE bits), packed into ONE word when the per-column
// significant bits fit in 64, otherwise sorted column by column (LSD over
// columns, stable) carrying the permutation. The sort is a hand-written
// stable LSD radix sort, 8-bit digits, only over the significant bits:
//   k_rs_hist    per-tile digit histograms (smem atomics), digit-major
//   k_scan_i64   exclusive scan of the histograms (decoupled look-back)
//   k_rs_scatter stable in-tile ranking with __match_any_sync + per-warp
//                digit counters, scatter of (key, row) pairs
#include "device_common.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

constexpr int RS_BLOCK = 256;
constexpr int RS_ROUNDS = 16;                      // items per thread
constexpr int RS_TILE = RS_BLOCK * RS_ROUNDS;      // 4096 keys per tile
constexpr int RS_WARPS = RS_BLOCK / 32;

__device__ __forceinline__ uint32_t rs_digit(uint64_t k, uint64_t sub, int shift) {
  return static_cast<uint32_t>(((k - sub) >> shift) & 0xff);
}

__global__ void __launch_bounds__(RS_BLOCK)
    k_rs_hist(const uint64_t* __restrict__ keys, int64_t n, uint64_t sub, int shift, int64_t tiles,
              int64_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
#pragma unroll 4
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int64_t i = base + r * RS_BLOCK + threadIdx.x;
    if (i < n) atomicAdd(&h[rs_digit(keys[i], sub, shift)], 1u);
  }
  __syncthreads();
  hist[static_cast<int64_t>(threadIdx.x) * tiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of an int64 array (in -> out), blocked ITEMS per thread
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK)
    k_scan_i64(const int64_t* __restrict__ in, int64_t n, LookBack lb, int64_t* __restrict__ out) {
  __shared__ uint64_t wt[BLOCK / 32 + 1];
  __shared__ uint64_t tile_base;
  const int64_t base = (static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x) * ITEMS;
  uint64_t x[ITEMS];
  uint64_t sum = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t i = base + k;
    x[k] = i < n ? static_cast<uint64_t>(ldg64(in, i)) : 0;
    sum += x[k];
  }
  uint64_t total;
  uint64_t off = block_exclusive<BLOCK>(sum, total, wt);
  if (threadIdx.x < 32) {
    const uint64_t b = lb.exclusive(blockIdx.x, total);
    if (threadIdx.x == 0) tile_base = b;
  }
  __syncthreads();
  off += tile_base;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int64_t i = base + k;
    if (i < n) out[i] = static_cast<int64_t>(off);
    off += x[k];
  }
}

// Stable scatter of one digit pass. Items are visited in index order
// (round, warp, lane); within a warp equal digits are ranked by lane with
// __match_any_sync, across warps by a per-round column scan of the warps'
// digit counts, across rounds by a running per-digit counter.
__global__ void __launch_bounds__(RS_BLOCK)
    k_rs_scatter(const uint64_t* __restrict__ keys, const int64_t* __restrict__ vals, int64_t n,
                 uint64_t sub, int shift, int64_t tiles, const int64_t* __restrict__ offs,
                 uint64_t* __restrict__ keys_out, int64_t* __restrict__ vals_out) {
  __shared__ uint32_t cnt[RS_WARPS][256];
  __shared__ uint32_t pre[RS_WARPS][256];
  __shared__ int64_t run[256];
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  run[t] = offs[static_cast<int64_t>(t) * tiles + blockIdx.x];
#pragma unroll
  for (int k = 0; k < RS_WARPS; ++k) cnt[k][t] = 0;
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int64_t i = base + r * RS_BLOCK + t;
    const bool ok = i < n;
    uint64_t key = 0;
    int64_t val = 0;
    uint32_t d = 256u + lane;  // unique per lane when out of range
    if (ok) {
      key = keys[i];
      val = vals[i];
      d = rs_digit(key, sub, shift);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lt);
    if (ok && rank == 0) cnt[w][d] = __popc(peers);
    __syncthreads();
    {  // column t: prefix over warps, reset counts, advance the running base
      uint32_t s = 0;
#pragma unroll
      for (int k = 0; k < RS_WARPS; ++k) {
        const uint32_t c = cnt[k][t];
        cnt[k][t] = 0;
        pre[k][t] = s;
        s += c;
      }
      __syncthreads();
      if (ok) {
        const int64_t pos = run[d] + pre[w][d] + rank;
        keys_out[pos] = key;
        vals_out[pos] = val;
      }
      __syncthreads();
      run[t] += s;
    }
  }
}

// order-preserving u64 image of a key column (optionally through perm);
// also folds the min / max image into mm[0..1]
__device__ __forceinline__ uint64_t key_image(const void* v, int dt, int64_t i) {
  if (dt_is_float_dev(dt)) {
    double x = ld_f64(v, dt, i);
    if (x == 0.0) x = 0.0;  // −0.0 == +0.0 under `<`
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
    return (u >> 63) ? ~u : (u | (1ull << 63));
  }
  return static_cast<uint64_t>(ld_i64(v, dt, i)) ^ (1ull << 63);
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_key_images(const void* __restrict__ v, int dt, const int64_t* __restrict__ perm, int64_t n,
                 uint64_t* __restrict__ out, unsigned long long* __restrict__ mm) {
  uint64_t mn = ~0ull, mx = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * BLOCK) {
    const uint64_t u = key_image(v, dt, perm ? ldg64(perm, i) : i);
    if (out) out[i] = u;
    mn = u < mn ? u : mn;
    mx = u > mx ? u : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, static_cast<unsigned long long>(mn));
    atomicMax(mm + 1, static_cast<unsigned long long>(mx));
  }
}

struct PackSpec {
  const void* v[8];
  int dt[8];
  uint64_t mn[8];
  int shift[8];
  int nk;
};

__global__ void k_pack_keys(PackSpec ps, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t k = 0;
    for (int c = 0; c < ps.nk; ++c) k |= (key_image(ps.v[c], ps.dt[c], i) - ps.mn[c]) << ps.shift[c];
    out[i] = k;
  }
}

// flags[i] = 1 where sorted row i starts a new group (composite key differs)
__global__ void k_group_bounds(PackSpec ps, const int64_t* __restrict__ perm, int64_t n,
                               int64_t* __restrict__ flags, uint8_t* __restrict__ bytes) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int f = 1;
    if (i > 0) {
      const int64_t a = ldg64(perm, i - 1), b = ldg64(perm, i);
      f = 0;
      for (int c = 0; c < ps.nk && !f; ++c)
        f = key_image(ps.v[c], ps.dt[c], a) != key_image(ps.v[c], ps.dt[c], b);
    }
    flags[i] = f;
    bytes[i] = static_cast<uint8_t>(f);
  }
}

// inverse[perm[i]] = (exclusive group count before i) + flag[i] − 1
__global__ void k_group_inverse(const int64_t* __restrict__ perm, const int64_t* __restrict__ excl,
                                const int64_t* __restrict__ flags, int64_t n, int64_t* __restrict__ inv) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    inv[ldg64(perm, i)] = ldg64(excl, i) + ldg64(flags, i) - 1;
}

}  // namespace dev

namespace {

int grid_for(const CtxPtr& ctx, int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

void launched(const CtxPtr& ctx) {
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
}

int sig_bits(uint64_t range) { return range == 0 ? 0 : 64 - __builtin_clzll(range); }

// min / max key image of one column (optionally through perm)
void key_minmax(const CtxPtr& ctx, const DArr& v, uint64_t& mn, uint64_t& mx) {
  DArr mm = alloc_arr(ctx, RQ_I64, 2);
  const uint64_t init[2] = {~0ull, 0};
  RQ_CUDA_CHECK(cudaMemcpyAsync(mm.raw_mut(), init, 16, cudaMemcpyHostToDevice, ctx->stream));
  dev::k_key_images<256><<<grid_for(ctx, v.n), 256, 0, ctx->stream>>>(
      v.raw(), v.dt, nullptr, v.n, nullptr, reinterpret_cast<unsigned long long*>(mm.raw_mut()));
  launched(ctx);
  const uint64_t* h = reinterpret_cast<const uint64_t*>(ctx->readback(mm.raw(), 16));
  mn = h[0];
  mx = h[1];
}

}  // namespace

void scan_exclusive_i64(const CtxPtr& ctx, const DArr& in, DArr& out) {
  constexpr int B = 256, IT = 8;
  out = alloc_arr(ctx, RQ_I64, in.n);
  if (in.n == 0) return;
  const int64_t ntiles = (in.n + B * IT - 1) / (B * IT);
  dev::LookBack lb{nullptr, 0};
  lb.status = ctx->lookback_status(ntiles, &lb.epoch);
  dev::k_scan_i64<B, IT><<<static_cast<unsigned>(ntiles), B, 0, ctx->stream>>>(in.pos(), in.n, lb,
                                                                             out.as<int64_t>());
  launched(ctx);
}

// Stable LSD radix sort of (keys, vals) on bits [0, bits) of (key − sub).
// keys are u64 stored in an I64 DArr. Returns sorted copies.
void radix_sort_pairs(const CtxPtr& ctx, DArr& keys, DArr& vals, int bits, uint64_t sub) {
  const int64_t n = keys.n;
  if (n <= 1 || bits <= 0) return;
  const int64_t tiles = (n + dev::RS_TILE - 1) / dev::RS_TILE;
  DArr hist = alloc_arr(ctx, RQ_I64, tiles * 256);
  DArr k2 = alloc_arr(ctx, RQ_I64, n), v2 = alloc_arr(ctx, RQ_I64, n);
  for (int shift = 0; shift < bits; shift += 8) {
    dev::k_rs_hist<<<static_cast<unsigned>(tiles), dev::RS_BLOCK, 0, ctx->stream>>>(
        keys.as<uint64_t>(), n, sub, shift, tiles, hist.as<int64_t>());
    launched(ctx);
    DArr offs;
    scan_exclusive_i64(ctx, hist, offs);
    dev::k_rs_scatter<<<static_cast<unsigned>(tiles), dev::RS_BLOCK, 0, ctx->stream>>>(
        keys.as<uint64_t>(), vals.pos(), n, sub, shift, tiles, offs.pos(), k2.as<uint64_t>(),
        v2.as<int64_t>());
    launched(ctx);
    std::swap(keys, k2);
    std::swap(vals, v2);
  }
}

namespace {

struct SortPlan {
  dev::PackSpec ps{};
  std::vector<uint64_t> mn;
  std::vector<int> bits;
};

// stable lexicographic permutation of rows by the key columns
DArr sort_perm_impl(const CtxPtr& ctx, const std::vector<DArr>& keyvals, SortPlan& sp) {
  const int nk = static_cast<int>(keyvals.size());
  require(nk >= 1 && nk <= 8, "sort: 1..8 key columns");
  const int64_t n = keyvals[0].n;
  for (const auto& k : keyvals) require(k.n == n, "sort: key column length mismatch");
  sp.ps.nk = nk;
  sp.mn.assign(nk, 0);
  sp.bits.assign(nk, 0);
  DArr perm = iota(ctx, n);
  if (n <= 1) return perm;
  int total_bits = 0;
  for (int c = 0; c < nk; ++c) {
    uint64_t lo, hi;
    key_minmax(ctx, keyvals[c], lo, hi);
    sp.mn[c] = lo;
    sp.bits[c] = sig_bits(hi - lo);
    total_bits += sp.bits[c];
    sp.ps.v[c] = keyvals[c].raw();
    sp.ps.dt[c] = keyvals[c].dt;
    sp.ps.mn[c] = lo;
  }
  if (total_bits <= 64) {
    // one packed word, most significant field = first key column
    int at = 0;
    for (int c = nk; c-- > 0;) {
      sp.ps.shift[c] = at;
      at += sp.bits[c];
    }
    DArr packed = alloc_arr(ctx, RQ_I64, n);
    dev::k_pack_keys<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(sp.ps, n, packed.as<uint64_t>());
    launched(ctx);
    radix_sort_pairs(ctx, packed, perm, total_bits, 0);
  } else {
    // LSD over columns: stable sort by the last column first
    for (int c = nk; c-- > 0;) {
      if (sp.bits[c] == 0) continue;
      DArr img = alloc_arr(ctx, RQ_I64, n);
      DArr mm = alloc_arr(ctx, RQ_I64, 2);
      const uint64_t init[2] = {~0ull, 0};
      RQ_CUDA_CHECK(cudaMemcpyAsync(mm.raw_mut(), init, 16, cudaMemcpyHostToDevice, ctx->stream));
      dev::k_key_images<256><<<grid_for(ctx, n), 256, 0, ctx->stream>>>(
          keyvals[c].raw(), keyvals[c].dt, perm.pos(), n, img.as<uint64_t>(),
          reinterpret_cast<unsigned long long*>(mm.raw_mut()));
      launched(ctx);
      radix_sort_pairs(ctx, img, perm, sp.bits[c], sp.mn[c]);
    }
  }
  return perm;
}

}  // namespace

DArr sort_permutation(const CtxPtr& ctx, const std::vector<DArr>& keyvals) {
  SortPlan sp;
  return sort_perm_impl(ctx, keyvals, sp);
}

SortedGroups group_ids_sorted(const CtxPtr& ctx, const std::vector<DArr>& keyvals) {
  const int64_t n = keyvals.empty() ? 0 : keyvals[0].n;
  SortedGroups g;
  g.inverse = alloc_arr(ctx, RQ_I64, n);
  if (n == 0) {
    g.first_rows = alloc_arr(ctx, RQ_I64, 0);
    return g;
  }
  SortPlan sp;
  DArr perm = sort_perm_impl(ctx, keyvals, sp);
  const dev::PackSpec& ps = sp.ps;
  DArr flags = alloc_arr(ctx, RQ_I64, n), fbytes = alloc_arr(ctx, RQ_I8, n);
  dev::k_group_bounds<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(ps, perm.pos(), n, flags.as<int64_t>(),
                                                                 fbytes.as<uint8_t>());
  launched(ctx);
  DArr excl;
  scan_exclusive_i64(ctx, flags, excl);
  dev::k_group_inverse<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(perm.pos(), excl.pos(), flags.pos(), n,
                                                                  g.inverse.as<int64_t>());
  launched(ctx);
  select_points(ctx, fbytes, perm, g.first_rows, nullptr);
  g.n_groups = g.first_rows.n;
  return g;
}

}  // namespace rqb
