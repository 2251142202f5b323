// k_encode.cu — device-side encoders (the step
// before the path, today host code in the reference).
//
//   enc::plain_to_rle        (primitives.cpp:223-250)
//   enc::plain_to_rle_index  (primitives.cpp:252-279)
//
// Run boundaries are where the STORAGE value changes (adjacent_ne on the
// stored array, kernels.cpp:235-244 — before decoding, so two stored values
// that decode equal still start separate runs, as in the reference); run
// values are the decoded values (logical dtype, centre added). Boundaries are
// compacted with the ordered warp-ballot select kernel (k_select.cu).
#include "device_common.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

// flag[i] = (i == 0) || !(v[i] == v[i-1]) over the raw storage
template <class S>
__global__ void k_adjacent_ne(const S* __restrict__ v, int64_t n, uint8_t* __restrict__ flag) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flag[i] = (i == 0 || !(v[i] == v[i - 1])) ? 1 : 0;
}

// e[k] = s[k + 1] − 1, last = n − 1
__global__ void k_ends_from_starts(const int64_t* __restrict__ s, int64_t k, int64_t n,
                                   int64_t* __restrict__ e) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < k;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    e[i] = i + 1 < k ? ldg64(s, i + 1) - 1 : n - 1;
}

// flag[i] = run length >= min_run (long) or < min_run (short, inverted)
__global__ void k_run_len_flags(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t n,
                                int64_t min_run, int want_long, uint8_t* __restrict__ flag) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool lng = ldg64(e, i) - ldg64(s, i) + 1 >= min_run;
    flag[i] = (lng == (want_long != 0)) ? 1 : 0;
  }
}

// storage + centre in int64 (values.to_i64() then `x += center`, no wrap at
// the logical width — primitives.cpp:305-307, ingest.cpp:201-203)
__global__ void k_decode_unwrapped(const void* __restrict__ v, int dt, int64_t n, int has_center,
                                   int64_t center, int64_t* __restrict__ out,
                                   long long* __restrict__ mm) {
  int64_t mn = INT64_MAX, mx = INT64_MIN;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t x = ld_i64(v, dt, i);
    if (has_center) x = static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(center));
    out[i] = x;
    mn = x < mn ? x : mn;
    mx = x > mx ? x : mx;
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, static_cast<long long>(mn));
    atomicMax(mm + 1, static_cast<long long>(mx));
  }
}

// radix select histogram: for each of two targets, digits (8 bits at
// `shift`) of the values whose higher bits equal that target's prefix
__global__ void k_rsel_hist(const int64_t* __restrict__ x, int64_t n, int64_t sub, int shift,
                            uint64_t pre0, uint64_t pre1, int have_prefix,
                            unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[2][256];
  h[0][threadIdx.x] = 0;
  h[1][threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t u = static_cast<uint64_t>(x[i]) - static_cast<uint64_t>(sub);
    const uint64_t hi = shift + 8 >= 64 ? 0 : (u >> (shift + 8));
    const unsigned d = static_cast<unsigned>((u >> shift) & 0xff);
    if (!have_prefix || hi == pre0) atomicAdd(&h[0][d], 1u);
    if (!have_prefix || hi == pre1) atomicAdd(&h[1][d], 1u);
  }
  __syncthreads();
  if (h[0][threadIdx.x]) atomicAdd(hist + threadIdx.x, h[0][threadIdx.x]);
  if (h[1][threadIdx.x]) atomicAdd(hist + 256 + threadIdx.x, h[1][threadIdx.x]);
}

// trimmed split: outlier iff x outside [lo_t, hi_t]; base = x − centre
template <class N>
__global__ void k_split_base(const int64_t* __restrict__ x, int64_t n, int64_t lo_t, int64_t hi_t,
                             int64_t center, N* __restrict__ base, uint8_t* __restrict__ flag) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = x[i];
    const bool out = v < lo_t || v > hi_t;
    flag[i] = out ? 1 : 0;
    base[i] = out ? N(0) : static_cast<N>(static_cast<uint64_t>(v) - static_cast<uint64_t>(center));
  }
}

// plain-centered encode: (x − centre) cast to the storage width (wraps)
template <class N>
__global__ void k_center_cast(const int64_t* __restrict__ x, int64_t n, int64_t center, N* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<N>(static_cast<uint64_t>(x[i]) - static_cast<uint64_t>(center));
}

// run profile over (s, e): unit runs, long runs, rows in long runs
__global__ void k_run_profile(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t r,
                              int64_t min_run, unsigned long long* __restrict__ out) {
  unsigned long long unit = 0, lng = 0, rows = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < r;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t len = ldg64(e, i) - ldg64(s, i) + 1;
    unit += len == 1;
    if (len >= min_run) {
      ++lng;
      rows += static_cast<unsigned long long>(len);
    }
  }
  unit = warp_sum(unit);
  lng = warp_sum(lng);
  rows = warp_sum(rows);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, unit);
    atomicAdd(out + 1, lng);
    atomicAdd(out + 2, rows);
  }
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

}  // namespace

DCol plain_to_rle(const CtxPtr& ctx, const DCol& c) {
  require(c.enc == RQ_ENC_PLAIN, "plain_to_rle: plain column required");
  const int64_t n = c.v.n;
  DCol out;
  out.enc = RQ_ENC_RLE;
  out.total = n;
  if (n == 0) {
    out.v.dt = c.logical;
    out.logical = c.logical;
    return out;
  }
  DArr flags = alloc_arr(ctx, RQ_I8, n);
  const int g = grid_for(ctx, n);
  switch (dt_width(c.v.dt)) {
    case 1: dev::k_adjacent_ne<int8_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int8_t>(), n, flags.as<uint8_t>()); break;
    case 2: dev::k_adjacent_ne<int16_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int16_t>(), n, flags.as<uint8_t>()); break;
    case 4:
      if (c.v.dt == RQ_F32) dev::k_adjacent_ne<float><<<g, 256, 0, ctx->stream>>>(c.v.as<float>(), n, flags.as<uint8_t>());
      else dev::k_adjacent_ne<int32_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int32_t>(), n, flags.as<uint8_t>());
      break;
    default:
      if (c.v.dt == RQ_F64) dev::k_adjacent_ne<double><<<g, 256, 0, ctx->stream>>>(c.v.as<double>(), n, flags.as<uint8_t>());
      else dev::k_adjacent_ne<int64_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int64_t>(), n, flags.as<uint8_t>());
  }
  launched(ctx);
  DArr starts;
  flagged_indices(ctx, flags, n, starts);
  const int64_t k = starts.n;
  out.s = starts;
  out.e = alloc_arr(ctx, RQ_I64, k);
  dev::k_ends_from_starts<<<grid_for(ctx, k), 256, 0, ctx->stream>>>(starts.pos(), k, n, out.e.as<int64_t>());
  launched(ctx);
  // runs carry decoded values so the RLE column stands on its own
  DCol raw = c;
  raw.v = gather(ctx, c.v, starts);
  out.v = decode_plain(ctx, raw);  // cast to logical + centre, wrapping
  out.logical = out.v.dt;
  out.gapless = 1;
  return out;
}

DCol plain_to_rle_index(const CtxPtr& ctx, const DCol& c, int64_t min_run) {
  require(min_run >= 2, "plain_to_rle_index: min_run must be >= 2");
  DCol all = plain_to_rle(ctx, c);
  DCol out;
  out.enc = RQ_ENC_RLE_INDEX;
  out.total = all.total;
  out.logical = all.v.dt;
  const int64_t r = all.s.n;
  DArr lflags = alloc_arr(ctx, RQ_I8, r), sflags = alloc_arr(ctx, RQ_I8, r);
  if (r > 0) {
    dev::k_run_len_flags<<<grid_for(ctx, r), 256, 0, ctx->stream>>>(all.s.pos(), all.e.pos(), r, min_run, 1,
                                                                     lflags.as<uint8_t>());
    launched(ctx);
    dev::k_run_len_flags<<<grid_for(ctx, r), 256, 0, ctx->stream>>>(all.s.pos(), all.e.pos(), r, min_run, 0,
                                                                     sflags.as<uint8_t>());
    launched(ctx);
  }
  // long runs stay runs
  DArr long_idx, short_idx, ls, ss;
  select_points(ctx, lflags, all.s, ls, &long_idx);
  out.s = ls;
  out.e = gather(ctx, all.e, long_idx);
  out.v = gather(ctx, all.v, long_idx);
  // short runs expand to one point per row, value repeated
  select_points(ctx, sflags, all.s, ss, &short_idx);
  DArr se = gather(ctx, all.e, short_idx);
  DArr pos, run;
  expand_runs(ctx, ss, se, &pos, &run);
  out.p2 = pos;
  out.v2 = gather(ctx, gather(ctx, all.v, short_idx), run);
  if (out.v.n == 0) out.v.dt = all.v.dt;
  if (out.v2.n == 0) out.v2.dt = all.v.dt;
  return out;
}

namespace {

int sig_bits64(uint64_t r) { return r == 0 ? 0 : 64 - __builtin_clzll(r); }

// values.to_i64() (+ centre), with min / max
DArr decode_unwrapped(const CtxPtr& ctx, const DCol& c, int64_t& lo, int64_t& hi) {
  const int64_t n = c.v.n;
  DArr x = alloc_arr(ctx, RQ_I64, n);
  DArr mm = alloc_arr(ctx, RQ_I64, 2);
  const int64_t init[2] = {INT64_MAX, INT64_MIN};
  RQ_CUDA_CHECK(cudaMemcpyAsync(mm.raw_mut(), init, 16, cudaMemcpyHostToDevice, ctx->stream));
  if (n > 0) {
    dev::k_decode_unwrapped<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(
        c.v.raw(), c.v.dt, n, c.has_center ? 1 : 0, c.center, x.as<int64_t>(), mm.as<long long>());
    launched(ctx);
  }
  const int64_t* h = ctx->readback(mm.raw(), 16);
  lo = h[0];
  hi = h[1];
  return x;
}

// k0-th and k1-th smallest of x (radix select, 8 bits per pass from the top
// significant digit of x − lo); the std::sort + index of primitives.cpp:310-314
void select_two(const CtxPtr& ctx, const DArr& x, int64_t lo, int64_t hi, int64_t k0, int64_t k1,
                int64_t& v0, int64_t& v1) {
  const int bits = sig_bits64(static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo));
  const int ndig = (bits + 7) / 8;
  uint64_t pre[2] = {0, 0};
  int64_t rank[2] = {k0, k1};
  DArr hist = alloc_arr(ctx, RQ_I64, 512);
  for (int d = ndig - 1; d >= 0; --d) {
    RQ_CUDA_CHECK(cudaMemsetAsync(hist.raw_mut(), 0, 512 * 8, ctx->stream));
    dev::k_rsel_hist<<<grid_for(ctx, x.n), 256, 0, ctx->stream>>>(
        x.pos(), x.n, lo, 8 * d, pre[0], pre[1], d < ndig - 1 ? 1 : 0,
        reinterpret_cast<unsigned long long*>(hist.raw_mut()));
    launched(ctx);
    const int64_t* h = ctx->readback(hist.raw(), 512 * 8);
    for (int t = 0; t < 2; ++t) {
      int64_t cum = 0;
      int b = 0;
      for (; b < 256; ++b) {
        const int64_t cnt = h[t * 256 + b];
        if (rank[t] < cum + cnt) break;
        cum += cnt;
      }
      require(b < 256, "select: rank out of range");
      rank[t] -= cum;
      pre[t] = (pre[t] << 8) | static_cast<uint64_t>(b);
    }
  }
  v0 = static_cast<int64_t>(static_cast<uint64_t>(lo) + pre[0]);
  v1 = static_cast<int64_t>(static_cast<uint64_t>(lo) + pre[1]);
}

int32_t narrowest_int(__int128 lo, __int128 hi) {  // primitives.cpp:283-289
  const __int128 a = lo < 0 ? -lo : lo, b = hi < 0 ? -hi : hi;
  const __int128 mag = a > b ? a : b;
  if (mag <= INT8_MAX) return RQ_I8;
  if (mag <= INT16_MAX) return RQ_I16;
  if (mag <= INT32_MAX) return RQ_I32;
  return RQ_I64;
}

void int_limits(int32_t dt, int64_t& mn, int64_t& mx) {
  switch (dt) {
    case RQ_I8: mn = INT8_MIN; mx = INT8_MAX; break;
    case RQ_I16: mn = INT16_MIN; mx = INT16_MAX; break;
    case RQ_I32: mn = INT32_MIN; mx = INT32_MAX; break;
    default: mn = INT64_MIN; mx = INT64_MAX; break;
  }
}

int64_t clamp128(__int128 v) {
  if (v < INT64_MIN) return INT64_MIN;
  if (v > INT64_MAX) return INT64_MAX;
  return static_cast<int64_t>(v);
}

template <class F>
void dispatch_narrow(int32_t dt, F&& f) {
  switch (dt) {
    case RQ_I8: f(int8_t{}); break;
    case RQ_I16: f(int16_t{}); break;
    case RQ_I32: f(int32_t{}); break;
    default: f(int64_t{}); break;
  }
}

}  // namespace

DCol plain_to_plain_index(const CtxPtr& ctx, const DCol& c, double trim) {
  require(c.enc == RQ_ENC_PLAIN, "plain_to_plain_index: plain column required");
  require(trim >= 0.0 && trim < 0.5, "plain_to_plain_index: trim_fraction must be in [0, 0.5)");
  const int64_t n = c.v.n;
  DCol out;
  out.enc = RQ_ENC_PLAIN_INDEX;
  out.total = n;
  if (dt_float(c.logical) || n == 0) {
    out.v = c.v;
    out.logical = c.logical;
    out.has_center = c.has_center;
    out.center = c.center;
    out.v2 = alloc_arr(ctx, c.logical, 0);
    out.p2 = alloc_arr(ctx, RQ_I64, 0);
    return out;
  }
  int64_t mn, mx;
  DArr x = decode_unwrapped(ctx, c, mn, mx);
  const int64_t k = static_cast<int64_t>(trim * static_cast<double>(n));
  int64_t lo, hi;
  select_two(ctx, x, mn, mx, k, n - 1 - k, lo, hi);
  const int64_t center = static_cast<int64_t>((static_cast<__int128>(lo) + hi) / 2);
  const int32_t narrow = narrowest_int(static_cast<__int128>(lo) - center, static_cast<__int128>(hi) - center);
  int64_t rmin, rmax;
  int_limits(narrow, rmin, rmax);
  const int64_t lo_t = clamp128(static_cast<__int128>(center) + rmin);
  const int64_t hi_t = clamp128(static_cast<__int128>(center) + rmax);
  DArr base = alloc_arr(ctx, narrow, n);
  DArr flags = alloc_arr(ctx, RQ_I8, n);
  dispatch_narrow(narrow, [&](auto tag) {
    using N = decltype(tag);
    dev::k_split_base<N><<<grid_for(ctx, n), 256, 0, ctx->stream>>>(x.pos(), n, lo_t, hi_t, center,
                                                                   base.as<N>(), flags.as<uint8_t>());
  });
  launched(ctx);
  DArr op;
  flagged_indices(ctx, flags, n, op);
  out.v = base;
  out.logical = c.logical;
  out.has_center = true;
  out.center = center;
  out.p2 = op;
  out.v2 = cast_values(ctx, gather(ctx, x, op), c.logical);
  return out;
}

EncodingChoiceD choose_encoding(const CtxPtr& ctx, const DCol& c, const HeuristicD& cfg) {
  require(c.enc == RQ_ENC_PLAIN, "choose_encoding: plain column required");
  EncodingChoiceD ch;
  ch.min_run = cfg.min_run;
  ch.trim = cfg.trim;
  ch.width = c.v.dt;
  const int64_t n = c.v.n;
  if (n < cfg.row_threshold) return ch;  // Plain
  const int64_t vw = dt_width(c.logical);
  const int64_t plain_bytes = n * vw;
  // run profile (profile_runs, ingest.cpp:171-196): runs over the storage values
  DCol runs = plain_to_rle(ctx, c);
  const int64_t n_runs = runs.s.n;
  int64_t unit_runs = 0, long_runs = 0, long_rows = 0;
  if (n_runs > 0) {
    DArr acc = alloc_arr(ctx, RQ_I64, 3);
    RQ_CUDA_CHECK(cudaMemsetAsync(acc.raw_mut(), 0, 24, ctx->stream));
    dev::k_run_profile<<<grid_for(ctx, n_runs), 256, 0, ctx->stream>>>(
        runs.s.pos(), runs.e.pos(), n_runs, cfg.min_run, reinterpret_cast<unsigned long long*>(acc.raw_mut()));
    launched(ctx);
    const int64_t* h = ctx->readback(acc.raw(), 24);
    unit_runs = h[0];
    long_runs = h[1];
    long_rows = h[2];
    const double rle_bytes = static_cast<double>(n_runs) * static_cast<double>(vw + 16);
    if (static_cast<double>(plain_bytes) / rle_bytes > cfg.ratio_threshold) {
      ch.scheme = RQ_SCHEME_RLE;
      return ch;
    }
  }
  if (n_runs > 0 && long_runs > 0 &&
      static_cast<double>(unit_runs) > cfg.unit_run_share * static_cast<double>(n_runs)) {
    const double long_bytes = static_cast<double>(long_runs) * static_cast<double>(vw + 16);
    const double long_plain = static_cast<double>(long_rows * vw);
    if (long_plain / long_bytes > cfg.ratio_threshold) {
      ch.scheme = RQ_SCHEME_RLE_INDEX;
      return ch;
    }
  }
  if (!dt_float(c.logical)) {
    DCol split = plain_to_plain_index(ctx, c, cfg.trim);
    if (split.p2.n > 0 && dt_width(split.v.dt) < vw) {
      ch.scheme = RQ_SCHEME_PLAIN_INDEX;
      ch.width = split.v.dt;
      ch.has_center = split.has_center;
      ch.center = split.center;
      return ch;
    }
    // centered_width (ingest.cpp:199-214): mid-range of the untrimmed values
    int64_t lo, hi;
    decode_unwrapped(ctx, c, lo, hi);
    const int64_t center = static_cast<int64_t>((static_cast<__int128>(lo) + hi) / 2);
    const __int128 a = static_cast<__int128>(hi) - center, b = center - static_cast<__int128>(lo);
    const __int128 mag = a > b ? a : b;
    int32_t w = RQ_I64;
    if (mag <= INT8_MAX) w = RQ_I8;
    else if (mag <= INT16_MAX) w = RQ_I16;
    else if (mag <= INT32_MAX) w = RQ_I32;
    if (dt_width(w) < vw) {
      ch.scheme = RQ_SCHEME_PLAIN_CENTERED;
      ch.width = w;
      ch.has_center = true;
      ch.center = center;
      return ch;
    }
  }
  ch.scheme = RQ_SCHEME_PLAIN;
  return ch;
}

DCol encode_column(const CtxPtr& ctx, const DCol& c, const EncodingChoiceD& ch) {
  require(c.enc == RQ_ENC_PLAIN, "encode: plain column required");
  switch (ch.scheme) {
    case RQ_SCHEME_PLAIN: return c;
    case RQ_SCHEME_PLAIN_CENTERED: {
      require(!dt_float(c.logical), "centering requires integer values");
      require(!dt_float(ch.width), "encode: centred width must be an integer type");
      int64_t lo, hi;
      DArr x = decode_unwrapped(ctx, c, lo, hi);
      const int64_t center = ch.has_center ? ch.center : 0;
      DCol out;
      out.enc = RQ_ENC_PLAIN;
      out.total = c.v.n;
      out.logical = c.logical;
      out.has_center = true;
      out.center = center;
      out.v = alloc_arr(ctx, ch.width, c.v.n);
      if (c.v.n > 0) {
        dispatch_narrow(ch.width, [&](auto tag) {
          using N = decltype(tag);
          dev::k_center_cast<N><<<grid_for(ctx, c.v.n), 256, 0, ctx->stream>>>(x.pos(), c.v.n, center,
                                                                                out.v.as<N>());
        });
        launched(ctx);
      }
      return out;
    }
    case RQ_SCHEME_RLE: return plain_to_rle(ctx, c);
    case RQ_SCHEME_RLE_INDEX: return plain_to_rle_index(ctx, c, ch.min_run);
    case RQ_SCHEME_PLAIN_INDEX: return plain_to_plain_index(ctx, c, ch.trim);
  }
  fail("encode: unknown scheme");
}

std::vector<DCol> sort_table(const CtxPtr& ctx, const std::vector<const DCol*>& cols,
                             const std::vector<int>& by) {
  require(!by.empty(), "sort_table: no sort columns");
  std::vector<DArr> keys;
  for (int b : by) {
    require(b >= 0 && b < static_cast<int>(cols.size()), "sort_table: key column index out of range");
    require(cols[b]->enc == RQ_ENC_PLAIN, "sort_table: expects plain columns (sort before encoding)");
    keys.push_back(decode_plain(ctx, *cols[b]));
  }
  const int64_t rows = keys[0].n;
  for (const DCol* c : cols)
    require(c->enc == RQ_ENC_PLAIN && c->v.n == rows, "sort_table: expects plain columns of equal length");
  DArr perm = sort_permutation(ctx, keys);
  std::vector<DCol> out;
  for (const DCol* c : cols) {
    DCol o;
    o.enc = RQ_ENC_PLAIN;
    o.total = rows;
    o.v = gather(ctx, decode_plain(ctx, *c), perm);
    o.logical = o.v.dt;
    out.push_back(std::move(o));
  }
  return out;
}

}  // namespace rqb
