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
  select_points(ctx, flags, iota(ctx, n), starts, nullptr);
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

}  // namespace rqb
