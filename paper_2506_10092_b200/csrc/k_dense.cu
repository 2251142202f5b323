// k_dense.cu — K9 bit-width-reduced unpack (decode_values), gathers and the
// point-wise value kernels behind arith/compare (align.cpp:320-349,
// 551-567). All grid-stride, 128-bit friendly where the layout allows.
#include "device_common.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

// ---- gather (kernels.cpp:195-219) -----------------------------------------------------

template <class T>
__global__ void k_gather(const T* __restrict__ v, const int64_t* __restrict__ idx, int64_t n,
                         T* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = v[ldg64(idx, i)];
}

// ---- decode_values (column.cpp:283-309) ---------------------------------------------
//
// Storage integer (i8/i16/i32/i64) -> logical integer + centre, wrapping at
// the logical width; float storage is cast. Generic over dtypes with the
// switch hoisted out of the loop by template specialisation on the storage.

template <class S>
__global__ void k_decode_int(const S* __restrict__ v, int64_t n, int logical, int has_center,
                             int64_t center, void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t x = wrap_to(logical, static_cast<int64_t>(v[i]));
    if (has_center)
      x = wrap_to(logical, static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(center)));
    switch (logical) {
      case RQ_I8: static_cast<int8_t*>(out)[i] = static_cast<int8_t>(x); break;
      case RQ_I16: static_cast<int16_t*>(out)[i] = static_cast<int16_t>(x); break;
      case RQ_I32: static_cast<int32_t*>(out)[i] = static_cast<int32_t>(x); break;
      case RQ_I64: static_cast<int64_t*>(out)[i] = x; break;
      case RQ_F32: static_cast<float*>(out)[i] = static_cast<float>(x); break;
      default: static_cast<double*>(out)[i] = static_cast<double>(x); break;
    }
  }
}

// generic cast (Array::cast, array.cpp:29-42)
__global__ void k_cast(const void* __restrict__ v, int dt, int64_t n, int to, void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (dt_is_float_dev(to)) {
      const double x = ld_f64(v, dt, i);
      if (to == RQ_F32) static_cast<float*>(out)[i] = static_cast<float>(x);
      else static_cast<double*>(out)[i] = x;
    } else {
      const int64_t x = ld_i64(v, dt, i);
      switch (to) {
        case RQ_I8: static_cast<int8_t*>(out)[i] = static_cast<int8_t>(x); break;
        case RQ_I16: static_cast<int16_t*>(out)[i] = static_cast<int16_t>(x); break;
        case RQ_I32: static_cast<int32_t*>(out)[i] = static_cast<int32_t>(x); break;
        default: static_cast<int64_t*>(out)[i] = x; break;
      }
    }
  }
}

// outlier overlay: dst[p[i]] = ov[i] (column.cpp:299-309)
__global__ void k_scatter_values(const void* __restrict__ ov, int odt, const int64_t* __restrict__ p,
                                 int64_t n, int dst_dt, void* __restrict__ dst) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pos = ldg64(p, i);
    if (dt_is_float_dev(dst_dt)) {
      const double x = ld_f64(ov, odt, i);
      if (dst_dt == RQ_F32) static_cast<float*>(dst)[pos] = static_cast<float>(x);
      else static_cast<double*>(dst)[pos] = x;
    } else {
      const int64_t x = ld_i64(ov, odt, i);
      switch (dst_dt) {
        case RQ_I8: static_cast<int8_t*>(dst)[pos] = static_cast<int8_t>(x); break;
        case RQ_I16: static_cast<int16_t*>(dst)[pos] = static_cast<int16_t>(x); break;
        case RQ_I32: static_cast<int32_t*>(dst)[pos] = static_cast<int32_t>(x); break;
        default: static_cast<int64_t*>(dst)[pos] = x; break;
      }
    }
  }
}

// ---- point-wise arithmetic / comparison (align.cpp:320-349, 551-567) -----------------

template <class T>
__global__ void k_arith(const void* __restrict__ a, int adt, const void* __restrict__ b, int bdt,
                        int64_t n, int op, T* __restrict__ out, int* __restrict__ err) {
  int local_err = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = arith_t<T>(ld_as<T>(a, adt, i), ld_as<T>(b, bdt, i), op, &local_err);
  if (local_err) atomicExch(err, 1);
}

template <class T>
__global__ void k_cmp(const void* __restrict__ a, int adt, const void* __restrict__ b, int bdt,
                      int64_t n, int op, uint8_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = cmp_t<T>(ld_as<T>(a, adt, i), ld_as<T>(b, bdt, i), op) ? 1 : 0;
}

template <class T>
__global__ void k_arith_scalar(const void* __restrict__ a, int adt, int64_t n, T k, int op,
                               int reversed, T* __restrict__ out, int* __restrict__ err) {
  int local_err = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T x = ld_as<T>(a, adt, i);
    out[i] = reversed ? arith_t<T>(k, x, op, &local_err) : arith_t<T>(x, k, op, &local_err);
  }
  if (local_err) atomicExch(err, 1);
}

template <class T>
__global__ void k_cmp_scalar(const void* __restrict__ a, int adt, int64_t n, T k, int op,
                             int reversed, uint8_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T x = ld_as<T>(a, adt, i);
    out[i] = (reversed ? cmp_t<T>(k, x, op) : cmp_t<T>(x, k, op)) ? 1 : 0;
  }
}

// K6+K9 fused for narrow integer plain columns: 16 rows per thread-iteration
// from 128-bit loads of the storage, decode (wrap + centre) inline, one
// 16-byte store of mask bytes. compare_scalar Plain branch (align.cpp:600-606
// decodes the full column first, then compares row by row).
template <class S, class T>
__global__ void __launch_bounds__(256)
    k_plain_cmp_scalar_vec(const S* __restrict__ v, int64_t n, int logical, int has_center,
                           int64_t center, T k, int op, int reversed, uint8_t* __restrict__ out) {
  constexpr int PER = 16;
  const int64_t nvec = n / PER;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < nvec;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    S vals[PER];
    const uint4* src = reinterpret_cast<const uint4*>(v + g * PER);
#pragma unroll
    for (int q = 0; q < static_cast<int>(sizeof(S) * PER / 16); ++q)
      reinterpret_cast<uint4*>(vals)[q] = __ldg(src + q);
    uint32_t packed[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      int64_t x = wrap_to(logical, static_cast<int64_t>(vals[j]));
      if (has_center)
        x = wrap_to(logical, static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(center)));
      const T xv = static_cast<T>(x);
      const bool f = reversed ? cmp_t<T>(k, xv, op) : cmp_t<T>(xv, k, op);
      packed[j >> 2] |= (f ? 1u : 0u) << ((j & 3) * 8);
    }
    reinterpret_cast<uint4*>(out)[g] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
  // tail
  for (int64_t i = nvec * PER + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t x = wrap_to(logical, static_cast<int64_t>(v[i]));
    if (has_center)
      x = wrap_to(logical, static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(center)));
    const T xv = static_cast<T>(x);
    out[i] = (reversed ? cmp_t<T>(k, xv, op) : cmp_t<T>(xv, k, op)) ? 1 : 0;
  }
}

__global__ void k_scatter_flags(uint8_t* __restrict__ bits, const int64_t* __restrict__ p,
                                const uint8_t* __restrict__ flags, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bits[ldg64(p, i)] = flags[i];
}

__global__ void k_bytes_and(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                            uint8_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = (a[i] && b[i]) ? 1 : 0;
}

__global__ void k_bytes_or(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                           uint8_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = (a[i] || b[i]) ? 1 : 0;
}

__global__ void k_bytes_not(const uint8_t* __restrict__ a, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = a[i] ? 0 : 1;
}

__global__ void k_set_bits(uint8_t* __restrict__ bits, const int64_t* __restrict__ p, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bits[ldg64(p, i)] = 1;
}

__global__ void k_normalize_bits(const uint8_t* __restrict__ a, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = a[i] ? 1 : 0;
}

// gapless run starts from ends: s_0 = 0, s_i = e_{i-1} + 1
__global__ void k_starts(const int64_t* __restrict__ e, int64_t n, int64_t* __restrict__ s) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s[i] = i == 0 ? 0 : ldg64(e, i - 1) + 1;
}

__global__ void k_iota(int64_t* __restrict__ out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = i;
}

}  // namespace dev

namespace {

int grid_for(const CtxPtr& ctx, int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

void check_launch(const CtxPtr& ctx) {
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
}

// integer division-by-zero flag readback (align.cpp:297-299)
struct ErrFlag {
  DArr buf;
  explicit ErrFlag(const CtxPtr& ctx) : buf(alloc_arr(ctx, RQ_I32, 1)) {
    RQ_CUDA_CHECK(cudaMemsetAsync(buf.raw_mut(), 0, 4, ctx->stream));
  }
  int* ptr() const { return buf.as<int>(); }
  void check(const CtxPtr& ctx) const {
    const int64_t* h = ctx->readback(buf.raw(), 8);
    if (static_cast<int32_t>(h[0] & 0xffffffff) != 0) fail("integer division by zero");
  }
};

}  // namespace

DArr gather(const CtxPtr& ctx, const DArr& v, const DArr& idx) {
  DArr out = alloc_arr(ctx, v.dt, idx.n);
  if (idx.n == 0) return out;
  const int g = grid_for(ctx, idx.n);
  switch (dt_width(v.dt)) {
    case 1: dev::k_gather<uint8_t><<<g, 256, 0, ctx->stream>>>(v.as<uint8_t>(), idx.pos(), idx.n, out.as<uint8_t>()); break;
    case 2: dev::k_gather<uint16_t><<<g, 256, 0, ctx->stream>>>(v.as<uint16_t>(), idx.pos(), idx.n, out.as<uint16_t>()); break;
    case 4: dev::k_gather<uint32_t><<<g, 256, 0, ctx->stream>>>(v.as<uint32_t>(), idx.pos(), idx.n, out.as<uint32_t>()); break;
    default: dev::k_gather<uint64_t><<<g, 256, 0, ctx->stream>>>(v.as<uint64_t>(), idx.pos(), idx.n, out.as<uint64_t>()); break;
  }
  check_launch(ctx);
  return out;
}

DArr cast_values(const CtxPtr& ctx, const DArr& v, int32_t to) {
  if (v.dt == to) return v;
  DArr out = alloc_arr(ctx, to, v.n);
  if (v.n == 0) return out;
  dev::k_cast<<<grid_for(ctx, v.n), 256, 0, ctx->stream>>>(v.raw(), v.dt, v.n, to, out.raw_mut());
  check_launch(ctx);
  return out;
}

DArr decode_plain(const CtxPtr& ctx, const DCol& c) {
  if (!c.has_center && c.v.dt == c.logical) return c.v;
  if (dt_float(c.v.dt) || dt_float(c.logical)) {
    require(!c.has_center, "decode: center on float column");
    return cast_values(ctx, c.v, c.logical);
  }
  DArr out = alloc_arr(ctx, c.logical, c.v.n);
  if (c.v.n == 0) return out;
  const int g = grid_for(ctx, c.v.n);
  const int hc = c.has_center ? 1 : 0;
  switch (c.v.dt) {
    case RQ_I8: dev::k_decode_int<int8_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int8_t>(), c.v.n, c.logical, hc, c.center, out.raw_mut()); break;
    case RQ_I16: dev::k_decode_int<int16_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int16_t>(), c.v.n, c.logical, hc, c.center, out.raw_mut()); break;
    case RQ_I32: dev::k_decode_int<int32_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int32_t>(), c.v.n, c.logical, hc, c.center, out.raw_mut()); break;
    default: dev::k_decode_int<int64_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int64_t>(), c.v.n, c.logical, hc, c.center, out.raw_mut()); break;
  }
  check_launch(ctx);
  return out;
}

DArr decode_plain_index(const CtxPtr& ctx, const DCol& c) {
  // column.cpp:299-309: decode the base, cast to the outliers' dtype, overlay
  DCol base = c;
  base.enc = RQ_ENC_PLAIN;
  DArr wide = cast_values(ctx, decode_plain(ctx, base), c.v2.dt);
  if (wide.buf == c.v.buf) wide = copy_prefix(ctx, wide, wide.n);  // never write into the input
  if (c.p2.n > 0) {
    dev::k_scatter_values<<<grid_for(ctx, c.p2.n), 256, 0, ctx->stream>>>(
        c.v2.raw(), c.v2.dt, c.p2.pos(), c.p2.n, wide.dt, wide.raw_mut());
    check_launch(ctx);
  }
  return wide;
}

DArr arith_values(const CtxPtr& ctx, const DArr& a, const DArr& b, int op) {
  require(a.n == b.n, "arith: value length mismatch");
  const int32_t dt = dt_promote(a.dt, b.dt);
  DArr out = alloc_arr(ctx, dt, a.n);
  if (a.n == 0) return out;
  const int g = grid_for(ctx, a.n);
  if (dt == RQ_F64) {
    dev::k_arith<double><<<g, 256, 0, ctx->stream>>>(a.raw(), a.dt, b.raw(), b.dt, a.n, op, out.as<double>(), nullptr);
    check_launch(ctx);
  } else {
    ErrFlag err(ctx);
    dev::k_arith<int64_t><<<g, 256, 0, ctx->stream>>>(a.raw(), a.dt, b.raw(), b.dt, a.n, op, out.as<int64_t>(), err.ptr());
    check_launch(ctx);
    if (op == RQ_DIV) err.check(ctx);
  }
  return out;
}

DArr cmp_values(const CtxPtr& ctx, const DArr& a, const DArr& b, int op) {
  require(a.n == b.n, "compare: value length mismatch");
  DArr out = alloc_arr(ctx, RQ_I8, a.n);
  if (a.n == 0) return out;
  const int g = grid_for(ctx, a.n);
  if (dt_float(a.dt) || dt_float(b.dt))
    dev::k_cmp<double><<<g, 256, 0, ctx->stream>>>(a.raw(), a.dt, b.raw(), b.dt, a.n, op, out.as<uint8_t>());
  else
    dev::k_cmp<int64_t><<<g, 256, 0, ctx->stream>>>(a.raw(), a.dt, b.raw(), b.dt, a.n, op, out.as<uint8_t>());
  check_launch(ctx);
  return out;
}

DArr scalar_arith_values(const CtxPtr& ctx, const DArr& v, Scalar k, int op, bool reversed) {
  const bool flt = dt_float(v.dt) || k.is_float;
  DArr out = alloc_arr(ctx, flt ? RQ_F64 : RQ_I64, v.n);
  if (v.n == 0) return out;
  const int g = grid_for(ctx, v.n);
  if (flt) {
    const double kd = k.is_float ? k.f : static_cast<double>(k.i);
    dev::k_arith_scalar<double><<<g, 256, 0, ctx->stream>>>(v.raw(), v.dt, v.n, kd, op, reversed, out.as<double>(), nullptr);
    check_launch(ctx);
  } else {
    ErrFlag err(ctx);
    dev::k_arith_scalar<int64_t><<<g, 256, 0, ctx->stream>>>(v.raw(), v.dt, v.n, k.i, op, reversed, out.as<int64_t>(), err.ptr());
    check_launch(ctx);
    if (op == RQ_DIV) err.check(ctx);
  }
  return out;
}

DArr scalar_cmp_values(const CtxPtr& ctx, const DArr& v, Scalar k, int op, bool reversed) {
  DArr out = alloc_arr(ctx, RQ_I8, v.n);
  if (v.n == 0) return out;
  const int g = grid_for(ctx, v.n);
  if (dt_float(v.dt) || k.is_float) {
    const double kd = k.is_float ? k.f : static_cast<double>(k.i);
    dev::k_cmp_scalar<double><<<g, 256, 0, ctx->stream>>>(v.raw(), v.dt, v.n, kd, op, reversed, out.as<uint8_t>());
  } else {
    dev::k_cmp_scalar<int64_t><<<g, 256, 0, ctx->stream>>>(v.raw(), v.dt, v.n, k.i, op, reversed, out.as<uint8_t>());
  }
  check_launch(ctx);
  return out;
}

DArr plain_cmp_scalar(const CtxPtr& ctx, const DCol& c, Scalar k, int op, bool reversed) {
  // float storage or float literal: decode then compare in f64 (align.cpp:551-567)
  if (dt_float(c.v.dt) || dt_float(c.logical) || k.is_float)
    return scalar_cmp_values(ctx, decode_plain(ctx, c), k, op, reversed);
  DArr out = alloc_arr(ctx, RQ_I8, c.v.n);
  if (c.v.n == 0) return out;
  const int g = grid_for(ctx, c.v.n / 16 + 1);
  const int hc = c.has_center ? 1 : 0;
  const int rv = reversed ? 1 : 0;
  switch (c.v.dt) {
    case RQ_I8: dev::k_plain_cmp_scalar_vec<int8_t, int64_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int8_t>(), c.v.n, c.logical, hc, c.center, k.i, op, rv, out.as<uint8_t>()); break;
    case RQ_I16: dev::k_plain_cmp_scalar_vec<int16_t, int64_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int16_t>(), c.v.n, c.logical, hc, c.center, k.i, op, rv, out.as<uint8_t>()); break;
    case RQ_I32: dev::k_plain_cmp_scalar_vec<int32_t, int64_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int32_t>(), c.v.n, c.logical, hc, c.center, k.i, op, rv, out.as<uint8_t>()); break;
    default: dev::k_plain_cmp_scalar_vec<int64_t, int64_t><<<g, 256, 0, ctx->stream>>>(c.v.as<int64_t>(), c.v.n, c.logical, hc, c.center, k.i, op, rv, out.as<uint8_t>()); break;
  }
  check_launch(ctx);
  return out;
}

void scatter_flags(const CtxPtr& ctx, DArr& bits, const DArr& p, const DArr& flags) {
  if (p.n == 0) return;
  dev::k_scatter_flags<<<grid_for(ctx, p.n), 256, 0, ctx->stream>>>(bits.as<uint8_t>(), p.pos(), flags.as<uint8_t>(), p.n);
  check_launch(ctx);
}

DArr bytes_and(const CtxPtr& ctx, const DArr& a, const DArr& b) {
  require(a.n == b.n, "and: length mismatch");
  DArr out = alloc_arr(ctx, RQ_I8, a.n);
  if (a.n == 0) return out;
  dev::k_bytes_and<<<grid_for(ctx, a.n), 256, 0, ctx->stream>>>(a.as<uint8_t>(), b.as<uint8_t>(), a.n, out.as<uint8_t>());
  check_launch(ctx);
  return out;
}

DArr bytes_or(const CtxPtr& ctx, const DArr& a, const DArr& b) {
  require(a.n == b.n, "or: length mismatch");
  DArr out = alloc_arr(ctx, RQ_I8, a.n);
  if (a.n == 0) return out;
  dev::k_bytes_or<<<grid_for(ctx, a.n), 256, 0, ctx->stream>>>(a.as<uint8_t>(), b.as<uint8_t>(), a.n, out.as<uint8_t>());
  check_launch(ctx);
  return out;
}

DArr bytes_not(const CtxPtr& ctx, const DArr& a) {
  DArr out = alloc_arr(ctx, RQ_I8, a.n);
  if (a.n == 0) return out;
  dev::k_bytes_not<<<grid_for(ctx, a.n), 256, 0, ctx->stream>>>(a.as<uint8_t>(), a.n, out.as<uint8_t>());
  check_launch(ctx);
  return out;
}

DArr bytes_copy01(const CtxPtr& ctx, const DArr& a) {
  DArr out = alloc_arr(ctx, RQ_I8, a.n);
  if (a.n == 0) return out;
  dev::k_normalize_bits<<<grid_for(ctx, a.n), 256, 0, ctx->stream>>>(a.as<uint8_t>(), a.n, out.as<uint8_t>());
  check_launch(ctx);
  return out;
}

void set_bits(const CtxPtr& ctx, DArr& bits, const DArr& p) {
  if (p.n == 0) return;
  dev::k_set_bits<<<grid_for(ctx, p.n), 256, 0, ctx->stream>>>(bits.as<uint8_t>(), p.pos(), p.n);
  check_launch(ctx);
}

DArr zeros_bytes(const CtxPtr& ctx, int64_t n) {
  DArr out = alloc_arr(ctx, RQ_I8, n);
  if (n) RQ_CUDA_CHECK(cudaMemsetAsync(out.raw_mut(), 0, static_cast<size_t>(n), ctx->stream));
  return out;
}

// dst[idx[i]] = src[i] (same dtype)
void scatter_values(const CtxPtr& ctx, DArr& dst, const DArr& idx, const DArr& src) {
  require(dst.dt == src.dt, "scatter: dtype mismatch");
  if (idx.n == 0) return;
  dev::k_scatter_values<<<grid_for(ctx, idx.n), 256, 0, ctx->stream>>>(src.raw(), src.dt, idx.pos(), idx.n,
                                                                      dst.dt, dst.raw_mut());
  check_launch(ctx);
}

DArr starts_from_ends(const CtxPtr& ctx, const DArr& e) {
  DArr s = alloc_arr(ctx, RQ_I64, e.n);
  if (e.n == 0) return s;
  dev::k_starts<<<grid_for(ctx, e.n), 256, 0, ctx->stream>>>(e.pos(), e.n, s.as<int64_t>());
  check_launch(ctx);
  return s;
}

DArr iota(const CtxPtr& ctx, int64_t n) {
  DArr out = alloc_arr(ctx, RQ_I64, n);
  if (n == 0) return out;
  dev::k_iota<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(out.as<int64_t>(), n);
  check_launch(ctx);
  return out;
}

}  // namespace rqb
