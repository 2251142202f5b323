// k_groupby.cu — K10 group-by over dictionary-code keys with run-length
// weighted aggregation (agg::group_aggregate, groupby.cpp:144-162).
//
// Grouping (unique_with_inverse, kernels.cpp:127-187) assigns ids in
// ascending lexicographic key order. For integer keys whose joint value
// range is small (dictionary codes, dates, flags — the path's keys) the id is
// the mixed-radix slot Σ (k_c − min_c)·stride_c, which is already ascending
// lexicographic, so no sort is needed: aggregates fold into per-CTA
// shared-memory tables indexed by slot and flush with one atomic per slot
// per CTA; absent slots are compacted away at the end.
//
// Alignment follows the reference's left fold (align_many, align.cpp:233-254)
// on the device. The fused per-aggregate kernels for the large-table shapes
// (RLE keys × RLE / plain / index data, no per-row materialisation) live in
// k_groupfused.cu and are dispatched from group_aggregate when applicable.
#include <cmath>
#include <limits>

#include "device_common.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

// per-slot accumulator kinds
enum AggKind { K_SUM_I = 0, K_SUM_F = 1, K_MIN_I = 2, K_MAX_I = 3, K_MIN_F = 4, K_MAX_F = 5, K_SQ = 6 };

struct KeySpec {
  const void* v[8];
  int dt[8];
  int64_t mn[8];
  int64_t stride[8];
  int nk;
};

__global__ void k_group_slots(KeySpec ks, int64_t n, int64_t* __restrict__ gid) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t g = 0;
    for (int c = 0; c < ks.nk; ++c) g += (ld_i64(ks.v[c], ks.dt[c], i) - ks.mn[c]) * ks.stride[c];
    gid[i] = g;
  }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_minmax_i64(const void* __restrict__ v, int dt, int64_t n, long long* __restrict__ out) {
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

__device__ __forceinline__ void atomic_min_f64(double* addr, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *a;
  while (__longlong_as_double(old) > v) {
    const unsigned long long prev = atomicCAS(a, old, __double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}
__device__ __forceinline__ void atomic_max_f64(double* addr, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *a;
  while (__longlong_as_double(old) < v) {
    const unsigned long long prev = atomicCAS(a, old, __double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}

// Accumulate into per-group tables: acc (8 B per group, kind-dependent) and
// cnt (Σ weights). Shared-memory staging when the table fits.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_scatter_agg(const int64_t* __restrict__ gid, const void* __restrict__ v, int dt,
                  const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t n,
                  int64_t G, int kind, const double* __restrict__ mean,
                  unsigned long long* __restrict__ acc, unsigned long long* __restrict__ cnt) {
  extern __shared__ unsigned long long smem[];
  const bool use_smem = G * 16 <= 48 * 1024;
  unsigned long long* sacc = smem;
  unsigned long long* scnt = smem + (use_smem ? G : 0);
  if (use_smem) {
    for (int64_t g = threadIdx.x; g < G; g += BLOCK) {
      unsigned long long init = 0;
      if (kind == K_MIN_I) init = static_cast<unsigned long long>(INT64_MAX);
      if (kind == K_MAX_I) init = static_cast<unsigned long long>(INT64_MIN);
      if (kind == K_MIN_F) init = __double_as_longlong(INFINITY);
      if (kind == K_MAX_F) init = __double_as_longlong(-INFINITY);
      sacc[g] = init;
      scnt[g] = 0;
    }
    __syncthreads();
  }
  unsigned long long* A = use_smem ? sacc : acc;
  unsigned long long* C = use_smem ? scnt : cnt;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * BLOCK) {
    const int64_t g = ldg64(gid, i);
    const int64_t w = s ? ldg64(e, i) - ldg64(s, i) + 1 : 1;
    switch (kind) {
      case K_SUM_I:
        atomicAdd(A + g, static_cast<unsigned long long>(ld_i64(v, dt, i)) * static_cast<unsigned long long>(w));
        break;
      case K_SUM_F:
        atomicAdd(reinterpret_cast<double*>(A) + g, ld_f64(v, dt, i) * static_cast<double>(w));
        break;
      case K_MIN_I: atomicMin(reinterpret_cast<long long*>(A) + g, ld_i64(v, dt, i)); break;
      case K_MAX_I: atomicMax(reinterpret_cast<long long*>(A) + g, ld_i64(v, dt, i)); break;
      case K_MIN_F: atomic_min_f64(reinterpret_cast<double*>(A) + g, ld_f64(v, dt, i)); break;
      case K_MAX_F: atomic_max_f64(reinterpret_cast<double*>(A) + g, ld_f64(v, dt, i)); break;
      default: {
        const double d = ld_f64(v, dt, i) - mean[g];
        atomicAdd(reinterpret_cast<double*>(A) + g, d * d * static_cast<double>(w));
      }
    }
    atomicAdd(C + g, static_cast<unsigned long long>(w));
  }
  if (use_smem) {
    __syncthreads();
    for (int64_t g = threadIdx.x; g < G; g += BLOCK) {
      if (scnt[g] == 0) continue;
      atomicAdd(cnt + g, scnt[g]);
      switch (kind) {
        case K_SUM_I: atomicAdd(acc + g, sacc[g]); break;
        case K_SUM_F:
        case K_SQ: atomicAdd(reinterpret_cast<double*>(acc) + g, __longlong_as_double(sacc[g])); break;
        case K_MIN_I: atomicMin(reinterpret_cast<long long*>(acc) + g, static_cast<long long>(sacc[g])); break;
        case K_MAX_I: atomicMax(reinterpret_cast<long long*>(acc) + g, static_cast<long long>(sacc[g])); break;
        case K_MIN_F: atomic_min_f64(reinterpret_cast<double*>(acc) + g, __longlong_as_double(sacc[g])); break;
        default: atomic_max_f64(reinterpret_cast<double*>(acc) + g, __longlong_as_double(sacc[g])); break;
      }
    }
  }
}

__global__ void k_init_table(unsigned long long* __restrict__ t, int64_t G, unsigned long long init) {
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < G;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x)
    t[g] = init;
}

__global__ void k_present_flags(const unsigned long long* __restrict__ cnt, int64_t G,
                                uint8_t* __restrict__ flags) {
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < G;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flags[g] = cnt[g] > 0;
}

// mean per group for VAR/STD pass 2 (f64 sum / count)
__global__ void k_group_mean(const unsigned long long* __restrict__ fsum,
                             const unsigned long long* __restrict__ cnt, int64_t G,
                             double* __restrict__ mean) {
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < G;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x)
    mean[g] = cnt[g] ? __longlong_as_double(fsum[g]) / static_cast<double>(cnt[g]) : 0.0;
}

// Final value per present group (groupby.cpp:67-135 output conventions).
__global__ void k_group_finish(const int64_t* __restrict__ slots, int64_t ng, int fn, int flt,
                               const unsigned long long* __restrict__ acc,
                               const unsigned long long* __restrict__ cnt,
                               const unsigned long long* __restrict__ sq, void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < ng;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = ldg64(slots, i);
    const double c = static_cast<double>(cnt[g]);
    switch (fn) {
      case RQ_SUM:
      case RQ_MIN:
      case RQ_MAX:
        static_cast<unsigned long long*>(out)[i] = acc[g];  // i64 or f64 bits
        break;
      case RQ_COUNT: static_cast<long long*>(out)[i] = static_cast<long long>(cnt[g]); break;
      case RQ_AVG: static_cast<double*>(out)[i] = __longlong_as_double(acc[g]) / c; break;
      default: {
        const double var = __longlong_as_double(sq[g]) / c;
        static_cast<double*>(out)[i] = fn == RQ_VAR ? var : sqrt(var);
      }
    }
  }
  (void)flt;
}

// keys from slots: key_c = min_c + (slot / stride_c) % range_c
__global__ void k_slot_keys(const int64_t* __restrict__ slots, int64_t ng, int64_t mn,
                            int64_t stride, int64_t range, int dt, void* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < ng;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = mn + (ldg64(slots, i) / stride) % range;
    switch (dt) {
      case RQ_I8: static_cast<int8_t*>(out)[i] = static_cast<int8_t>(k); break;
      case RQ_I16: static_cast<int16_t*>(out)[i] = static_cast<int16_t>(k); break;
      case RQ_I32: static_cast<int32_t*>(out)[i] = static_cast<int32_t>(k); break;
      default: static_cast<int64_t*>(out)[i] = k; break;
    }
  }
}

}  // namespace dev

namespace {

constexpr int64_t kDenseSlotLimit = int64_t{1} << 24;

int grid_for(const CtxPtr& ctx, int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

void launched(const CtxPtr& ctx) {
  ctx->count_launch();
  RQ_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

Decomp decompose_for_group(const CtxPtr& ctx, const DCol& c) {
  Decomp d;
  switch (c.enc) {
    case RQ_ENC_PLAIN:
      d.kind = 0;
      d.n = c.total;
      d.values = decode_plain(ctx, c);
      return d;
    case RQ_ENC_PLAIN_INDEX:
      d.kind = 0;
      d.n = c.total;
      d.values = decode_plain_index(ctx, c);
      return d;
    case RQ_ENC_RLE:
      d.kind = 1;
      d.s = c.s;
      d.e = c.e;
      d.values = c.v;
      return d;
    case RQ_ENC_INDEX:
      d.kind = 2;
      d.p = c.p;
      d.values = c.v;
      return d;
    default:
      fail("decompose: rle+index has two positional parts; distribute first");
  }
}

DCol col_from_decomp(const Decomp& d, const DArr& v, int64_t total) {
  DCol c;
  c.total = total;
  c.v = v;
  c.logical = v.dt;
  if (d.kind == 0) {
    c.enc = RQ_ENC_PLAIN;
    c.total = v.n;
  } else if (d.kind == 1) {
    c.enc = RQ_ENC_RLE;
    c.s = d.s;
    c.e = d.e;
  } else {
    c.enc = RQ_ENC_INDEX;
    c.p = d.p;
  }
  return c;
}

// Left-fold alignment of all columns (align_many, align.cpp:233-254): the
// shape of column 0 is intersected with each next column; accumulated value
// arrays are re-gathered through the new take indices.
MultiAligned align_many(const CtxPtr& ctx, const std::vector<const DCol*>& cols) {
  require(!cols.empty(), "align_many: no columns");
  const int64_t total = cols[0]->total;
  for (auto* c : cols) require(c->total == total, "align_many: total_size mismatch");
  MultiAligned acc;
  acc.shape = decompose_for_group(ctx, *cols[0]);
  acc.values.push_back(acc.shape.values);
  for (size_t i = 1; i < cols.size(); ++i) {
    Decomp di = decompose_for_group(ctx, *cols[i]);
    // reuse the pairwise align on carrier columns whose values are slot ids
    DCol shape_col = col_from_decomp(acc.shape, iota(ctx, acc.values[0].n), total);
    DCol next_col = col_from_decomp(di, iota(ctx, di.values.n), total);
    Aligned ap = align(ctx, shape_col, next_col);
    // ap.v1 / ap.v2 hold the source slot of every output slot (take indices)
    for (auto& v : acc.values) v = gather(ctx, v, ap.v1);
    acc.values.push_back(gather(ctx, di.values, ap.v2));
    acc.shape.kind = ap.kind;
    acc.shape.s = ap.s;
    acc.shape.e = ap.e;
    acc.shape.p = ap.p;
    acc.shape.n = ap.kind == 0 ? ap.v1.n : 0;
  }
  return acc;
}

GroupAggOut group_aggregate(const CtxPtr& ctx, const std::vector<const DCol*>& keys,
                            const std::vector<const DCol*>& data, const std::vector<int>& fns,
                            bool normalize) {
  require(!keys.empty(), "group: empty key list");
  require(data.size() == fns.size(), "group_aggregate: data/function count mismatch");
  require(keys.size() <= 8, "group: at most 8 key columns");
  for (int fn : fns) require(fn >= RQ_SUM && fn <= RQ_VAR, "aggregate: unknown function");
  std::vector<const DCol*> all(keys.begin(), keys.end());
  all.insert(all.end(), data.begin(), data.end());
  if (!normalize)
    for (auto* c : all)
      if (c->enc == RQ_ENC_RLE_INDEX) fail("decompose: rle+index has two positional parts; distribute first");
  {
    GroupAggOut fused;
    if (group_aggregate_fused(ctx, keys, data, fns, fused)) return fused;
  }
  std::vector<DCol> normalized;
  if (normalize) {
    normalized.reserve(all.size());
    for (auto*& c : all) {
      normalized.push_back(normalize_basic(ctx, *c));
      c = &normalized.back();
    }
  }
  MultiAligned ma = align_many(ctx, all);
  const size_t nk = keys.size();
  const int64_t slots = ma.values[0].n;
  const DArr* ws = ma.shape.kind == 1 ? &ma.shape.s : nullptr;
  const DArr* we = ma.shape.kind == 1 ? &ma.shape.e : nullptr;

  // dense slot ids over the joint key range when it is small (dictionary
  // codes, dates, flags); otherwise sort-based ids (K11, k_sort.cu)
  dev::KeySpec ks{};
  ks.nk = static_cast<int>(nk);
  std::vector<int64_t> mn(nk, 0), range(nk, 1);
  int64_t G = 1;
  bool dense = true;
  for (size_t c = 0; c < nk; ++c)
    if (dt_float(ma.values[c].dt)) dense = false;
  for (size_t c = 0; c < nk && dense && slots > 0; ++c) {
    const DArr& kv = ma.values[c];
    DArr mm = alloc_arr(ctx, RQ_I64, 2);
    const int64_t init[2] = {INT64_MAX, INT64_MIN};
    RQ_CUDA_CHECK(cudaMemcpyAsync(mm.raw_mut(), init, 16, cudaMemcpyHostToDevice, ctx->stream));
    dev::k_minmax_i64<256><<<grid_for(ctx, kv.n), 256, 0, ctx->stream>>>(kv.raw(), kv.dt, kv.n,
                                                                        mm.as<long long>());
    launched(ctx);
    const int64_t* h = ctx->readback(mm.raw(), 16);
    mn[c] = h[0];
    const uint64_t r = static_cast<uint64_t>(h[1]) - static_cast<uint64_t>(h[0]) + 1;
    if (r == 0 || r > static_cast<uint64_t>(kDenseSlotLimit / G)) {
      dense = false;
      break;
    }
    range[c] = static_cast<int64_t>(r);
    G *= range[c];
  }
  DArr gid;
  SortedGroups sg;
  std::vector<int64_t> strides(nk, 1);
  if (dense) {
    int64_t stride = 1;
    for (size_t c = nk; c-- > 0;) {
      strides[c] = stride;
      stride *= range[c];
    }
    for (size_t c = 0; c < nk; ++c) {
      ks.v[c] = ma.values[c].raw();
      ks.dt[c] = ma.values[c].dt;
      ks.mn[c] = mn[c];
      ks.stride[c] = strides[c];
    }
    gid = alloc_arr(ctx, RQ_I64, slots);
    if (slots) {
      dev::k_group_slots<<<grid_for(ctx, slots), 256, 0, ctx->stream>>>(ks, slots, gid.as<int64_t>());
      launched(ctx);
    }
  } else {
    sg = group_ids_sorted(ctx, std::vector<DArr>(ma.values.begin(), ma.values.begin() + nk));
    gid = sg.inverse;
    G = sg.n_groups > 0 ? sg.n_groups : 1;
  }

  auto table = [&](unsigned long long init) {
    DArr t = alloc_arr(ctx, RQ_I64, G);
    dev::k_init_table<<<grid_for(ctx, G), 256, 0, ctx->stream>>>(reinterpret_cast<unsigned long long*>(t.raw_mut()), G, init);
    launched(ctx);
    return t;
  };
  const size_t smem = static_cast<size_t>(G * 16 <= 48 * 1024 ? G * 16 : 0);
  auto scatter = [&](const DArr& v, int kind, const DArr* mean, DArr& acc, DArr& cnt) {
    if (slots == 0) return;
    dev::k_scatter_agg<256><<<grid_for(ctx, slots), 256, smem, ctx->stream>>>(
        gid.pos(), v.raw(), v.dt, ws ? ws->pos() : nullptr, we ? we->pos() : nullptr, slots, G,
        kind, mean ? mean->as<double>() : nullptr,
        reinterpret_cast<unsigned long long*>(acc.raw_mut()),
        reinterpret_cast<unsigned long long*>(cnt.raw_mut()));
    launched(ctx);
  };

  // presence of each slot = count of covered rows with that key
  DArr pres_acc = table(0), pres_cnt = table(0);
  {
    DArr zero_vals = ma.values[0];
    scatter(zero_vals, dev::K_SUM_I, nullptr, pres_acc, pres_cnt);
  }
  DArr flags = alloc_arr(ctx, RQ_I8, G);
  dev::k_present_flags<<<grid_for(ctx, G), 256, 0, ctx->stream>>>(
      reinterpret_cast<const unsigned long long*>(pres_cnt.raw()), G, flags.as<uint8_t>());
  launched(ctx);
  DArr all_slots = iota(ctx, G);
  DArr present;
  select_points(ctx, flags, all_slots, present, nullptr);
  const int64_t ng = present.n;

  GroupAggOut out;
  out.n_groups = ng;
  for (size_t c = 0; c < nk; ++c) {
    const int32_t kdt = ma.values[c].dt;
    if (!dense) {  // the group's key = its first row in stable sorted order
      out.keys.push_back(gather(ctx, ma.values[c], gather(ctx, sg.first_rows, present)));
      continue;
    }
    DArr k = alloc_arr(ctx, kdt, ng);
    if (ng) {
      dev::k_slot_keys<<<grid_for(ctx, ng), 256, 0, ctx->stream>>>(present.pos(), ng, mn[c], strides[c],
                                                                   range[c], kdt, k.raw_mut());
      launched(ctx);
    }
    out.keys.push_back(k);
  }
  for (size_t d = 0; d < data.size(); ++d) {
    const DArr& v = ma.values[nk + d];
    const int fn = fns[d];
    const bool flt = dt_float(v.dt);
    if ((flt && fn == RQ_SUM) || fn == RQ_AVG || fn == RQ_STD || fn == RQ_VAR) {
      // f64 sums folded per group in slot order (aggregate_array, k_boundary.cu):
      // bit-identical to the reference's loop and from run to run
      out.vals.push_back(gather(ctx, aggregate_array(ctx, ma.shape, v, gid, G, fn), present));
      continue;
    }
    int kind;
    unsigned long long init = 0;
    int32_t odt = RQ_F64;
    switch (fn) {
      case RQ_SUM: kind = flt ? dev::K_SUM_F : dev::K_SUM_I; odt = flt ? RQ_F64 : RQ_I64; break;
      case RQ_COUNT: kind = dev::K_SUM_I; odt = RQ_I64; break;
      case RQ_MIN:
        kind = flt ? dev::K_MIN_F : dev::K_MIN_I;
        odt = flt ? RQ_F64 : RQ_I64;
        init = flt ? 0x7ff0000000000000ull : static_cast<unsigned long long>(INT64_MAX);
        break;
      case RQ_MAX:
        kind = flt ? dev::K_MAX_F : dev::K_MAX_I;
        odt = flt ? RQ_F64 : RQ_I64;
        init = flt ? 0xfff0000000000000ull : static_cast<unsigned long long>(INT64_MIN);
        break;
      default: kind = dev::K_SUM_F; odt = RQ_F64; break;  // AVG / STD / VAR
    }
    DArr acc = table(init), cnt = table(0);
    scatter(v, kind, nullptr, acc, cnt);
    DArr sq;
    if (fn == RQ_STD || fn == RQ_VAR) {
      DArr mean = alloc_arr(ctx, RQ_F64, G);
      dev::k_group_mean<<<grid_for(ctx, G), 256, 0, ctx->stream>>>(
          reinterpret_cast<const unsigned long long*>(acc.raw()),
          reinterpret_cast<const unsigned long long*>(cnt.raw()), G, mean.as<double>());
      launched(ctx);
      sq = table(0);
      DArr cnt2 = table(0);
      scatter(v, dev::K_SQ, &mean, sq, cnt2);
    }
    DArr res = alloc_arr(ctx, odt, ng);
    if (ng) {
      dev::k_group_finish<<<grid_for(ctx, ng), 256, 0, ctx->stream>>>(
          present.pos(), ng, fn, flt ? 1 : 0, reinterpret_cast<const unsigned long long*>(acc.raw()),
          reinterpret_cast<const unsigned long long*>(cnt.raw()),
          sq.n ? reinterpret_cast<const unsigned long long*>(sq.raw()) : nullptr, res.raw_mut());
      launched(ctx);
    }
    out.vals.push_back(res);
  }
  return out;
}

// The filtered-aggregate query shape (runner.cpp:243-336 for one predicate):
// aggregate_all(arith(filter(a, m), filter(b, m), op), fn), m = compare_scalar(c, k, cmp),
// run as the device operator chain; fused single-pass kernels replace it for
// the RLE/Index shapes (k_fused.cu).
AggOut filtered_aggregate_binop_chain(const CtxPtr& ctx, const DCol& c, Scalar k, int cmp,
                                      const DCol& a, const DCol& b, int op, int fn) {
  DMask m = compare_scalar(ctx, c, k, cmp, false);
  DCol fa = filter(ctx, a, m);
  DCol fb = filter(ctx, b, m);
  DCol prod = arith(ctx, fa, fb, op);
  return aggregate_column(ctx, prod, fn);
}

}  // namespace rqb
