// k_join.cu — joins::semi_join_mask (join.cpp:368-406) on encoded columns,
// the first §8f-row-3 operator (the production queries' semi-joins).
//
// The reference views each side as hashable entries — one per run (RLE),
// point (Index) or row (Plain; composites through normalize_basic) — with
// keys in a common domain (any float side → f64 bits with −0 folded into +0,
// else int64, join.cpp:31-44), builds a chained hash table on the build side
// and marks every probe entry with at least one match. The mask keeps the
// probe's shape: the hit runs of an RLE probe (unmerged), a byte per row for
// a Plain probe, the hit positions otherwise.
//
// Here: one kernel maps both sides to 64-bit keys; the build side is
// inserted into an open-addressing table (power of two ≥ 2× entries, the
// reference's splitmix64 finaliser, linear probing; a slot is claimed with
// atomicCAS on its state word, duplicates may occupy several slots — a set
// only answers membership); one thread per probe entry walks its probe
// sequence; the hit flags are compacted by the existing ordered selects
// (select_runs / select_points), so entry order — and so the mask — is the
// reference's. Work is O(build + probe) entries: runs are never expanded.
#include "device_common.cuh"
#include "rq_internal.hpp"

namespace rqb {
namespace dev {

__device__ __forceinline__ uint64_t join_mix(uint64_t x) {  // splitmix64 finaliser (join.cpp:46-52)
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void k_join_keys(const void* __restrict__ v, int dt, int64_t n, int as_float, uint64_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (as_float) {
      double x = ld_f64(v, dt, i);
      if (x == 0.0) x = 0.0;  // fold -0.0 into +0.0
      out[i] = static_cast<uint64_t>(__double_as_longlong(x));
    } else {
      out[i] = static_cast<uint64_t>(ld_i64(v, dt, i));
    }
  }
}

__global__ void k_hash_insert(const uint64_t* __restrict__ keys, int64_t n, unsigned long long* __restrict__ tkeys,
                              unsigned* __restrict__ tstate, uint64_t mask) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    uint64_t h = join_mix(k) & mask;
    while (atomicCAS(tstate + h, 0u, 1u) != 0u) h = (h + 1) & mask;
    tkeys[h] = k;
  }
}

__global__ void k_hash_probe(const uint64_t* __restrict__ keys, int64_t n, const unsigned long long* __restrict__ tkeys,
                             const unsigned* __restrict__ tstate, uint64_t mask, uint8_t* __restrict__ hit) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    uint64_t h = join_mix(k) & mask;
    uint8_t found = 0;
    while (__ldg(tstate + h)) {
      if (static_cast<uint64_t>(__ldg(tkeys + h)) == k) {
        found = 1;
        break;
      }
      h = (h + 1) & mask;
    }
    hit[i] = found;
  }
}

}  // namespace dev

namespace {

int grid_of(const CtxPtr& ctx, int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 16;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

struct Entries {  // JoinEntries (join.cpp:90-101)
  DArr values;
  bool is_rle = false;
  DArr s, e;  // is_rle
  DArr rows;  // otherwise (positions; empty for a plain column: rows are 0..n-1)
  bool plain_rows = false;
};

Entries entries_of(const CtxPtr& ctx, const DCol& c) {  // join.cpp:103-129
  Entries je;
  switch (c.enc) {
    case RQ_ENC_RLE:
      je.is_rle = true;
      je.values = c.v;
      je.s = c.s.n || c.e.n == 0 ? c.s : starts_from_ends(ctx, c.e);
      je.e = c.e;
      return je;
    case RQ_ENC_INDEX:
      je.values = c.v;
      je.rows = c.p;
      return je;
    case RQ_ENC_PLAIN:
      je.values = decode_plain(ctx, c);
      je.plain_rows = true;
      return je;
    default:
      return entries_of(ctx, normalize_basic(ctx, c));
  }
}

DArr join_keys(const CtxPtr& ctx, const DArr& v, bool as_float) {
  DArr k = alloc_arr(ctx, RQ_I64, v.n);
  if (v.n) {
    dev::k_join_keys<<<grid_of(ctx, v.n), 256, 0, ctx->stream>>>(v.raw(), v.dt, v.n, as_float ? 1 : 0,
                                                                  k.as<uint64_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  return k;
}

DMask make_mask_rle(DArr s, DArr e, int64_t total) {
  DMask m;
  m.enc = RQ_MASK_RLE;
  m.total = total;
  m.s = std::move(s);
  m.e = std::move(e);
  return m;
}

}  // namespace

DMask semi_join_mask(const CtxPtr& ctx, const DCol& probe, const DCol& build) {
  Entries pe = entries_of(ctx, probe);
  Entries be = entries_of(ctx, build);
  const bool as_float = dt_float(pe.values.dt) || dt_float(be.values.dt);
  KTimer timer(ctx, "semi_join");
  DArr pk = join_keys(ctx, pe.values, as_float);
  DArr bk = join_keys(ctx, be.values, as_float);
  // build: power-of-two table of at least twice the build entries (≥ 16)
  uint64_t cap = 16;
  while (cap < static_cast<uint64_t>(bk.n) * 2) cap <<= 1;
  DArr tkeys = alloc_arr(ctx, RQ_I64, static_cast<int64_t>(cap));
  DArr tstate = alloc_arr(ctx, RQ_I32, static_cast<int64_t>(cap));
  RQ_CUDA_CHECK(cudaMemsetAsync(tstate.raw_mut(), 0, cap * 4, ctx->stream));
  if (bk.n) {
    dev::k_hash_insert<<<grid_of(ctx, bk.n), 256, 0, ctx->stream>>>(
        bk.as<uint64_t>(), bk.n, tkeys.as<unsigned long long>(), tstate.as<unsigned>(), cap - 1);
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  DArr hit = alloc_arr(ctx, RQ_I8, std::max<int64_t>(1, pk.n));
  if (pk.n) {
    dev::k_hash_probe<<<grid_of(ctx, pk.n), 256, 0, ctx->stream>>>(
        pk.as<uint64_t>(), pk.n, tkeys.as<unsigned long long>(), tstate.as<unsigned>(), cap - 1,
        hit.as<uint8_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  hit.n = pk.n;
  const int64_t total = probe.total;
  if (pe.is_rle) {  // the hit runs, in run order (join.cpp:385-394)
    DArr s, e;
    select_runs(ctx, hit, pe.s, pe.e, s, e);
    return make_mask_rle(s, e, total);
  }
  if (probe.enc == RQ_ENC_PLAIN) {  // a byte per row (join.cpp:395-400)
    DMask m;
    m.enc = RQ_MASK_PLAIN;
    m.total = total;
    m.bits = hit;
    return m;
  }
  DArr rows = pe.plain_rows ? iota(ctx, pk.n) : pe.rows;  // hit positions (join.cpp:401-405)
  DArr p;
  select_points(ctx, hit, rows, p, nullptr);
  DMask m;
  m.enc = RQ_MASK_INDEX;
  m.total = total;
  m.p = p;
  return m;
}

}  // namespace rqb
