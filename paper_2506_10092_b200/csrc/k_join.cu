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
#include <algorithm>

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

// ---- get_join_index (join.cpp:183-238) ----
// build keys sorted (stable radix on the 64-bit key pattern) so the matches
// of a probe entry are one equal range, in build-entry order — the order of
// the reference's insertion-ordered hash chains.
__device__ __forceinline__ int64_t u64_lower(const uint64_t* a, int64_t n, uint64_t k) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(reinterpret_cast<const unsigned long long*>(a) + mid) < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t u64_upper(const uint64_t* a, int64_t n, uint64_t k) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(reinterpret_cast<const unsigned long long*>(a) + mid) <= k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_join_ranges(const uint64_t* __restrict__ pk, int64_t np, const uint64_t* __restrict__ bsorted,
                              int64_t nb, int64_t* __restrict__ lo, int64_t* __restrict__ cnt) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < np;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = pk[i];
    const int64_t l = u64_lower(bsorted, nb, k);
    lo[i] = l;
    cnt[i] = u64_upper(bsorted, nb, k) - l;
  }
}

struct JSide {  // one side's entries
  int is_rle;
  const int64_t* s;
  const int64_t* e;
  const int64_t* rows;  // null: plain rows (entry index = row)
};
__device__ __forceinline__ int64_t jlen(const JSide& x, int64_t i) {
  return x.is_rle ? ldg64(x.e, i) - ldg64(x.s, i) + 1 : 1;
}
__device__ __forceinline__ int64_t jrow(const JSide& x, int64_t i) { return x.rows ? ldg64(x.rows, i) : i; }

// per probe entry: its matches (p, b) in order, with each side's entry counts
__global__ void k_join_matches(const int64_t* __restrict__ lo, const int64_t* __restrict__ moff, int64_t np,
                               const int64_t* __restrict__ bidx, JSide P, JSide B, int64_t* __restrict__ mp,
                               int64_t* __restrict__ mb, int64_t* __restrict__ cp, int64_t* __restrict__ cb,
                               unsigned long long* __restrict__ card) {
  unsigned long long c = 0;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < np;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = moff[p], m = moff[p + 1] - o, l = lo[p];
    const int64_t lp = jlen(P, p);
    for (int64_t k = 0; k < m; ++k) {
      const int64_t b = ldg64(bidx, l + k);
      const int64_t lb = jlen(B, b);
      mp[o + k] = p;
      mb[o + k] = b;
      c += static_cast<unsigned long long>(lp * lb);
      if (!P.is_rle && !B.is_rle) {
        cp[o + k] = 1;
        cb[o + k] = 1;
      } else if (!P.is_rle) {  // one probe row repeated by the run length, one build range
        cp[o + k] = lb;
        cb[o + k] = 1;
      } else if (!B.is_rle) {  // one probe range, the build row repeated
        cp[o + k] = 1;
        cb[o + k] = lp;
      } else {  // build rows outer: lb probe ranges, lb·lp single-row build ranges
        cp[o + k] = lb;
        cb[o + k] = lb * lp;
      }
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(card, c);
}

// writes one side's join index entries for every match
__global__ void k_join_emit(const int64_t* __restrict__ mp, const int64_t* __restrict__ mb, int64_t nm,
                            const int64_t* __restrict__ off, JSide P, JSide B, int probe_side,
                            int64_t* __restrict__ rows, int64_t* __restrict__ v, int64_t* __restrict__ s,
                            int64_t* __restrict__ e) {
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < nm;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = mp[j], b = mb[j];
    const int64_t at = off[j];
    const int64_t lp = jlen(P, p), lb = jlen(B, b);
    if (probe_side) {
      if (!P.is_rle) {
        const int64_t r = jrow(P, p), n = B.is_rle ? lb : 1;
        for (int64_t k = 0; k < n; ++k) rows[at + k] = r;
      } else {
        const int64_t n = B.is_rle ? lb : 1, ps = ldg64(P.s, p), pe = ldg64(P.e, p);
        for (int64_t k = 0; k < n; ++k) {
          v[at + k] = p;
          s[at + k] = ps;
          e[at + k] = pe;
        }
      }
    } else {
      if (!B.is_rle) {
        const int64_t r = jrow(B, b), n = P.is_rle ? lp : 1;
        for (int64_t k = 0; k < n; ++k) rows[at + k] = r;
      } else if (!P.is_rle) {
        v[at] = b;
        s[at] = ldg64(B.s, b);
        e[at] = ldg64(B.e, b);
      } else {
        const int64_t bs = ldg64(B.s, b);
        for (int64_t k = 0; k < lb * lp; ++k) {
          const int64_t row = bs + k / lp;
          v[at + k] = b;
          s[at + k] = row;
          e[at + k] = row;
        }
      }
    }
  }
}

// ---- apply_join_index (join.cpp:245-362) ----
__global__ void k_xg_lengths_join(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t n,
                                  int64_t* __restrict__ len) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    len[i] = ldg64(e, i) - ldg64(s, i) + 1;
}
// index join into an RLE column: the run holding each referenced row
__global__ void k_join_run_of(const int64_t* __restrict__ rows, const int64_t* __restrict__ bin, int64_t n,
                              const int64_t* __restrict__ e, const int64_t* __restrict__ p, int64_t* __restrict__ at,
                              int* __restrict__ err) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = bin[i] - 1, r = rows[i];
    const bool ok = b >= 0 && (e ? r <= ldg64(e, b) : ldg64(p, b) == r);
    if (!ok) atomicOr(err, 1);
    at[i] = ok ? b : 0;
  }
}

// RLE join into an RLE column: fragment counts per reference range, with
// the coverage checks of apply_rle_join (start inside a run, no gap inside)
__global__ void k_join_frag_count(const int64_t* __restrict__ qs, const int64_t* __restrict__ qe, int64_t nq,
                                  const int64_t* __restrict__ cs, const int64_t* __restrict__ ce, int64_t nr,
                                  const int64_t* __restrict__ gaps, int64_t* __restrict__ r0, int64_t* __restrict__ cnt,
                                  int* __restrict__ err) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nq;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = qs[k], e = qe[k];
    const int64_t a = upper_bound_g(cs, nr, s) - 1;  // run with start <= s
    const int64_t b = upper_bound_g(cs, nr, e) - 1;
    bool ok = a >= 0 && s <= ldg64(ce, a) && ldg64(ce, b) >= e && ldg64(gaps, b) == ldg64(gaps, a);
    if (!ok) atomicOr(err, 1);
    r0[k] = ok ? a : 0;
    cnt[k] = ok ? b - a + 1 : 0;
  }
}
__global__ void k_join_frag_emit(const int64_t* __restrict__ qs, const int64_t* __restrict__ qe, int64_t nq,
                                 const int64_t* __restrict__ at_rows, const int64_t* __restrict__ r0,
                                 const int64_t* __restrict__ foff, const int64_t* __restrict__ cs,
                                 const int64_t* __restrict__ ce, int64_t* __restrict__ os, int64_t* __restrict__ oe,
                                 int64_t* __restrict__ src) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nq;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = qs[k], e = qe[k], o = foff[k], n = foff[k + 1] - o;
    int64_t at = at_rows[k], pos = s;
    for (int64_t f = 0; f < n; ++f) {
      const int64_t r = r0[k] + f;
      const int64_t fe = min(e, ldg64(ce, r));
      os[o + f] = at;
      oe[o + f] = at + (fe - pos);
      src[o + f] = r;
      at += fe - pos + 1;
      pos = fe + 1;
    }
    (void)cs;
  }
}
// gap flags of a run list: gaps[r] = number of runs r' <= r starting after e[r'-1] + 1
__global__ void k_gap_flags(const int64_t* __restrict__ s, const int64_t* __restrict__ e, int64_t n,
                            int64_t* __restrict__ flag) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flag[i] = (i > 0 && ldg64(s, i) > ldg64(e, i - 1) + 1) ? 1 : 0;
}
// RLE join into an Index column: points inside each reference range
__global__ void k_join_pts_count(const int64_t* __restrict__ qs, const int64_t* __restrict__ qe, int64_t nq,
                                 const int64_t* __restrict__ p, int64_t np, int64_t* __restrict__ lo,
                                 int64_t* __restrict__ cnt) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nq;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = lower_bound_g(p, np, qs[k]);
    lo[k] = a;
    cnt[k] = upper_bound_g(p, np, qe[k]) - a;
  }
}
__global__ void k_join_pts_emit(const int64_t* __restrict__ qs, int64_t nq, const int64_t* __restrict__ at_rows,
                                const int64_t* __restrict__ lo, const int64_t* __restrict__ poff,
                                const int64_t* __restrict__ p, int64_t* __restrict__ op, int64_t* __restrict__ take) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nq;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = poff[k], n = poff[k + 1] - o, a = lo[k], s = qs[k], at = at_rows[k];
    for (int64_t f = 0; f < n; ++f) {
      op[o + f] = at + (ldg64(p, a + f) - s);
      take[o + f] = a + f;
    }
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


// joins::get_join_index (join.cpp:183-238)
JoinResultD get_join_index(const CtxPtr& ctx, const DCol& left, const DCol& right) {
  Entries le = entries_of(ctx, left);
  Entries re = entries_of(ctx, right);
  const bool build_right = re.values.n <= le.values.n;  // ties: the left side probes
  Entries& be = build_right ? re : le;
  Entries& pe = build_right ? le : re;
  const bool as_float = dt_float(le.values.dt) || dt_float(re.values.dt);
  KTimer timer(ctx, "join_index");
  DArr pk = join_keys(ctx, pe.values, as_float);
  DArr bk = join_keys(ctx, be.values, as_float);
  DArr bidx = iota(ctx, bk.n);
  if (bk.n > 1) radix_sort_pairs(ctx, bk, bidx, 64, 0);  // stable: equal keys keep build order
  const int64_t np = pk.n;
  DArr lo = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, np));
  DArr cnt = alloc_arr(ctx, RQ_I64, np + 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(cnt.raw_mut(), 0, (np + 1) * 8, ctx->stream));
  if (np) {
    dev::k_join_ranges<<<grid_of(ctx, np), 256, 0, ctx->stream>>>(pk.as<uint64_t>(), np, bk.as<uint64_t>(), bk.n,
                                                                   lo.as<int64_t>(), cnt.as<int64_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  DArr moff;
  scan_exclusive_i64(ctx, cnt, moff);  // np + 1 entries: moff[np] = matches
  const int64_t nm = np ? ctx->readback(moff.as<int64_t>() + np, 8)[0] : 0;
  dev::JSide P{pe.is_rle ? 1 : 0, pe.s.pos(), pe.e.pos(), pe.plain_rows ? nullptr : pe.rows.pos()};
  dev::JSide B{be.is_rle ? 1 : 0, be.s.pos(), be.e.pos(), be.plain_rows ? nullptr : be.rows.pos()};
  DArr mp = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, nm)), mb = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, nm));
  DArr cp = alloc_arr(ctx, RQ_I64, nm + 1), cb = alloc_arr(ctx, RQ_I64, nm + 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(cp.raw_mut(), 0, (nm + 1) * 8, ctx->stream));
  RQ_CUDA_CHECK(cudaMemsetAsync(cb.raw_mut(), 0, (nm + 1) * 8, ctx->stream));
  DArr card = alloc_arr(ctx, RQ_I64, 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(card.raw_mut(), 0, 8, ctx->stream));
  if (np) {
    dev::k_join_matches<<<grid_of(ctx, np), 256, 0, ctx->stream>>>(
        lo.pos(), moff.pos(), np, bidx.pos(), P, B, mp.as<int64_t>(), mb.as<int64_t>(), cp.as<int64_t>(),
        cb.as<int64_t>(), card.as<unsigned long long>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  JoinResultD out;
  out.cardinality = ctx->readback(card.raw(), 8)[0];
  auto emit = [&](int probe_side, const DArr& c, bool is_rle) {
    DArr off;
    scan_exclusive_i64(ctx, c, off);
    const int64_t n = ctx->readback(off.as<int64_t>() + nm, 8)[0];
    JoinSideD js;
    js.is_rle = is_rle;
    if (is_rle) {
      js.v = alloc_arr(ctx, RQ_I64, n);
      js.s = alloc_arr(ctx, RQ_I64, n);
      js.e = alloc_arr(ctx, RQ_I64, n);
    } else {
      js.rows = alloc_arr(ctx, RQ_I64, n);
    }
    if (nm) {
      dev::k_join_emit<<<grid_of(ctx, nm), 256, 0, ctx->stream>>>(
          mp.pos(), mb.pos(), nm, off.pos(), P, B, probe_side, is_rle ? nullptr : js.rows.as<int64_t>(),
          is_rle ? js.v.as<int64_t>() : nullptr, is_rle ? js.s.as<int64_t>() : nullptr,
          is_rle ? js.e.as<int64_t>() : nullptr);
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
    }
    return js;
  };
  JoinSideD po = emit(1, cp, pe.is_rle);
  JoinSideD bo = emit(0, cb, be.is_rle);
  out.left = build_right ? po : bo;
  out.right = build_right ? bo : po;
  return out;
}


namespace {

DCol plain_of(DArr values) {
  DCol c;
  c.enc = RQ_ENC_PLAIN;
  c.total = values.n;
  c.logical = values.dt;
  c.v = std::move(values);
  return c;
}

int64_t readback_i64(const CtxPtr& ctx, const DArr& a, int64_t i) { return ctx->readback(a.as<int64_t>() + i, 8)[0]; }

void check_err(const CtxPtr& ctx, const DArr& err, const char* msg) {
  if (ctx->readback(err.raw(), 8)[0] & 0xffffffff) fail(msg);
}

DArr decoded(const CtxPtr& ctx, const DCol& c) {  // decode_full of a plain-shaped column
  return c.enc == RQ_ENC_PLAIN ? decode_plain(ctx, c) : decode_plain_index(ctx, c);
}

DArr starts_of(const CtxPtr& ctx, const DCol& c) {
  return c.s.n || c.e.n == 0 ? c.s : starts_from_ends(ctx, c.e);
}

}  // namespace

// joins::apply_join_index (join.cpp:245-366)
DCol apply_join_index(const CtxPtr& ctx, const DCol& col, const JoinSideD& j) {
  if (col.enc == RQ_ENC_RLE_INDEX) return apply_join_index(ctx, normalize_basic(ctx, col), j);
  KTimer timer(ctx, "apply_join");
  DArr err = alloc_arr(ctx, RQ_I64, 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(err.raw_mut(), 0, 8, ctx->stream));
  if (!j.is_rle) {  // apply_index_join (join.cpp:247-282): a plain column of the referenced rows
    const DArr& rows = j.rows;
    if (col.enc == RQ_ENC_PLAIN || col.enc == RQ_ENC_PLAIN_INDEX) return plain_of(gather(ctx, decoded(ctx, col), rows));
    const bool rle = col.enc == RQ_ENC_RLE;
    DArr keys = rle ? starts_of(ctx, col) : col.p;
    DArr bin = bucketize(ctx, rows, keys, true);
    DArr at = alloc_arr(ctx, RQ_I64, rows.n);
    if (rows.n) {
      dev::k_join_run_of<<<grid_of(ctx, rows.n), 256, 0, ctx->stream>>>(
          rows.pos(), bin.pos(), rows.n, rle ? col.e.pos() : nullptr, rle ? nullptr : col.p.pos(), at.as<int64_t>(),
          reinterpret_cast<int*>(err.raw_mut()));
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
      check_err(ctx, err, "apply_join_index: reference outside covered rows");
    }
    return plain_of(gather(ctx, col.v, at));
  }
  // apply_rle_join (join.cpp:284-362)
  const int64_t nq = j.s.n;
  DArr lens_off;  // exclusive offsets of the reference ranges in output row space
  int64_t out_rows = 0;
  DArr len = alloc_arr(ctx, RQ_I64, nq + 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(len.raw_mut(), 0, (nq + 1) * 8, ctx->stream));
  if (nq) {
    dev::k_xg_lengths_join<<<grid_of(ctx, nq), 256, 0, ctx->stream>>>(j.s.pos(), j.e.pos(), nq, len.as<int64_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  scan_exclusive_i64(ctx, len, lens_off);
  out_rows = nq ? readback_i64(ctx, lens_off, nq) : 0;
  if (col.enc == RQ_ENC_PLAIN || col.enc == RQ_ENC_PLAIN_INDEX) {
    DArr flat;
    expand_runs(ctx, j.s, j.e, &flat, nullptr);
    return plain_of(gather(ctx, decoded(ctx, col), flat));
  }
  if (col.enc == RQ_ENC_RLE) {
    DArr cs = starts_of(ctx, col);
    const int64_t nr = col.e.n;
    DArr gflag = alloc_arr(ctx, RQ_I64, nr + 1), gaps;
    RQ_CUDA_CHECK(cudaMemsetAsync(gflag.raw_mut(), 0, (nr + 1) * 8, ctx->stream));
    if (nr) {
      dev::k_gap_flags<<<grid_of(ctx, nr), 256, 0, ctx->stream>>>(cs.pos(), col.e.pos(), nr, gflag.as<int64_t>());
      ctx->count_launch();
    }
    scan_exclusive_i64(ctx, gflag, gaps);
    // gaps[r + 1] - gaps[a + 1] counts the gaps between runs a and r: shift by one
    DArr r0 = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, nq)), cnt = alloc_arr(ctx, RQ_I64, nq + 1);
    RQ_CUDA_CHECK(cudaMemsetAsync(cnt.raw_mut(), 0, (nq + 1) * 8, ctx->stream));
    if (nq) {
      dev::k_join_frag_count<<<grid_of(ctx, nq), 256, 0, ctx->stream>>>(
          j.s.pos(), j.e.pos(), nq, cs.pos(), col.e.pos(), nr, gaps.pos() + 1, r0.as<int64_t>(), cnt.as<int64_t>(),
          reinterpret_cast<int*>(err.raw_mut()));
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
      check_err(ctx, err, "apply_join_index: range outside covered rows or across a coverage gap");
    }
    DArr foff;
    scan_exclusive_i64(ctx, cnt, foff);
    const int64_t nf = nq ? readback_i64(ctx, foff, nq) : 0;
    DArr os = alloc_arr(ctx, RQ_I64, nf), oe = alloc_arr(ctx, RQ_I64, nf), src = alloc_arr(ctx, RQ_I64, nf);
    if (nf) {
      dev::k_join_frag_emit<<<grid_of(ctx, nq), 256, 0, ctx->stream>>>(
          j.s.pos(), j.e.pos(), nq, lens_off.pos(), r0.pos(), foff.pos(), cs.pos(), col.e.pos(), os.as<int64_t>(),
          oe.as<int64_t>(), src.as<int64_t>());
      ctx->count_launch();
      RQ_CUDA_CHECK(cudaGetLastError());
    }
    DCol out;
    out.enc = RQ_ENC_RLE;
    out.total = out_rows;
    out.v = gather(ctx, col.v, src);
    out.s = os;
    out.e = oe;
    return out;
  }
  // Index column: points inside each range, at their offset in output row space
  DArr lo = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, nq)), cnt = alloc_arr(ctx, RQ_I64, nq + 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(cnt.raw_mut(), 0, (nq + 1) * 8, ctx->stream));
  if (nq) {
    dev::k_join_pts_count<<<grid_of(ctx, nq), 256, 0, ctx->stream>>>(j.s.pos(), j.e.pos(), nq, col.p.pos(), col.p.n,
                                                                      lo.as<int64_t>(), cnt.as<int64_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  DArr poff;
  scan_exclusive_i64(ctx, cnt, poff);
  const int64_t npts = nq ? readback_i64(ctx, poff, nq) : 0;
  DArr op = alloc_arr(ctx, RQ_I64, npts), take = alloc_arr(ctx, RQ_I64, npts);
  if (npts) {
    dev::k_join_pts_emit<<<grid_of(ctx, nq), 256, 0, ctx->stream>>>(j.s.pos(), nq, lens_off.pos(), lo.pos(),
                                                                     poff.pos(), col.p.pos(), op.as<int64_t>(),
                                                                     take.as<int64_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  DCol out;
  out.enc = RQ_ENC_INDEX;
  out.total = out_rows;
  out.v = gather(ctx, col.v, take);
  out.p = op;
  return out;
}


// joins::hash_build_probe (join.cpp:167-181): matching (build, probe)
// positions of two value arrays, probe-major, build matches in entry order
void hash_build_probe(const CtxPtr& ctx, const DArr& build_values, const DArr& probe_values, DArr& build_pos,
                      DArr& probe_pos) {
  const bool as_float = dt_float(build_values.dt) || dt_float(probe_values.dt);
  KTimer timer(ctx, "hash_build_probe");
  DArr pk = join_keys(ctx, probe_values, as_float);
  DArr bk = join_keys(ctx, build_values, as_float);
  DArr bidx = iota(ctx, bk.n);
  if (bk.n > 1) radix_sort_pairs(ctx, bk, bidx, 64, 0);
  const int64_t np = pk.n;
  DArr lo = alloc_arr(ctx, RQ_I64, std::max<int64_t>(1, np));
  DArr cnt = alloc_arr(ctx, RQ_I64, np + 1);
  RQ_CUDA_CHECK(cudaMemsetAsync(cnt.raw_mut(), 0, (np + 1) * 8, ctx->stream));
  if (np) {
    dev::k_join_ranges<<<grid_of(ctx, np), 256, 0, ctx->stream>>>(pk.as<uint64_t>(), np, bk.as<uint64_t>(), bk.n,
                                                                   lo.as<int64_t>(), cnt.as<int64_t>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
  DArr moff;
  scan_exclusive_i64(ctx, cnt, moff);
  const int64_t nm = np ? ctx->readback(moff.as<int64_t>() + np, 8)[0] : 0;
  build_pos = alloc_arr(ctx, RQ_I64, nm);
  probe_pos = alloc_arr(ctx, RQ_I64, nm);
  if (nm) {
    const dev::JSide plain{0, nullptr, nullptr, nullptr};
    DArr cp = alloc_arr(ctx, RQ_I64, nm + 1), cb = alloc_arr(ctx, RQ_I64, nm + 1), card = alloc_arr(ctx, RQ_I64, 1);
    dev::k_join_matches<<<grid_of(ctx, np), 256, 0, ctx->stream>>>(
        lo.pos(), moff.pos(), np, bidx.pos(), plain, plain, probe_pos.as<int64_t>(), build_pos.as<int64_t>(),
        cp.as<int64_t>(), cb.as<int64_t>(), card.as<unsigned long long>());
    ctx->count_launch();
    RQ_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace rqb
