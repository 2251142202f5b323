// comm.cu — row-range sharded execution over several GPUs.
//
// A table is cut by row range (rq_shard_host_column, cuts snapped to run
// boundaries); every rank runs the ordinary single-GPU path on its shard and
// the partial aggregates are combined with ONE collective:
//   * global aggregates (no keys): one grouped ncclAllReduce of 8-byte
//     partials (uint64 sums — int64 SUM/COUNT wrap exactly like the
//     reference's accumulators, groupby.cpp:82-89 — f64 sums, min / max);
//   * group tables: one ncclAllGather of fixed-capacity (key, partials)
//     packets, then a device merge that regroups the gathered rows with the
//     library's own group_aggregate (keys ascending, kernels.cpp:154-186):
//     SUM / COUNT partials summed, MIN / MAX re-reduced.
// AVG is carried as (SUM, COUNT) and recomputed after the merge as
// f64(sum) / count (groupby.cpp:103-106), never averaged. STD / VAR are not
// exact under a merge and are rejected.
//
// Transports: NCCL (libnccl.so.2 loaded on first use; the collectives run on
// the context stream, async errors polled with ncclCommGetAsyncError →
// RQ_NCCL) or a host callback that all-gathers host buffers (used to drive
// several ranks on ONE device in tests, where NCCL refuses duplicate GPUs).
// The reference is single-process: this file has no counterpart
// there.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <functional>
#include <mutex>

#include "rq_internal.hpp"

namespace rqb {

// ---- NCCL, resolved at run time ---------------------------------------------------

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp) api.why = std::string("NCCL symbol missing: ") + name;
      return fp != nullptr;
    };
    api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
             sym(api.CommDestroy, "ncclCommDestroy") && sym(api.CommAbort, "ncclCommAbort") &&
             sym(api.CommGetAsyncError, "ncclCommGetAsyncError") && sym(api.AllReduce, "ncclAllReduce") &&
             sym(api.AllGather, "ncclAllGather") && sym(api.GroupStart, "ncclGroupStart") &&
             sym(api.GroupEnd, "ncclGroupEnd") && sym(api.GetErrorString, "ncclGetErrorString");
  });
  if (!api.ok) fail(api.why, RQ_NCCL);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(std::string(what) + ": " + nccl().GetErrorString(r), RQ_NCCL);
}

}  // namespace

struct Comm {
  CtxPtr ctx;
  int nranks = 1, rank = 0;
  ncclComm_t nc = nullptr;
  rq_host_allgather_fn host_fn = nullptr;
  void* user = nullptr;
  ~Comm() {
    if (nc) nccl().CommDestroy(nc);
  }
  // polls the communicator after the stream has drained
  void check_async() {
    if (!nc) return;
    ncclResult_t st = ncclSuccess;
    nccl_check(nccl().CommGetAsyncError(nc, &st), "ncclCommGetAsyncError");
    nccl_check(st, "NCCL async error");
  }
};

// ---- exchange primitives (device buffers, context stream) ---------------------------

namespace {

enum PKind { P_SUM_U64, P_SUM_F64, P_MIN_I64, P_MAX_I64, P_MIN_F64, P_MAX_F64 };

struct RedBuf {
  void* dev;
  int64_t count;
  PKind kind;
};

// Every rank's `bytes` from `send` into recv[rank * bytes ...].
void allgather(Comm& cm, const void* send, size_t bytes, void* recv) {
  Ctx& c = *cm.ctx;
  if (cm.nc) {
    nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, cm.nc, c.stream), "ncclAllGather");
    return;
  }
  std::vector<char> hs(bytes), hr(bytes * static_cast<size_t>(cm.nranks));
  if (bytes) RQ_CUDA_CHECK(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, c.stream));
  c.wait_stream();
  int st = cm.host_fn(hs.data(), static_cast<int64_t>(bytes), hr.data(), cm.user);
  if (st != 0) fail("host allgather callback failed", RQ_NCCL);
  if (!hr.empty()) RQ_CUDA_CHECK(cudaMemcpyAsync(recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, c.stream));
  c.wait_stream();  // hr must outlive the copy
}

template <class T, class F>
void host_reduce(std::vector<char>& all, int nranks, int64_t count, void* out, F op) {
  T* o = static_cast<T*>(out);
  for (int64_t i = 0; i < count; ++i) {
    T acc = reinterpret_cast<const T*>(all.data())[i];
    for (int r = 1; r < nranks; ++r) acc = op(acc, reinterpret_cast<const T*>(all.data() + r * count * 8)[i]);
    o[i] = acc;
  }
}

// In-place grouped all-reduce of 8-byte partial buffers: ONE NCCL group.
void allreduce(Comm& cm, const std::vector<RedBuf>& bufs) {
  Ctx& c = *cm.ctx;
  if (cm.nc) {
    auto& N = nccl();
    nccl_check(N.GroupStart(), "ncclGroupStart");
    for (const RedBuf& b : bufs) {
      ncclDataType_t t = (b.kind == P_SUM_U64) ? ncclUint64
                         : (b.kind == P_MIN_I64 || b.kind == P_MAX_I64) ? ncclInt64
                                                                        : ncclFloat64;
      ncclRedOp_t op = (b.kind == P_MIN_I64 || b.kind == P_MIN_F64)   ? ncclMin
                       : (b.kind == P_MAX_I64 || b.kind == P_MAX_F64) ? ncclMax
                                                                      : ncclSum;
      nccl_check(N.AllReduce(b.dev, b.dev, static_cast<size_t>(b.count), t, op, cm.nc, c.stream), "ncclAllReduce");
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
    return;
  }
  // host transport: all-gather, then reduce in rank order (deterministic)
  for (const RedBuf& b : bufs) {
    const size_t bytes = static_cast<size_t>(b.count) * 8;
    std::vector<char> mine(bytes), all(bytes * static_cast<size_t>(cm.nranks)), out(bytes);
    RQ_CUDA_CHECK(cudaMemcpyAsync(mine.data(), b.dev, bytes, cudaMemcpyDeviceToHost, c.stream));
    c.wait_stream();
    if (cm.host_fn(mine.data(), static_cast<int64_t>(bytes), all.data(), cm.user) != 0)
      fail("host allgather callback failed", RQ_NCCL);
    switch (b.kind) {
      case P_SUM_U64: host_reduce<uint64_t>(all, cm.nranks, b.count, out.data(), [](uint64_t a, uint64_t x) { return a + x; }); break;
      case P_SUM_F64: host_reduce<double>(all, cm.nranks, b.count, out.data(), [](double a, double x) { return a + x; }); break;
      case P_MIN_I64: host_reduce<int64_t>(all, cm.nranks, b.count, out.data(), [](int64_t a, int64_t x) { return x < a ? x : a; }); break;
      case P_MAX_I64: host_reduce<int64_t>(all, cm.nranks, b.count, out.data(), [](int64_t a, int64_t x) { return x > a ? x : a; }); break;
      case P_MIN_F64: host_reduce<double>(all, cm.nranks, b.count, out.data(), [](double a, double x) { return x < a ? x : a; }); break;
      case P_MAX_F64: host_reduce<double>(all, cm.nranks, b.count, out.data(), [](double a, double x) { return x > a ? x : a; }); break;
    }
    RQ_CUDA_CHECK(cudaMemcpyAsync(b.dev, out.data(), bytes, cudaMemcpyHostToDevice, c.stream));
    c.wait_stream();
  }
}

PKind pkind(int fn, int32_t dt) {
  const bool f = dt_float(dt);
  switch (fn) {
    case RQ_MIN: return f ? P_MIN_F64 : P_MIN_I64;
    case RQ_MAX: return f ? P_MAX_F64 : P_MAX_I64;
    case RQ_COUNT: return P_SUM_U64;
    default: return f ? P_SUM_F64 : P_SUM_U64;
  }
}

// unpacks the gathered packets: column c of rank r's rows → dst[c][off_r + i]
struct UnpackArgs {
  static constexpr int kMaxCols = 32;
  long long* dst[kMaxCols];
};

__global__ void k_unpack_tables(const char* __restrict__ gathered, long long packet_bytes, int ncols, long long cap,
                                const long long* __restrict__ n_of, const long long* __restrict__ off_of, int nranks,
                                UnpackArgs a) {
  const long long per_rank = cap * ncols;
  const long long total = per_rank * nranks;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(t / per_rank);
    const long long rem = t - r * per_rank;
    const int c = static_cast<int>(rem / cap);
    const long long i = rem - c * cap;
    if (i >= n_of[r]) continue;
    const long long* col = reinterpret_cast<const long long*>(gathered + r * packet_bytes + 8) + c * cap;
    a.dst[c][off_of[r] + i] = col[i];
  }
}

DCol plain_of(const DArr& v) {
  DCol c;
  c.enc = RQ_ENC_PLAIN;
  c.total = v.n;
  c.v = v;
  c.logical = v.dt;
  return c;
}

}  // namespace

// Merges per-rank partial tables (SUM / COUNT / MIN / MAX per column, 8-byte
// values) into the global table on every rank.
GroupAggOut merge_group_tables(const CtxPtr& ctx, Comm& cm, const GroupAggOut& local,
                               const std::vector<int>& part_fns) {
  const size_t nk = local.keys.size(), nv = local.vals.size();
  require(nv == part_fns.size(), "merge: partial/function count mismatch");
  for (const DArr& v : local.vals) require(dt_width(v.dt) == 8, "merge: partials must be 8-byte values");
  Ctx& c = *ctx;
  if (nk == 0) {  // global aggregates: one grouped all-reduce, in place on copies
    GroupAggOut out;
    out.n_groups = 1;
    std::vector<RedBuf> bufs;
    for (size_t i = 0; i < nv; ++i) {
      out.vals.push_back(copy_prefix(ctx, local.vals[i], local.vals[i].n));
      bufs.push_back({out.vals.back().raw_mut(), out.vals.back().n, pkind(part_fns[i], local.vals[i].dt)});
    }
    allreduce(cm, bufs);
    c.wait_stream();
    cm.check_async();
    return out;
  }
  require(nk + nv <= static_cast<size_t>(UnpackArgs::kMaxCols), "merge: at most 32 key + value columns");
  // 1. capacity = max groups over ranks
  DArr cap_d = alloc_arr(ctx, RQ_I64, 1);
  RQ_CUDA_CHECK(cudaMemcpyAsync(cap_d.raw_mut(), &local.n_groups, 8, cudaMemcpyHostToDevice, c.stream));
  allreduce(cm, {{cap_d.raw_mut(), 1, P_MAX_I64}});
  const int64_t cap = *c.readback(cap_d.raw(), 8);
  cm.check_async();
  // 2. packet = [n][key columns widened to 8 B][value columns], cap rows each
  const int ncols = static_cast<int>(nk + nv);
  const size_t packet = 8 + static_cast<size_t>(cap) * ncols * 8;
  DArr send = alloc_arr(ctx, RQ_I8, static_cast<int64_t>(packet));
  DArr recv = alloc_arr(ctx, RQ_I8, static_cast<int64_t>(packet) * cm.nranks);
  RQ_CUDA_CHECK(cudaMemcpyAsync(send.raw_mut(), &local.n_groups, 8, cudaMemcpyHostToDevice, c.stream));
  std::vector<int32_t> key_dt(nk);
  std::vector<DArr> keep;
  for (int col = 0; col < ncols; ++col) {
    DArr v;
    if (static_cast<size_t>(col) < nk) {
      const DArr& k = local.keys[col];
      key_dt[col] = k.dt;
      v = cast_values(ctx, k, dt_float(k.dt) ? RQ_F64 : RQ_I64);
    } else {
      v = local.vals[col - nk];
    }
    if (local.n_groups > 0)
      RQ_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(send.raw_mut()) + 8 + static_cast<size_t>(col) * cap * 8,
                                    v.raw(), static_cast<size_t>(local.n_groups) * 8, cudaMemcpyDeviceToDevice,
                                    c.stream));
    keep.push_back(std::move(v));
  }
  // 3. ONE all-gather of the packets
  allgather(cm, send.raw(), packet, recv.raw_mut());
  // 4. per-rank row counts (one strided copy) → offsets
  std::vector<int64_t> n_of(cm.nranks), off_of(cm.nranks);
  RQ_CUDA_CHECK(cudaMemcpy2DAsync(c.pinned, 8, recv.raw(), packet, 8, cm.nranks, cudaMemcpyDeviceToHost, c.stream));
  c.wait_stream();
  cm.check_async();
  int64_t total = 0;
  for (int r = 0; r < cm.nranks; ++r) {
    n_of[r] = c.pinned[r];
    off_of[r] = total;
    total += n_of[r];
  }
  DArr meta = upload_arr(ctx, RQ_I64, n_of.data(), cm.nranks);
  DArr offs = upload_arr(ctx, RQ_I64, off_of.data(), cm.nranks);
  std::vector<DArr> cols(ncols);
  UnpackArgs ua{};
  for (int col = 0; col < ncols; ++col) {
    const int32_t dt = static_cast<size_t>(col) < nk ? (dt_float(key_dt[col]) ? RQ_F64 : RQ_I64)
                                                     : local.vals[col - nk].dt;
    cols[col] = alloc_arr(ctx, dt, total);
    ua.dst[col] = cols[col].as<long long>();
  }
  if (total > 0 && cap > 0) {
    const long long work = static_cast<long long>(cap) * ncols * cm.nranks;
    const int grid = static_cast<int>(std::min<long long>((work + 255) / 256, 4LL * c.sm_count));
    k_unpack_tables<<<grid, 256, 0, c.stream>>>(static_cast<const char*>(recv.raw()), static_cast<long long>(packet),
                                                ncols, cap, meta.as<long long>(), offs.as<long long>(), cm.nranks, ua);
    RQ_CUDA_CHECK(cudaGetLastError());
    c.count_launch();
  }
  // 5. regroup the gathered rows: keys ascending, partials re-reduced
  std::vector<DCol> kc, vc;
  for (size_t i = 0; i < nk; ++i) kc.push_back(plain_of(cols[i]));
  for (size_t i = 0; i < nv; ++i) vc.push_back(plain_of(cols[nk + i]));
  std::vector<const DCol*> kp, vp;
  for (auto& x : kc) kp.push_back(&x);
  for (auto& x : vc) vp.push_back(&x);
  std::vector<int> merge_fns;
  for (int f : part_fns) merge_fns.push_back(f == RQ_COUNT ? RQ_SUM : f);
  GroupAggOut out;
  if (total == 0) {
    out.n_groups = 0;
    for (size_t i = 0; i < nk; ++i) out.keys.push_back(alloc_arr(ctx, key_dt[i], 0));
    for (size_t i = 0; i < nv; ++i) out.vals.push_back(alloc_arr(ctx, local.vals[i].dt, 0));
    return out;
  }
  out = group_aggregate(ctx, kp, vp, merge_fns, false);
  for (size_t i = 0; i < nk; ++i) out.keys[i] = cast_values(ctx, out.keys[i], key_dt[i]);
  // a COUNT partial is int64 after its SUM merge; SUM / MIN / MAX keep their types
  return out;
}

// The partial form of a list of aggregate functions: AVG → (SUM, COUNT) of
// the same input; STD / VAR are not exact under a merge.
PartialPlan partial_plan(const std::vector<int>& fns, const std::function<bool(int, int)>& same_input) {
  PartialPlan p;
  // one partial per distinct (function, input); COUNT partials are all the
  // same — a GroupAgg aligns every input jointly (groupby.cpp:144-162), so
  // every input has the same rows per group
  auto find_or_add = [&](int fn, int src) {
    for (size_t j = 0; j < p.local_fns.size(); ++j)
      if (p.local_fns[j] == fn && (fn == RQ_COUNT || same_input(p.src[j], src))) return static_cast<int>(j);
    p.local_fns.push_back(fn);
    p.src.push_back(src);
    return static_cast<int>(p.local_fns.size() - 1);
  };
  for (size_t i = 0; i < fns.size(); ++i) {
    const int f = fns[i];
    require(f != RQ_STD && f != RQ_VAR, "sharded aggregation: STD / VAR do not merge exactly across shards");
    require(f >= RQ_SUM && f <= RQ_AVG, "aggregate: unknown function");
    p.sum_of.push_back(find_or_add(f == RQ_AVG ? RQ_SUM : f, static_cast<int>(i)));
    p.cnt_of.push_back(f == RQ_AVG ? find_or_add(RQ_COUNT, static_cast<int>(i)) : -1);
  }
  return p;
}

// merged partials → the original functions' outputs (AVG = f64(sum) / count)
GroupAggOut finalize(const CtxPtr& ctx, GroupAggOut merged, const std::vector<int>& fns, const PartialPlan& p) {
  GroupAggOut out;
  out.n_groups = merged.n_groups;
  out.keys = std::move(merged.keys);
  for (size_t i = 0; i < fns.size(); ++i) {
    const DArr& s = merged.vals[p.sum_of[i]];
    if (fns[i] != RQ_AVG) {
      out.vals.push_back(s);
      continue;
    }
    out.vals.push_back(arith_values(ctx, cast_values(ctx, s, RQ_F64), merged.vals[p.cnt_of[i]], RQ_DIV));
  }
  return out;
}

GroupAggOut sharded(const CtxPtr& ctx, Comm& cm, const std::vector<int>& fns,
                    const std::function<GroupAggOut(const PartialPlan&)>& local,
                    const std::function<bool(int, int)>& same_input) {
  PartialPlan p = partial_plan(fns, same_input ? same_input : [](int a, int b) { return a == b; });
  GroupAggOut part = local(p);
  return finalize(ctx, merge_group_tables(ctx, cm, part, p.local_fns), fns, p);
}

AggOut sharded_scalar(const CtxPtr& ctx, Comm& cm, int fn, const std::function<AggOut(int)>& local) {
  GroupAggOut r = sharded(ctx, cm, {fn}, [&](const PartialPlan& p) {
    GroupAggOut g;
    g.n_groups = 1;
    for (int f : p.local_fns) {
      AggOut a = local(f);
      int64_t bits;
      std::memcpy(&bits, a.dtype == RQ_F64 ? static_cast<const void*>(&a.f) : static_cast<const void*>(&a.i), 8);
      g.vals.push_back(upload_arr(ctx, a.dtype, &bits, 1));
    }
    return g;
  });
  const int64_t* h = ctx->readback(r.vals[0].raw(), 8);
  AggOut a;
  a.dtype = r.vals[0].dt;
  if (a.dtype == RQ_F64) std::memcpy(&a.f, h, 8);
  else a.i = h[0];
  return a;
}

}  // namespace rqb

using namespace rqb;

struct rq_comm_s {
  std::shared_ptr<Comm> c;
};

namespace rqb {
Comm& comm_of(rq_comm_t c) {
  require(c != nullptr && c->c != nullptr, "null communicator");
  return *c->c;
}
}  // namespace rqb

namespace {
CtxPtr get_ctx(rq_ctx_t c) {
  if (!c || !c->ctx) fail("null context");
  RQ_CUDA_CHECK(cudaSetDevice(c->ctx->device));
  return c->ctx;
}
const DArr& arr_of(rq_arr_t a) {
  if (!a) fail("null array handle");
  return a->a;
}
}  // namespace

extern "C" {

int rq_comm_unique_id(void* id, int64_t cap) {
  return api_guard([&] {
    require(id != nullptr && cap >= static_cast<int64_t>(sizeof(ncclUniqueId)), "rq_comm_unique_id: buffer < 128 B");
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int rq_comm_init_nccl(rq_ctx_t c, const void* id, int32_t nranks, int32_t rank, rq_comm_t* out) {
  return api_guard([&] {
    require(out != nullptr && id != nullptr, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "rq_comm_init_nccl: bad rank / size");
    auto cm = std::make_shared<Comm>();
    cm->ctx = get_ctx(c);
    cm->nranks = nranks;
    cm->rank = rank;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    RQ_CUDA_CHECK(cudaSetDevice(cm->ctx->device));
    nccl_check(nccl().CommInitRank(&cm->nc, nranks, u, rank), "ncclCommInitRank");
    *out = new rq_comm_s{cm};
  });
}

int rq_comm_init_host(rq_ctx_t c, int32_t nranks, int32_t rank, rq_host_allgather_fn fn, void* user,
                      rq_comm_t* out) {
  return api_guard([&] {
    require(out != nullptr && fn != nullptr, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "rq_comm_init_host: bad rank / size");
    auto cm = std::make_shared<Comm>();
    cm->ctx = get_ctx(c);
    cm->nranks = nranks;
    cm->rank = rank;
    cm->host_fn = fn;
    cm->user = user;
    *out = new rq_comm_s{cm};
  });
}

int rq_comm_info(rq_comm_t c, int32_t* nranks, int32_t* rank, int32_t* transport) {
  return api_guard([&] {
    Comm& cm = comm_of(c);
    if (nranks) *nranks = cm.nranks;
    if (rank) *rank = cm.rank;
    if (transport) *transport = cm.nc ? RQ_COMM_NCCL : RQ_COMM_HOST;
  });
}

int rq_comm_destroy(rq_comm_t c) {
  return api_guard([&] { delete c; });
}

int rq_merge_group_tables(rq_ctx_t c, rq_comm_t comm, const rq_arr_t* keys, int32_t n_keys, const rq_arr_t* parts,
                          const int32_t* part_fns, int32_t n_parts, int64_t n_groups, int64_t* out_groups,
                          rq_arr_t* out_keys, rq_arr_t* out_parts) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    GroupAggOut local;
    local.n_groups = n_groups;
    for (int i = 0; i < n_keys; ++i) local.keys.push_back(arr_of(keys[i]));
    std::vector<int> f;
    for (int i = 0; i < n_parts; ++i) {
      require(part_fns[i] >= RQ_SUM && part_fns[i] <= RQ_MAX, "merge: partials are SUM / COUNT / MIN / MAX");
      local.vals.push_back(arr_of(parts[i]));
      f.push_back(part_fns[i]);
    }
    for (auto& a : local.keys) require(a.n == n_groups, "merge: key length != n_groups");
    for (auto& a : local.vals) require(a.n == n_groups, "merge: partial length != n_groups");
    GroupAggOut r = merge_group_tables(ctx, comm_of(comm), local, f);
    if (out_groups) *out_groups = r.n_groups;
    for (int i = 0; i < n_keys; ++i) out_keys[i] = wrap_arr(r.keys[i]);
    for (int i = 0; i < n_parts; ++i) out_parts[i] = wrap_arr(r.vals[i]);
  });
}

}  // extern "C"
