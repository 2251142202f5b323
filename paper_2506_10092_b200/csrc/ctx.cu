#include <chrono>
// ctx.cu — context, stream-ordered allocation, device arrays, column/mask
// upload/download and the handle half of the C ABI (include/runq_b200.h).
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "rq_internal.hpp"

namespace rqb {

int kernel_occupancy(int device, const void* fn, int block, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(fn, device, block, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (smem > 48 * 1024)
    RQ_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int occ = 0;
  RQ_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, smem));
  if (occ < 1) occ = 1;
  cache.emplace(key, occ);
  return occ;
}


namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void cuda_fail(cudaError_t err, const char* what, const char* file, int line) {
  int code = (err == cudaErrorMemoryAllocation) ? RQ_RESOURCE : RQ_CUDA;
  cudaGetLastError();  // clear sticky-free errors
  throw RqError(code, std::string("CUDA error ") + cudaGetErrorName(err) + " (" +
                          cudaGetErrorString(err) + ") at " + file + ":" + std::to_string(line) +
                          ": " + what);
}

cudaEvent_t Ctx::get_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  RQ_CUDA_CHECK(cudaEventCreate(&e));
  return e;
}

void Ctx::collect_profile() {
  while (!graph_timers_unread.empty()) read_graph_timer(graph_timers_unread.front().a);
  if (pending.empty()) return;
  RQ_CUDA_CHECK(cudaStreamSynchronize(stream));
  for (auto& p : pending) {
    float ms = 0;
    RQ_CUDA_CHECK(cudaEventElapsedTime(&ms, p.a, p.b));
    bool found = false;
    for (auto& kv : kstats) {
      if (kv.first == p.tag) {
        kv.second.ms += ms;
        kv.second.count += 1;
        found = true;
        break;
      }
    }
    if (!found) kstats.push_back({p.tag, KStat{ms, 1}});
    event_pool.push_back(p.a);
    event_pool.push_back(p.b);
  }
  pending.clear();
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  graph_timers_unread.clear();
  graphs.clear();  // their blocks go back through free() while the cache is alive
  for (auto& kv : block_cache)
    for (void* p : kv.second) cudaFree(p);
  for (auto& p : pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : event_pool) cudaEventDestroy(e);
  if (tile_status) cudaFree(tile_status);
  if (scratch) cudaFree(scratch);
  if (tickets) cudaFree(tickets);
  if (pinned) cudaFreeHost(pinned);
  if (stream) cudaStreamDestroy(stream);
}

// Size classes of the context's block cache: powers of two up to 4 KB, then
// eight steps per power of two (<= 12.5% slack).
static size_t size_class(size_t bytes) {
  size_t r = bytes < 256 ? 256 : bytes;
  if (r <= 4096) {
    size_t p = 256;
    while (p < r) p <<= 1;
    return p;
  }
  size_t p = size_t(1) << (63 - __builtin_clzll(r));
  const size_t step = p / 8;
  return (r + step - 1) / step * step;
}

// Blocks up to 64 MB are recycled through per-class free lists (at most 1 GB
// held): every use of a block is ordered on this context's one stream, so a
// block freed by one operator is safe to hand to the next launch at once —
// no cudaMallocAsync / cudaFreeAsync round trip per intermediate array.
void* Ctx::alloc(size_t bytes, size_t* cap) {
  if (bytes == 0) return nullptr;
  const size_t c = size_class(bytes);
  if (cap) *cap = c;
  if (c <= kCacheMaxBlock) {
    auto it = block_cache.find(c);
    if (it != block_cache.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      cached_bytes -= c;
      return p;
    }
  }
  void* p = nullptr;
  if (capturing) {  // no allocation node in the graph: a plain allocation, kept by the graph
    if (cudaMalloc(&p, c) != cudaSuccess) {
      cudaGetLastError();
      capture_broken = true;
      throw RqError(RQ_RESOURCE, "device allocation during graph capture failed");
    }
    return p;
  }
  cudaError_t err = cudaMallocAsync(&p, c, stream);
  if (err != cudaSuccess) {  // give the cached blocks back and retry once
    cudaGetLastError();
    release_cache();
    err = cudaMallocAsync(&p, c, stream);
  }
  if (err != cudaSuccess) {
    cudaGetLastError();
    throw RqError(RQ_RESOURCE, "device allocation of " + std::to_string(bytes) +
                                   " bytes failed: " + cudaGetErrorString(err));
  }
  return p;
}

void Ctx::free(void* p, size_t cap) {
  if (!p) return;
  if (capturing) {  // a captured kernel may still use it on every replay
    capture_owned.push_back({p, cap});
    return;
  }
  if (cap && cap <= kCacheMaxBlock && cached_bytes + cap <= kCacheMaxBytes) {
    block_cache[cap].push_back(p);
    cached_bytes += cap;
    return;
  }
  cudaSetDevice(device);
  cudaFreeAsync(p, stream);
}

void Ctx::release_cache() {
  for (auto& kv : block_cache)
    for (void* p : kv.second) cudaFreeAsync(p, stream);
  block_cache.clear();
  cached_bytes = 0;
  cudaStreamSynchronize(stream);
}

// Stream synchronisation; under profiling its host wall time is recorded as
// the pseudo-tag "host_sync_wait" (time the host spent blocked on the GPU).
void Ctx::wait_stream() {
  if (capturing) {  // a plan that syncs cannot be captured: the caller runs it uncaptured
    capture_broken = true;
    throw RqError(RQ_CUDA, "stream sync during graph capture");
  }
  if (!profiling) {
    RQ_CUDA_CHECK(cudaStreamSynchronize(stream));
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  RQ_CUDA_CHECK(cudaStreamSynchronize(stream));
  add_host_stat("host_sync_wait",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
}

void Ctx::sync() { wait_stream(); }

const int64_t* Ctx::readback(const void* dev, size_t bytes) {
  if (bytes > 4096) fail("readback too large");
  RQ_CUDA_CHECK(cudaMemcpyAsync(pinned, dev, bytes, cudaMemcpyDeviceToHost, stream));
  wait_stream();
  return pinned;
}

uint32_t Ctx::next_epoch(int64_t tiles) {
  if (tiles + 1 > tile_status_cap) {
    if (tile_status) {
      RQ_CUDA_CHECK(cudaStreamSynchronize(stream));
      cudaFree(tile_status);
      tile_status = nullptr;
    }
    int64_t cap = tiles + 1 < 4096 ? 4096 : (tiles + 1) * 2;
    RQ_CUDA_CHECK(cudaMalloc(&tile_status, static_cast<size_t>(cap) * 8));
    RQ_CUDA_CHECK(cudaMemsetAsync(tile_status, 0, static_cast<size_t>(cap) * 8, stream));
    tile_status_cap = cap;
    epoch = 0;
  }
  epoch = (epoch + 1) & 0x3fffff;
  if (epoch == 0) {  // wrapped: old tags could alias; clear once
    RQ_CUDA_CHECK(cudaMemsetAsync(tile_status, 0, static_cast<size_t>(tile_status_cap) * 8, stream));
    epoch = 1;
  }
  return epoch;
}

unsigned long long* Ctx::lookback_status(int64_t tiles, uint32_t* epoch_out) {
  if (!capturing) {
    *epoch_out = next_epoch(tiles);
    return tile_status;
  }
  const size_t bytes = static_cast<size_t>(tiles + 1) * 8;
  size_t cap = 0;
  void* p = alloc(bytes, &cap);
  capture_owned.push_back({p, cap});
  RQ_CUDA_CHECK(cudaMemsetAsync(p, 0, bytes, stream));
  *epoch_out = 1;
  return static_cast<unsigned long long*>(p);
}

void Ctx::read_graph_timer(cudaEvent_t a) {
  for (size_t i = 0; i < graph_timers_unread.size(); ++i) {
    const CapTimer t = graph_timers_unread[i];
    if (t.a != a) continue;
    RQ_CUDA_CHECK(cudaEventSynchronize(t.b));
    float ms = 0;
    RQ_CUDA_CHECK(cudaEventElapsedTime(&ms, t.a, t.b));
    add_host_stat(t.tag, ms);  // (tag, ms, +1 launch) like a pending pair
    graph_timers_unread.erase(graph_timers_unread.begin() + static_cast<std::ptrdiff_t>(i));
    return;
  }
}

void Ctx::drop_graphs() {
  if (graphs.empty()) return;
  RQ_CUDA_CHECK(cudaStreamSynchronize(stream));
  collect_profile();  // reads the graphs' unread timers before their events go
  graphs.clear();
}

void* Ctx::get_scratch(size_t bytes) {
  if (capturing) {
    capture_broken = true;
    throw RqError(RQ_CUDA, "scratch resize during graph capture");
  }
  if (bytes > scratch_bytes) {
    if (scratch) {
      RQ_CUDA_CHECK(cudaStreamSynchronize(stream));
      cudaFree(scratch);
      scratch = nullptr;
    }
    size_t cap = bytes < (1 << 20) ? (1 << 20) : bytes * 2;
    RQ_CUDA_CHECK(cudaMalloc(&scratch, cap));
    scratch_bytes = cap;
  }
  return scratch;
}

Buffer::~Buffer() {
  if (owned && ptr && ctx) {
    ctx->free(ptr, cap);
  }
}

DArr alloc_arr(const CtxPtr& ctx, int32_t dt, int64_t n) {
  require(dt_valid(dt), "invalid dtype");
  require(n >= 0, "negative array length");
  DArr a;
  a.dt = dt;
  a.n = n;
  if (n > 0) {
    auto b = std::make_shared<Buffer>();
    b->ctx = ctx;
    b->bytes = static_cast<size_t>(n) * dt_width(dt);
    b->ptr = ctx->alloc(b->bytes, &b->cap);
    a.buf = std::move(b);
  }
  return a;
}

DArr upload_arr(const CtxPtr& ctx, int32_t dt, const void* host, int64_t n) {
  DArr a = alloc_arr(ctx, dt, n);
  if (n > 0) {
    require(host != nullptr, "upload: null host pointer");
    RQ_CUDA_CHECK(cudaMemcpyAsync(a.raw_mut(), host, a.bytes(), cudaMemcpyHostToDevice, ctx->stream));
  }
  return a;
}

void download_arr(const CtxPtr& ctx, const DArr& a, void* host) {
  if (a.n == 0) return;
  require(host != nullptr, "download: null host pointer");
  RQ_CUDA_CHECK(cudaMemcpyAsync(host, a.raw(), a.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
}

DArr copy_prefix(const CtxPtr& ctx, const DArr& a, int64_t n) {
  DArr out = alloc_arr(ctx, a.dt, n);
  if (n > 0)
    RQ_CUDA_CHECK(cudaMemcpyAsync(out.raw_mut(), a.raw(), out.bytes(), cudaMemcpyDeviceToDevice,
                                  ctx->stream));
  return out;
}

}  // namespace rqb

using namespace rqb;

namespace {

CtxPtr get_ctx(rq_ctx_t c) {
  if (!c || !c->ctx) fail("null context");
  RQ_CUDA_CHECK(cudaSetDevice(c->ctx->device));
  return c->ctx;
}

const DArr& get_arr(rq_arr_t a) {
  if (!a) fail("null array handle");
  return a->a;
}

const DCol& get_col(rq_col_t c) {
  if (!c) fail("null column handle");
  return c->c;
}

const DMask& get_mask(rq_mask_t m) {
  if (!m) fail("null mask handle");
  return m->m;
}

DArr up_pos(const CtxPtr& ctx, const int64_t* p, int64_t n) { return upload_arr(ctx, RQ_I64, p, n); }

}  // namespace

extern "C" {

const char* rq_last_error(void) { return g_last_error.c_str(); }

const char* rq_version(void) {
  return "runq_b200 0.1 (sm_100a; compressed-execution path of arXiv 2506.10092)";
}

int rq_ctx_create(int device, rq_ctx_t* out) {
  return api_guard([&] {
    require(out != nullptr, "null out");
    int ndev = 0;
    RQ_CUDA_CHECK(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, "device ordinal out of range");
    RQ_CUDA_CHECK(cudaSetDevice(device));
    auto ctx = std::make_shared<Ctx>();
    ctx->device = device;
    RQ_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    cudaDeviceProp prop;
    RQ_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    ctx->sm_count = prop.multiProcessorCount;
    RQ_CUDA_CHECK(cudaHostAlloc(&ctx->pinned, 8192, cudaHostAllocMapped));
    ctx->result_host = reinterpret_cast<char*>(ctx->pinned) + 4096;
    RQ_CUDA_CHECK(cudaHostGetDevicePointer(&ctx->result_dev, ctx->result_host, 0));
    RQ_CUDA_CHECK(cudaMalloc(&ctx->tickets, 256));
    RQ_CUDA_CHECK(cudaMemsetAsync(ctx->tickets, 0, 256, ctx->stream));
    // keep freed blocks cached in the stream-ordered pool (no trim between ops)
    cudaMemPool_t pool;
    RQ_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    RQ_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    *out = new rq_ctx_s{ctx};
  });
}

int rq_ctx_destroy(rq_ctx_t ctx) {
  return api_guard([&] { delete ctx; });
}

int rq_ctx_synchronize(rq_ctx_t c) {
  return api_guard([&] { get_ctx(c)->sync(); });
}

void* rq_ctx_stream(rq_ctx_t c) { return (c && c->ctx) ? c->ctx->stream : nullptr; }

int64_t rq_ctx_launches(rq_ctx_t c) { return (c && c->ctx) ? c->ctx->launches : -1; }

int rq_ctx_set_profiling(rq_ctx_t c, int32_t enable) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    ctx->collect_profile();
    ctx->profiling = enable != 0;
  });
}

int rq_ctx_profile_only(rq_ctx_t c, const char* tags) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    ctx->collect_profile();
    ctx->profile_only.clear();
    std::string cur;
    for (const char* q = tags ? tags : ""; ; ++q) {
      if (*q == ',' || *q == 0) {
        if (!cur.empty()) ctx->profile_only.push_back(cur);
        cur.clear();
        if (*q == 0) break;
      } else {
        cur += *q;
      }
    }
  });
}

int rq_ctx_profile_report(rq_ctx_t c, int32_t reset, char* buf, int64_t cap) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    ctx->collect_profile();
    std::string out = "{";
    bool first = true;
    for (auto& kv : ctx->kstats) {
      if (!first) out += ",";
      first = false;
      out += "\"" + kv.first + "\":{\"ms\":" + std::to_string(kv.second.ms) +
             ",\"count\":" + std::to_string(kv.second.count) + "}";
    }
    out += "}";
    if (reset) ctx->kstats.clear();
    require(buf != nullptr && cap > static_cast<int64_t>(out.size()), "profile report buffer too small");
    std::memcpy(buf, out.c_str(), out.size() + 1);
  });
}

// ---- arrays ---------------------------------------------------------------------

int rq_arr_upload(rq_ctx_t c, int32_t dtype, const void* host, int64_t n, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    *out = wrap_arr(upload_arr(ctx, dtype, host, n));
  });
}

int rq_arr_alloc(rq_ctx_t c, int32_t dtype, int64_t n, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    require(dt_valid(dtype), "invalid dtype");
    require(n >= 0, "rq_arr_alloc: negative size");
    *out = wrap_arr(alloc_arr(ctx, dtype, n));
  });
}

int rq_arr_write(rq_ctx_t c, rq_arr_t a, int64_t offset, const void* host, int64_t count) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    require(a != nullptr, "rq_arr_write: null array");
    DArr& x = a->a;
    require(offset >= 0 && count >= 0 && offset + count <= x.n, "rq_arr_write: range outside the array");
    if (count == 0) return;
    require(host != nullptr, "rq_arr_write: null host pointer");
    size_t w = dt_width(x.dt);
    RQ_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(x.raw_mut()) + static_cast<size_t>(offset) * w, host,
                                  static_cast<size_t>(count) * w, cudaMemcpyHostToDevice, ctx->stream));
  });
}

int rq_arr_wrap_device(rq_ctx_t c, int32_t dtype, void* dev, int64_t n, rq_arr_t* out) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    require(dt_valid(dtype), "invalid dtype");
    DArr a;
    a.dt = dtype;
    a.n = n;
    if (n > 0) {
      auto b = std::make_shared<Buffer>();
      b->ctx = ctx;
      b->ptr = dev;
      b->bytes = static_cast<size_t>(n) * dt_width(dtype);
      b->cap = b->bytes;
      b->owned = false;
      a.buf = std::move(b);
    }
    *out = wrap_arr(std::move(a));
  });
}

int rq_arr_info(rq_arr_t a, int32_t* dtype, int64_t* n) {
  return api_guard([&] {
    const DArr& x = get_arr(a);
    if (dtype) *dtype = x.dt;
    if (n) *n = x.n;
  });
}

void* rq_arr_device_ptr(rq_arr_t a) { return a ? a->a.raw_mut() : nullptr; }

int rq_arr_download(rq_ctx_t c, rq_arr_t a, void* host) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    download_arr(ctx, get_arr(a), host);
    ctx->sync();
  });
}

int rq_arr_download_many(rq_ctx_t c, int32_t n, const rq_arr_t* arrs, void* const* hosts) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    for (int32_t i = 0; i < n; ++i) download_arr(ctx, get_arr(arrs[i]), hosts[i]);
    ctx->sync();  // one synchronisation for the whole result set
  });
}

int rq_arr_free(rq_arr_t a) {
  return api_guard([&] { delete a; });
}

// ---- columns ----------------------------------------------------------------------

int rq_col_upload(rq_ctx_t c, const rq_host_column* h, rq_col_t* out) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    require(h != nullptr && out != nullptr, "null argument");
    DCol col;
    col.enc = h->encoding;
    col.total = h->total_size;
    switch (h->encoding) {
      case RQ_ENC_PLAIN:
        require(dt_valid(h->dtype) && dt_valid(h->logical), "invalid dtype");
        col.v = upload_arr(ctx, h->dtype, h->v, h->n);
        col.logical = h->logical;
        col.has_center = h->has_center != 0;
        col.center = h->center;
        col.total = h->n;
        break;
      case RQ_ENC_RLE:
        col.v = upload_arr(ctx, h->dtype, h->v, h->n);
        col.e = up_pos(ctx, h->e, h->n);
        if (h->s == nullptr && h->n > 0) {  // gapless: starts implied by the ends
          col.s = starts_from_ends(ctx, col.e);
          col.gapless = 1;
        } else {
          col.s = up_pos(ctx, h->s, h->n);
        }
        col.logical = h->dtype;
        break;
      case RQ_ENC_INDEX:
        col.v = upload_arr(ctx, h->dtype, h->v, h->n);
        col.p = up_pos(ctx, h->p, h->n);
        col.logical = h->dtype;
        break;
      case RQ_ENC_PLAIN_INDEX:
        col.v = upload_arr(ctx, h->dtype, h->v, h->n);
        col.logical = h->logical;
        col.has_center = h->has_center != 0;
        col.center = h->center;
        col.total = h->n;
        col.v2 = upload_arr(ctx, h->dtype2, h->v2, h->n2);
        col.p2 = up_pos(ctx, h->p2, h->n2);
        break;
      case RQ_ENC_RLE_INDEX:
        col.v = upload_arr(ctx, h->dtype, h->v, h->n);
        col.s = up_pos(ctx, h->s, h->n);
        col.e = up_pos(ctx, h->e, h->n);
        col.logical = h->dtype;
        col.v2 = upload_arr(ctx, h->dtype2, h->v2, h->n2);
        col.p2 = up_pos(ctx, h->p2, h->n2);
        break;
      default:
        fail("unknown encoding");
    }
    *out = wrap_col(std::move(col));
  });
}

int rq_col_describe(rq_col_t c, rq_host_column* h) {
  return api_guard([&] {
    const DCol& col = get_col(c);
    std::memset(h, 0, sizeof(*h));
    h->encoding = col.enc;
    h->total_size = col.total;
    h->dtype = col.v.dt;
    h->logical = (col.enc == RQ_ENC_PLAIN || col.enc == RQ_ENC_PLAIN_INDEX) ? col.logical : col.v.dt;
    h->has_center = col.has_center;
    h->center = col.center;
    h->n = (col.enc == RQ_ENC_RLE || col.enc == RQ_ENC_RLE_INDEX) ? col.s.n
           : (col.enc == RQ_ENC_INDEX)                             ? col.p.n
                                                                   : col.v.n;
    if (col.enc == RQ_ENC_PLAIN_INDEX || col.enc == RQ_ENC_RLE_INDEX) {
      h->dtype2 = col.v2.dt;
      h->n2 = col.p2.n;
    }
  });
}

int rq_col_download(rq_ctx_t c, rq_col_t col_h, rq_host_column* h) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    const DCol& col = get_col(col_h);
    download_arr(ctx, col.v, h->v);
    if (col.enc == RQ_ENC_RLE || col.enc == RQ_ENC_RLE_INDEX) {
      download_arr(ctx, col.s, h->s);
      download_arr(ctx, col.e, h->e);
    }
    if (col.enc == RQ_ENC_INDEX) download_arr(ctx, col.p, h->p);
    if (col.enc == RQ_ENC_PLAIN_INDEX || col.enc == RQ_ENC_RLE_INDEX) {
      download_arr(ctx, col.v2, h->v2);
      download_arr(ctx, col.p2, h->p2);
    }
    ctx->sync();
  });
}

int rq_col_free(rq_col_t c) {
  return api_guard([&] { delete c; });
}

int rq_col_encoding(rq_col_t c) { return c ? c->c.enc : -1; }
int64_t rq_col_total_size(rq_col_t c) { return c ? c->c.total : -1; }
int rq_col_value_type(rq_col_t c) { return c ? c->c.value_type() : -1; }

int rq_col_make_rle(rq_ctx_t c, rq_arr_t v, rq_arr_t s, rq_arr_t e, int64_t total_size,
                    rq_col_t* out) {
  return api_guard([&] {
    get_ctx(c);
    DCol col;
    col.enc = RQ_ENC_RLE;
    col.total = total_size;
    col.v = get_arr(v);
    col.s = get_arr(s);
    col.e = get_arr(e);
    require(col.s.dt == RQ_I64 && col.e.dt == RQ_I64, "positions must be i64");
    require(col.v.n == col.s.n && col.s.n == col.e.n, "rle: length mismatch");
    col.logical = col.v.dt;
    *out = wrap_col(std::move(col));
  });
}

int rq_col_make_index(rq_ctx_t c, rq_arr_t v, rq_arr_t p, int64_t total_size, rq_col_t* out) {
  return api_guard([&] {
    get_ctx(c);
    DCol col;
    col.enc = RQ_ENC_INDEX;
    col.total = total_size;
    col.v = get_arr(v);
    col.p = get_arr(p);
    require(col.p.dt == RQ_I64, "positions must be i64");
    require(col.v.n == col.p.n, "index: length mismatch");
    col.logical = col.v.dt;
    *out = wrap_col(std::move(col));
  });
}

int rq_col_make_plain(rq_ctx_t c, rq_arr_t values, int32_t logical, int32_t has_center,
                      int64_t center, rq_col_t* out) {
  return api_guard([&] {
    get_ctx(c);
    DCol col;
    col.enc = RQ_ENC_PLAIN;
    col.v = get_arr(values);
    col.total = col.v.n;
    require(dt_valid(logical), "invalid logical dtype");
    col.logical = logical;
    col.has_center = has_center != 0;
    col.center = center;
    *out = wrap_col(std::move(col));
  });
}

int rq_col_part(rq_col_t c, int which, rq_arr_t* out) {
  return api_guard([&] {
    const DCol& col = get_col(c);
    const DArr* a = nullptr;
    switch (which) {
      case 0: a = &col.v; break;
      case 1: a = &col.s; break;
      case 2: a = &col.e; break;
      case 3: a = &col.p; break;
      case 4: a = &col.v2; break;
      case 5: a = &col.p2; break;
      default: fail("rq_col_part: bad part index");
    }
    *out = wrap_arr(*a);
  });
}

// ---- masks ----------------------------------------------------------------------------

int rq_mask_upload(rq_ctx_t c, const rq_host_mask* h, rq_mask_t* out) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    DMask m;
    m.enc = h->encoding;
    m.total = h->total_size;
    switch (h->encoding) {
      case RQ_MASK_PLAIN:
        m.bits = upload_arr(ctx, RQ_I8, h->bits, h->n);
        m.total = h->n;
        break;
      case RQ_MASK_RLE:
        m.s = up_pos(ctx, h->s, h->n);
        m.e = up_pos(ctx, h->e, h->n);
        break;
      case RQ_MASK_INDEX:
        m.p = up_pos(ctx, h->p, h->n);
        break;
      case RQ_MASK_COMPOSITE:
        m.s = up_pos(ctx, h->s, h->n);
        m.e = up_pos(ctx, h->e, h->n);
        m.p = up_pos(ctx, h->p2, h->n2);
        break;
      default:
        fail("unknown mask encoding");
    }
    *out = wrap_mask(std::move(m));
  });
}

int rq_mask_describe(rq_mask_t mh, rq_host_mask* h) {
  return api_guard([&] {
    const DMask& m = get_mask(mh);
    std::memset(h, 0, sizeof(*h));
    h->encoding = m.enc;
    h->total_size = m.total;
    switch (m.enc) {
      case RQ_MASK_PLAIN: h->n = m.bits.n; break;
      case RQ_MASK_RLE: h->n = m.s.n; break;
      case RQ_MASK_INDEX: h->n = m.p.n; break;
      default:
        h->n = m.s.n;
        h->n2 = m.p.n;
    }
  });
}

int rq_mask_download(rq_ctx_t c, rq_mask_t mh, rq_host_mask* h) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    const DMask& m = get_mask(mh);
    switch (m.enc) {
      case RQ_MASK_PLAIN: download_arr(ctx, m.bits, h->bits); break;
      case RQ_MASK_RLE:
        download_arr(ctx, m.s, h->s);
        download_arr(ctx, m.e, h->e);
        break;
      case RQ_MASK_INDEX: download_arr(ctx, m.p, h->p); break;
      default:
        download_arr(ctx, m.s, h->s);
        download_arr(ctx, m.e, h->e);
        download_arr(ctx, m.p, h->p2);
    }
    ctx->sync();
  });
}

int rq_mask_free(rq_mask_t m) {
  return api_guard([&] { delete m; });
}

int rq_mask_true_count(rq_ctx_t c, rq_mask_t m, int64_t* out) {
  return api_guard([&] {
    auto ctx = get_ctx(c);
    *out = mask_true_count(ctx, get_mask(m));
  });
}

}  // extern "C"
