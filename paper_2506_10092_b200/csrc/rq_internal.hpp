// rq_internal.hpp — host-side internals of the B200 compressed-execution
// library: device column model, context, allocation, error plumbing.
//
// Device layout: every column part is a separate
// structure-of-arrays device buffer (runq::Array / PosVec in the reference,
// array.hpp:16, column.hpp:22-76): values at their storage width, positions
// int64. Buffers are 256-B aligned (cudaMallocAsync) so kernels may issue
// 128-bit loads; buffers are reference counted so operators that keep an
// input's positions share them instead of copying (the reference copies,
// align.cpp:86-100).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/runq_b200.h"

namespace rqb {

// ---- errors -----------------------------------------------------------------

struct RqError : std::runtime_error {
  int code;
  RqError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(const std::string& msg, int code = RQ_INVALID) {
  throw RqError(code, msg);
}
inline void require(bool cond, const char* msg) {
  if (!cond) fail(msg);
}

void cuda_fail(cudaError_t err, const char* what, const char* file, int line);
#define RQ_CUDA_CHECK(x)                                          \
  do {                                                            \
    cudaError_t err__ = (x);                                      \
    if (err__ != cudaSuccess) ::rqb::cuda_fail(err__, #x, __FILE__, __LINE__); \
  } while (0)

// ---- dtypes (runq::DType, dtype.hpp:11-71) -------------------------------------

inline int dt_width(int32_t t) {
  switch (t) {
    case RQ_I8: return 1;
    case RQ_I16: return 2;
    case RQ_I32: return 4;
    case RQ_F32: return 4;
    default: return 8;
  }
}
inline bool dt_float(int32_t t) { return t == RQ_F32 || t == RQ_F64; }
inline bool dt_valid(int32_t t) { return t >= RQ_I8 && t <= RQ_F64; }
// dtype_promote (dtype.hpp:69-71)
inline int32_t dt_promote(int32_t a, int32_t b) {
  return (dt_float(a) || dt_float(b)) ? RQ_F64 : RQ_I64;
}

// ---- context -------------------------------------------------------------------

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  int64_t launches = 0;
  int64_t* pinned = nullptr;  // host-pinned readback slots
  // host-pinned slot kernels write their final result into directly
  // (device-visible alias of pinned + 2048 B): no copy launch per query
  void* result_host = nullptr;
  void* result_dev = nullptr;
  // decoupled look-back tile status (epoch-tagged, see device_common.cuh)
  unsigned long long* tile_status = nullptr;
  int64_t tile_status_cap = 0;
  uint32_t epoch = 0;
  // last-CTA-done ticket counters (zeroed once; every kernel using one
  // leaves it at 0 again via atomicInc wrap-around)
  unsigned* tickets = nullptr;
  // small device scratch for counters / reduction partials
  void* scratch = nullptr;
  size_t scratch_bytes = 0;

  // per-kernel CUDA-event timing (rq_ctx_set_profiling / rq_ctx_profile_report)
  bool profiling = false;
  struct Pending {
    std::string tag;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  struct KStat {
    double ms = 0;
    int64_t count = 0;
  };
  std::vector<std::pair<std::string, KStat>> kstats;
  cudaEvent_t get_event();
  // A size a select kernel writes straight into mapped pinned memory (one
  // slot, read right after the sync that follows the launch): no D2H copy.
  int64_t* count_slot_dev() const { return reinterpret_cast<int64_t*>(static_cast<char*>(result_dev) + 2048); }
  int64_t read_count_slot() {
    wait_stream();
    return *reinterpret_cast<volatile int64_t*>(static_cast<char*>(result_host) + 2048);
  }
  bool host_profiling = std::getenv("RQ_HOST_PROFILE") != nullptr;
  // tags the profile records (empty: every tag) — a timed loop that needs one
  // kernel's time pays two event records per step, not one pair per scope
  std::vector<std::string> profile_only;
  bool profile_wants(const char* tag) const {
    if (profile_only.empty()) return true;
    for (const auto& t : profile_only)
      if (t == tag) return true;
    return false;
  }
  void add_host_stat(const std::string& tag, double ms) {
    for (auto& kv : kstats)
      if (kv.first == tag) {
        kv.second.ms += ms;
        kv.second.count += 1;
        return;
      }
    kstats.push_back({tag, KStat{ms, 1}});
  }
  void wait_stream();
  void collect_profile();

  ~Ctx();
  void* alloc(size_t bytes, size_t* cap = nullptr);
  void free(void* p, size_t cap = 0);
  void release_cache();
  static constexpr size_t kCacheMaxBlock = size_t(64) << 20, kCacheMaxBytes = size_t(1) << 30;
  std::unordered_map<size_t, std::vector<void*>> block_cache;
  size_t cached_bytes = 0;
  void sync();
  // Copies `bytes` from device to the pinned slots and waits (one sync).
  const int64_t* readback(const void* dev, size_t bytes);
  // Ensures tile_status can hold `tiles` entries; returns the epoch to use.
  uint32_t next_epoch(int64_t tiles);
  // Look-back status words for a launch of `tiles` tiles: the shared
  // epoch-tagged buffer, or — while a CUDA graph is being captured — a
  // graph-owned buffer zeroed by a captured memset on every replay.
  unsigned long long* lookback_status(int64_t tiles, uint32_t* epoch_out);
  void* get_scratch(size_t bytes);
  void count_launch(int n = 1) { launches += n; }

  // ---- CUDA-graph capture of repeated query plans (k_groupfused.cu) ----
  // While capturing, blocks freed are kept for the graph (capture_owned)
  // instead of returning to the cache, cache misses use cudaMalloc (no
  // stream-ordered allocation nodes), syncs / readbacks abort the capture,
  // and profiled regions record graph-owned events (capture_timers).
  bool capturing = false;
  bool capture_broken = false;
  std::vector<std::pair<void*, size_t>> capture_owned;
  // a profiled region inside a capture records two events of its own (event
  // nodes of the graph, re-recorded by every replay); a replay's times are
  // read just before the next replay re-records them, or by collect_profile
  struct CapTimer {
    std::string tag;
    cudaEvent_t a, b;
  };
  std::vector<CapTimer> capture_timers;
  std::vector<CapTimer> graph_timers_unread;
  void read_graph_timer(cudaEvent_t a);  // the unread run of the timer starting with event a, if any
  // graph cache key of the current API call (set by the C API for calls on
  // user handles only; consumed by the first fused pass of the call)
  std::string graph_key;
  struct GraphEntry {
    virtual ~GraphEntry() = default;
  };
  std::unordered_map<std::string, std::shared_ptr<GraphEntry>> graphs;
  void drop_graphs();  // syncs, then releases every cached graph and its blocks
};

using CtxPtr = std::shared_ptr<Ctx>;

// Resident CTAs per SM of `fn` at (block, smem) on `device`, setting the
// dynamic shared-memory opt-in first when smem > 48 KB. The attribute applies
// per device context, so it is set (and the occupancy cached) once per
// (kernel, device, block, smem) — a process with contexts on several devices
// opts in on each before its first launch there. Thread-safe.
int kernel_occupancy(int device, const void* fn, int block, size_t smem);
template <class K>
int kernel_occupancy(const CtxPtr& ctx, K* fn, int block, size_t smem) {
  return kernel_occupancy(ctx->device, reinterpret_cast<const void*>(fn), block, smem);
}

// Brackets the kernel launches issued in its scope with CUDA events on the
// context stream when profiling is enabled (no-op otherwise).
struct KTimer {
  Ctx* c;
  const char* tag;
  cudaEvent_t a = nullptr;
  std::chrono::steady_clock::time_point h0;
  bool captured = false;  // events owned by a graph being captured
  KTimer(const CtxPtr& ctx, const char* t) : c(ctx.get()), tag(t) {
    if (c->profiling && c->profile_wants(t)) {
      captured = c->capturing;
      if (captured) {  // an event-record node of the graph (External: not a capture-internal join point)
        cudaEventCreate(&a);
        cudaEventRecordWithFlags(a, c->stream, cudaEventRecordExternal);
      } else {
        a = c->get_event();
        cudaEventRecord(a, c->stream);
      }
      if (c->host_profiling) h0 = std::chrono::steady_clock::now();
    }
  }
  ~KTimer() {
    if (a && captured) {
      cudaEvent_t b;
      cudaEventCreate(&b);
      cudaEventRecordWithFlags(b, c->stream, cudaEventRecordExternal);
      c->capture_timers.push_back({tag, a, b});
      return;
    }
    if (a) {
      cudaEvent_t b = c->get_event();
      cudaEventRecord(b, c->stream);
      c->pending.push_back({tag, a, b});
      if (c->host_profiling)  // host wall time of the region (RQ_HOST_PROFILE=1)
        c->add_host_stat(std::string("host:") + tag,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    }
  }
};

// ---- buffers and arrays ----------------------------------------------------------

struct Buffer {
  CtxPtr ctx;  // keeps the stream alive for the stream-ordered free
  void* ptr = nullptr;
  size_t bytes = 0;
  size_t cap = 0;  // readable bytes from ptr (allocation rounded up to 256 B)
  bool owned = true;
  ~Buffer();
};

struct DArr {
  int32_t dt = RQ_I64;
  int64_t n = 0;
  std::shared_ptr<Buffer> buf;

  const void* raw() const { return buf ? buf->ptr : nullptr; }
  void* raw_mut() const { return buf ? buf->ptr : nullptr; }
  template <class T>
  T* as() const {
    return static_cast<T*>(raw_mut());
  }
  const int64_t* pos() const { return as<int64_t>(); }
  size_t bytes() const { return static_cast<size_t>(n) * dt_width(dt); }
};

DArr alloc_arr(const CtxPtr& ctx, int32_t dt, int64_t n);
// bulk copies need 16-B aligned bases and room to round a copy up to 16
// elements inside the allocation
inline bool tma_ok(const DArr& a) {
  if (!a.buf || !a.buf->ptr) return a.n == 0;
  const size_t w = static_cast<size_t>(dt_width(a.dt));
  return (reinterpret_cast<uintptr_t>(a.buf->ptr) & 15) == 0 &&
         a.buf->cap >= static_cast<size_t>((a.n + 15) & ~int64_t(15)) * w;
}

DArr upload_arr(const CtxPtr& ctx, int32_t dt, const void* host, int64_t n);
void download_arr(const CtxPtr& ctx, const DArr& a, void* host);
// Device-side copy of the first n elements into a new array.
DArr copy_prefix(const CtxPtr& ctx, const DArr& a, int64_t n);

// ---- columns (runq::Column, column.hpp:22-107) --------------------------------------

struct DCol {
  int32_t enc = RQ_ENC_PLAIN;
  int64_t total = 0;
  // PLAIN / PLAIN_INDEX base: v = storage values, logical, center
  // RLE / RLE_INDEX runs: v, s, e ; INDEX: v, p
  DArr v;
  int32_t logical = RQ_I64;
  bool has_center = false;
  int64_t center = 0;
  DArr s, e, p;
  // PLAIN_INDEX outliers / RLE_INDEX points
  DArr v2, p2;
  // RLE facts computed on demand: 1 if runs tile [0,total) with no gaps
  mutable int gapless = -1;
  // min / max of v (integer columns; computed on first use by the group-by
  // key builder — columns are immutable, so the facts stay valid)
  mutable bool has_minmax = false;
  mutable int64_t vmin = 0, vmax = 0;
  // rank directories of the run ends (e) and of the index positions (p2):
  // dir[b] = lower_bound(a, b << shift), built on first use (rank_dir)
  struct RankDir {
    DArr dir;
    int shift = -1;
    int64_t nb = 0;
  };
  mutable RankDir dir_e, dir_p2;

  int32_t value_type() const {  // column.cpp:88-97
    switch (enc) {
      case RQ_ENC_PLAIN: return logical;
      case RQ_ENC_PLAIN_INDEX: return v2.dt;
      default: return v.dt;
    }
  }
  int64_t runs() const { return s.n; }
};

struct DMask {
  int32_t enc = RQ_MASK_RLE;
  int64_t total = 0;
  DArr bits;    // PLAIN (uint8 per row, dt = I8)
  DArr s, e;    // RLE / COMPOSITE runs
  DArr p;       // INDEX / COMPOSITE points
  mutable int64_t true_count = -1;
  // RLE / composite-run masks: positions of the covered rows, expanded once
  // and shared by every plain column filtered with this mask
  mutable std::shared_ptr<DArr> positions;
};

}  // namespace rqb

// ---- opaque handle definitions -----------------------------------------------------

struct rq_ctx_s {
  rqb::CtxPtr ctx;
};
struct rq_arr_s {
  rqb::DArr a;
};
namespace rqb {
// handle ids: a graph cache key names the user handles of a call, never an
// address a later handle could reuse
inline uint64_t next_handle_uid() {
  static std::atomic<uint64_t> n{0};
  return ++n;
}
}  // namespace rqb
struct rq_col_s {
  rqb::DCol c;
  uint64_t uid = rqb::next_handle_uid();
};
struct rq_mask_s {
  rqb::DMask m;
  uint64_t uid = rqb::next_handle_uid();
};

namespace rqb {

void set_last_error(const std::string& msg);

template <class F>
int api_guard(F&& f) {
  try {
    f();
    set_last_error("");
    return RQ_OK;
  } catch (const RqError& ex) {
    set_last_error(ex.what());
    return ex.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return RQ_RESOURCE;
  } catch (const std::exception& ex) {
    set_last_error(ex.what());
    return RQ_INVALID;
  }
}

inline rq_arr_t wrap_arr(DArr a) { return new rq_arr_s{std::move(a)}; }
inline rq_col_t wrap_col(DCol c) { return new rq_col_s{std::move(c)}; }
inline rq_mask_t wrap_mask(DMask m) { return new rq_mask_s{std::move(m)}; }

// ---- operator entry points (ops.cpp / kernels) ----------------------------------------

struct Scalar {
  bool is_float = false;
  int64_t i = 0;
  double f = 0.0;
};

// primitives (k_merge.cu)
struct Intersection {
  DArr s, e, idx1, idx2;
};
Intersection range_intersect(const CtxPtr& ctx, const DArr& s1, const DArr& e1, const DArr& s2,
                             const DArr& e2, bool want_idx1, bool want_idx2);
struct PointsInRuns {
  DArr p_out, run_of, idx_of;
};
PointsInRuns points_in_runs(const CtxPtr& ctx, const DArr& p, const DArr& s, const DArr& e,
                            bool want_run_of, bool want_idx_of);
struct PointsIntersect {
  DArr p_out, idx1, idx2;
};
PointsIntersect points_intersect(const CtxPtr& ctx, const DArr& p1, const DArr& p2,
                                 bool want_idx1, bool want_idx2);
DArr bucketize(const CtxPtr& ctx, const DArr& x, const DArr& b, bool right);
// merge of two disjoint sorted lists (keys + optional run ends + values)
void merge_disjoint(const CtxPtr& ctx, const DArr& kA, const DArr* eA, const DArr* vA,
                    const DArr& kB, const DArr* eB, const DArr* vB, DArr& k_out, DArr* e_out,
                    DArr* v_out);
// sorted de-duplicated union of two position lists
DArr union_points(const CtxPtr& ctx, const DArr& p1, const DArr& p2);
// points of p not inside any run (subtract_runs)
DArr points_not_in_runs(const CtxPtr& ctx, const DArr& p, const DArr& s, const DArr& e);
// merge of two sorted lists keeping duplicates
DArr merge_keys(const CtxPtr& ctx, const DArr& a, const DArr& b);
// complement_rle / complement_index (primitives.cpp:141-167)
void complement_runs(const CtxPtr& ctx, const DArr& s, const DArr& e, int64_t total, DArr& s_out,
                     DArr& e_out);
// range_union tail over merged starts / ends (primitives.cpp:102-123)
void union_from_merged(const CtxPtr& ctx, const DArr& S, const DArr& E, DArr& s_out, DArr& e_out);
// byte-mask helpers
DArr bytes_or(const CtxPtr& ctx, const DArr& a, const DArr& b);
DArr bytes_not(const CtxPtr& ctx, const DArr& a);
DArr bytes_and(const CtxPtr& ctx, const DArr& a, const DArr& b);
DArr bytes_copy01(const CtxPtr& ctx, const DArr& a);
void set_bits(const CtxPtr& ctx, DArr& bits, const DArr& p);
DArr zeros_bytes(const CtxPtr& ctx, int64_t n);

// gathers / elementwise (k_dense.cu)
DArr gather(const CtxPtr& ctx, const DArr& v, const DArr& idx);
DArr decode_plain(const CtxPtr& ctx, const DCol& c);             // Plain -> logical values
DArr decode_plain_index(const CtxPtr& ctx, const DCol& c);       // P+I -> logical values
DArr arith_values(const CtxPtr& ctx, const DArr& a, const DArr& b, int op);
DArr cmp_values(const CtxPtr& ctx, const DArr& a, const DArr& b, int op);  // uint8 flags
DArr scalar_arith_values(const CtxPtr& ctx, const DArr& v, Scalar k, int op, bool reversed);
DArr scalar_cmp_values(const CtxPtr& ctx, const DArr& v, Scalar k, int op, bool reversed);
DArr cast_values(const CtxPtr& ctx, const DArr& v, int32_t to);
// Plain (narrow, centered) compare -> uint8 mask bytes, decode fused (K6/K9)
DArr plain_cmp_scalar(const CtxPtr& ctx, const DCol& c, Scalar k, int op, bool reversed);
// set bits[p[i]] = flags[i] (P+I outlier overlay)
void scatter_flags(const CtxPtr& ctx, DArr& bits, const DArr& p, const DArr& flags);
DArr iota(const CtxPtr& ctx, int64_t n);
// sort-based grouping (k_sort.cu): unique_with_inverse over aligned key values
struct SortedGroups {
  DArr inverse;     // group id per slot, ascending lexicographic key order
  DArr first_rows;  // first slot of each group in stable sorted order
  int64_t n_groups = 0;
};
SortedGroups group_ids_sorted(const CtxPtr& ctx, const std::vector<DArr>& keyvals);
// stable lexicographic row permutation (sort_table's comparator, ingest.cpp:318-333)
DArr sort_permutation(const CtxPtr& ctx, const std::vector<DArr>& keyvals);
void radix_sort_pairs(const CtxPtr& ctx, DArr& keys, DArr& vals, int bits, uint64_t sub);
void scan_exclusive_i64(const CtxPtr& ctx, const DArr& in, DArr& out);
// encoders (k_encode.cu): enc::plain_to_rle / plain_to_rle_index
DCol plain_to_rle(const CtxPtr& ctx, const DCol& c);
DCol plain_to_rle_index(const CtxPtr& ctx, const DCol& c, int64_t min_run);
DCol plain_to_plain_index(const CtxPtr& ctx, const DCol& c, double trim);
struct HeuristicD {  // io::HeuristicConfig (ingest.hpp:41-48)
  int64_t row_threshold = 1000000;
  double ratio_threshold = 20.0;
  double trim = 0.05;
  int64_t min_run = 2;
  double unit_run_share = 0.5;
};
struct EncodingChoiceD {  // io::EncodingChoice (ingest.hpp:33-39)
  int32_t scheme = RQ_SCHEME_PLAIN;
  int32_t width = RQ_I64;
  int64_t min_run = 2;
  double trim = 0.05;
  bool has_center = false;
  int64_t center = 0;
};
EncodingChoiceD choose_encoding(const CtxPtr& ctx, const DCol& c, const HeuristicD& cfg);
DCol encode_column(const CtxPtr& ctx, const DCol& c, const EncodingChoiceD& ch);
std::vector<DCol> sort_table(const CtxPtr& ctx, const std::vector<const DCol*>& cols,
                             const std::vector<int>& by);
DArr starts_from_ends(const CtxPtr& ctx, const DArr& e);  // gapless RLE starts
void scatter_values(const CtxPtr& ctx, DArr& dst, const DArr& idx, const DArr& src);

// compaction (k_select.cu)
// keep (s,e) of runs whose flag is set
void select_runs(const CtxPtr& ctx, const DArr& flags, const DArr& s, const DArr& e, DArr& s_out,
                 DArr& e_out);
// keep p of points whose flag is set (optionally also their index)
void select_points(const CtxPtr& ctx, const DArr& flags, const DArr& p, DArr& p_out,
                   DArr* idx_out);
void flagged_indices(const CtxPtr& ctx, const DArr& flags, int64_t n, DArr& out);
// RLE-column compare_scalar fused: flags computed inline from v
void rle_cmp_scalar_select(const CtxPtr& ctx, const DArr& v, const DArr& s, const DArr& e,
                           Scalar k, int op, bool reversed, DArr& s_out, DArr& e_out);
void index_cmp_scalar_select(const CtxPtr& ctx, const DArr& v, const DArr& p, Scalar k, int op,
                             bool reversed, DArr& p_out);
void plain_mask_to_rle(const CtxPtr& ctx, const DArr& bits, DArr& s, DArr& e);
DArr plain_mask_to_index(const CtxPtr& ctx, const DArr& bits);
// run expansion: positions of every row covered by runs (range_arange), and
// optionally the source run of each row.
void expand_runs(const CtxPtr& ctx, const DArr& s, const DArr& e, DArr* positions,
                 DArr* run_idx);
int64_t covered_rows(const CtxPtr& ctx, const DArr& s, const DArr& e);
int64_t count_nonzero(const CtxPtr& ctx, const DArr& bits);
bool runs_gapless(const CtxPtr& ctx, const DArr& s, const DArr& e, int64_t total);
DArr compact_positions(const CtxPtr& ctx, const DArr& s, const DArr& e, DArr& e_out,
                       int64_t* covered);

// reductions (k_agg.cu)
struct AggOut {
  int32_t dtype = RQ_I64;
  int64_t i = 0;
  double f = 0.0;
};
// Aggregate over slots with weights (run lengths) — shape given as RLE runs
// (s,e), or unit weights (points / dense) when s is empty.
AggOut reduce_slots(const CtxPtr& ctx, const DArr& v, const DArr* s, const DArr* e, int fn);
AggOut aggregate_column(const CtxPtr& ctx, const DCol& c, int fn);
AggOut aggregate_binop(const CtxPtr& ctx, const DCol& a, const DCol& b, int op, int fn);
AggOut filtered_aggregate_binop(const CtxPtr& ctx, const DCol& c, Scalar k, int cmp,
                                const DCol& a, const DCol& b, int op, int fn);

// high-level ops (ops.cpp)
struct Aligned {
  int kind = 0;  // 0 dense, 1 run, 2 point
  DArr s, e, p;
  DArr v1, v2;
  int64_t total = 0;
};
Aligned align(const CtxPtr& ctx, const DCol& a, const DCol& b);
DCol arith(const CtxPtr& ctx, const DCol& a, const DCol& b, int op);
DMask compare(const CtxPtr& ctx, const DCol& a, const DCol& b, int op);
DCol arith_scalar(const CtxPtr& ctx, const DCol& a, Scalar k, int op, bool reversed);
DMask compare_scalar(const CtxPtr& ctx, const DCol& a, Scalar k, int op, bool reversed);
DCol filter(const CtxPtr& ctx, const DCol& a, const DMask& m);
DMask mask_and(const CtxPtr& ctx, const DMask& a, const DMask& b);
DMask mask_or(const CtxPtr& ctx, const DMask& a, const DMask& b);
DMask mask_not(const CtxPtr& ctx, const DMask& a);
DCol normalize_basic(const CtxPtr& ctx, const DCol& c);
// joins (join.hpp:7-59), k_join.cu
DMask semi_join_mask(const CtxPtr& ctx, const DCol& probe, const DCol& build);
struct JoinSideD {  // joins::JoinIndex: rows (UnsortedIndexJoin) or (v, s, e) ranges (UnsortedRleJoin)
  bool is_rle = false;
  DArr rows;
  DArr v, s, e;
};
struct JoinResultD {
  JoinSideD left, right;
  int64_t cardinality = 0;
};
JoinResultD get_join_index(const CtxPtr& ctx, const DCol& left, const DCol& right);
void hash_build_probe(const CtxPtr& ctx, const DArr& build_values, const DArr& probe_values, DArr& build_pos,
                      DArr& probe_pos);
DCol apply_join_index(const CtxPtr& ctx, const DCol& col, const JoinSideD& j);
int64_t mask_true_count(const CtxPtr& ctx, const DMask& m);
bool col_gapless(const CtxPtr& ctx, const DCol& c);
// every row of [0, total) covered (Plain / Plain+Index, gapless RLE, full Index)
bool col_full_coverage(const CtxPtr& ctx, const DCol& c);

struct GroupAggOut {
  int64_t n_groups = 0;
  std::vector<DArr> keys;
  std::vector<DArr> vals;
};
// normalize=false: agg::group_aggregate semantics (RLE+Index inputs are an
// error, groupby.cpp:144-162 → decompose). normalize=true: the query
// runner's GroupAgg (normalize_basic on every input first, runner.cpp:306-336).
GroupAggOut group_aggregate(const CtxPtr& ctx, const std::vector<const DCol*>& keys,
                            const std::vector<const DCol*>& data, const std::vector<int>& fns,
                            bool normalize = false);
// Filter → expression → GroupAgg (runner.cpp:243-336) as one pass (K12):
// each expression is a left-deep chain ((t0 op0 t1) op1 t2) of terms
// `col` or `col sop k` / `k sop col` (reversed); no terms = COUNT(*).
// mask may be null; keys may be empty (one global group). Falls back to the
// operator chain for shapes the fused kernels do not take (*fused = false).
struct XTerm {
  const DCol* col = nullptr;
  int sop = -1;
  bool rev = false;
  Scalar k;
};
struct XExpr {
  std::vector<XTerm> terms;
  std::vector<int> ops;
};
namespace dev {
struct XgPlan;
struct XgSegs;
}  // namespace dev
// jit_xg.cpp: run-time specialised K12 row kernel (NVRTC)
bool xg_jit_available();
int xg_row_blocks_per_sm(int64_t avg_len);
bool xg_jit_launch(const CtxPtr& ctx, const dev::XgPlan& P, const dev::XgSegs& S, int64_t chunk,
                   unsigned long long* tab, int64_t G, int* err, unsigned blocks, int64_t avg_len);
// WHERE conjunct for the pushdown form: `col op k`, or `col IN (in)` when
// `in` is non-empty (the runner's OR of equalities)
struct XPred {
  const DCol* col = nullptr;
  int op = RQ_EQ;
  Scalar k;
  std::vector<Scalar> in;
};
GroupAggOut group_aggregate_exprs(const CtxPtr& ctx, const DMask* mask, const std::vector<const DCol*>& keys,
                                  const std::vector<XExpr>& exprs, const std::vector<int>& fns,
                                  bool* fused = nullptr, const std::vector<XPred>* preds = nullptr,
                                  bool fused_only = false);
bool group_aggregate_fused(const CtxPtr& ctx, const std::vector<const DCol*>& keys,
                           const std::vector<const DCol*>& data, const std::vector<int>& fns,
                           GroupAggOut& out);

// compute::decompose (align.cpp:86-100): shape + values of a basic column
// (kind 0 dense with n slots, 1 runs s/e, 2 points p); RLE+Index raises.
struct Decomp {
  int kind = 0;  // 0 dense, 1 run, 2 point
  int64_t n = 0;
  DArr s, e, p, values;
};
Decomp decompose_for_group(const CtxPtr& ctx, const DCol& c);
DCol col_from_decomp(const Decomp& d, const DArr& v, int64_t total);
// compute::align_many (align.cpp:233-254)
struct MultiAligned {
  Decomp shape;
  std::vector<DArr> values;
};
MultiAligned align_many(const CtxPtr& ctx, const std::vector<const DCol*>& cols);

// ---- the rest of the operator API surface (k_boundary.cu) ----------------------------

// kernels::cumsum / checked_sum (kernels.cpp:21-38): exact int64 prefix sums;
// the first element whose running sum leaves int64 raises RQ_OVERFLOW
DArr checked_cumsum(const CtxPtr& ctx, const DArr& x, bool exclusive);
int64_t checked_sum(const CtxPtr& ctx, const DArr& x);
// kernels::repeat_interleave / range_arange (kernels.cpp:40-60)
DArr repeat_interleave(const CtxPtr& ctx, const DArr& values, const DArr& counts);
DArr range_arange(const CtxPtr& ctx, const DArr& start, const DArr& length);
// kernels::scatter_reduce (kernels.cpp:97-125): op 0 sum, 1 min, 2 max, 3 count;
// values fold in input order within each group (bit-exact f64 sums)
DArr scatter_reduce(const CtxPtr& ctx, const DArr& values, const DArr& index, int64_t n_groups, int op);
// kernels::unique_with_inverse (kernels.cpp:127-187)
struct Unique {
  std::vector<DArr> keys;
  DArr inverse;
  int64_t n_groups = 0;
};
Unique unique_with_inverse(const CtxPtr& ctx, const std::vector<DArr>& cols);
// kernels::gather with the reference's bounds check (kernels.cpp:189-219)
DArr gather_checked(const CtxPtr& ctx, const DArr& values, const DArr& idx);
// kernels::sort_with_perm / adjacent_ne (kernels.cpp:221-245)
void sort_with_perm(const CtxPtr& ctx, const DArr& values, DArr& sorted, DArr& perm);
DArr adjacent_ne(const CtxPtr& ctx, const DArr& x);
// compute::shape_weights (align.cpp:57-70)
DArr shape_weights(const CtxPtr& ctx, const Decomp& shape);
// agg::aggregate_array (groupby.cpp:67-135)
DArr aggregate_array(const CtxPtr& ctx, const Decomp& shape, const DArr& values, const DArr& inverse,
                     int64_t n_groups, int fn);
// enc::rle_to_index / rle_to_plain / compact_rle_index (primitives.cpp:172-220, 381-420)
DCol rle_to_index(const CtxPtr& ctx, const DCol& c, int64_t budget);
DMask rle_mask_to_index(const CtxPtr& ctx, const DMask& m, int64_t budget);
DCol rle_to_plain(const CtxPtr& ctx, const DCol& c, double fill, int64_t budget);
DMask rle_mask_to_plain(const CtxPtr& ctx, const DMask& m, int64_t budget);
DCol compact_rle_index(const CtxPtr& ctx, const DCol& c);
// decode_full / to_rows (column.cpp:311-376)
DArr decode_full(const CtxPtr& ctx, const DCol& c);
void col_to_rows(const CtxPtr& ctx, const DCol& c, DArr& positions, DArr& values);

// ---- row-range sharded execution (comm.cu) ---------------------------------------

struct Comm;
Comm& comm_of(rq_comm_t c);
// AVG → (SUM, COUNT) partials; one partial per distinct (function, input)
// (same_input(i, j): inputs i and j are the same column / expression);
// local_fns / src per partial, sum_of / cnt_of per original function
// (cnt_of = -1 unless AVG)
struct PartialPlan {
  std::vector<int> local_fns, src, sum_of, cnt_of;
};
PartialPlan partial_plan(const std::vector<int>& fns, const std::function<bool(int, int)>& same_input);
GroupAggOut merge_group_tables(const CtxPtr& ctx, Comm& cm, const GroupAggOut& local,
                               const std::vector<int>& part_fns);
// local(plan) computes this rank's partial table; the result is the merged,
// finalised table (identical on every rank)
GroupAggOut sharded(const CtxPtr& ctx, Comm& cm, const std::vector<int>& fns,
                    const std::function<GroupAggOut(const PartialPlan&)>& local,
                    const std::function<bool(int, int)>& same_input = nullptr);
AggOut sharded_scalar(const CtxPtr& ctx, Comm& cm, int fn, const std::function<AggOut(int)>& local);

}  // namespace rqb
