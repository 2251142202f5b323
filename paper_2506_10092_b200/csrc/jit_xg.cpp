// jit_xg.cpp — run-time specialisation of the K12 row kernel.
//
// The interpreted row kernel (k_groupfused.cu, k_xg_rows) pays for its
// generality on every row: operand selection, type promotion and operator
// dispatch are data the kernel reads. Query engines on GPUs compile the
// expression instead. This file emits CUDA source for ONE plan shape —
// operand storage types, decode (logical width, centre present), term and
// chain operators, promotion, accumulator types — with the rows of a lane
// unrolled, compiles it with NVRTC for sm_100a (loaded with dlopen; no
// link-time dependency), loads the cubin with the runtime's library API and
// caches the kernel by its source text. Literal values and centres are kernel
// arguments, so plans that differ only in constants share one kernel.
// Semantics are the interpreted kernel's (and so the reference's): int64
// wrapping arithmetic, any float → f64, int ÷0 raises, AVG sums in f64.
// If NVRTC is unavailable the caller runs the interpreted kernel.
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "rq_internal.hpp"
#include "xg_plan.hpp"

namespace rqb {

namespace {

constexpr int ROWS = 8;  // rows per lane per window (one 8-byte load of an i8 column)

struct Nvrtc {
  bool ok = false;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  Nvrtc() {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                           "/usr/local/cuda/lib64/libnvrtc.so"};
    void* h = nullptr;
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return;
    create = reinterpret_cast<decltype(create)>(dlsym(h, "nvrtcCreateProgram"));
    compile = reinterpret_cast<decltype(compile)>(dlsym(h, "nvrtcCompileProgram"));
    log_size = reinterpret_cast<decltype(log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
    log = reinterpret_cast<decltype(log)>(dlsym(h, "nvrtcGetProgramLog"));
    cubin_size = reinterpret_cast<decltype(cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
    cubin = reinterpret_cast<decltype(cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    ok = create && compile && log_size && log && cubin_size && cubin && destroy;
  }
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  return n;
}

// Fixed part of every generated kernel: segment walk over covered rows
// (same schedule as k_xg_rows), warp reductions, table flush.
const char* kPrelude = R"(
typedef long long i64;
typedef unsigned long long u64;
struct XgSegs { const i64* s; const i64* e; const i64* off; const i64* slot; const u64* cst; i64 n; i64 ncov;
                double* dpart; i64 dcells; const i64* dims; i64 cstride; const i64* cstart;
                unsigned* fticket; i64 fchunks; unsigned fmask; };
struct XgCol { const void* v; i64 center; };
struct XgK { i64 i[24]; double f[24]; };
__device__ __forceinline__ i64 ldg64(const i64* p, i64 i) { return __ldg(p + i); }
__device__ __forceinline__ i64 warp_lb(const i64* a, i64 n, i64 key) {
  const int lane = threadIdx.x & 31;
  i64 lo = 0, hi = n;
  while (hi - lo > 32) {
    const i64 step = (hi - lo + 31) / 32;
    i64 x = lo + (i64)(lane + 1) * step - 1;
    if (x > hi - 1) x = hi - 1;
    const bool pred = __ldg(a + x) < key;
    const int c = __popc(__ballot_sync(0xffffffffu, pred));
    const i64 nlo = c == 0 ? lo : __shfl_sync(0xffffffffu, x, c - 1) + 1;
    const i64 nhi = c == 32 ? hi : __shfl_sync(0xffffffffu, x, c);
    lo = nlo;
    hi = nhi;
  }
  const i64 x = lo + lane;
  const bool pred = x < hi && __ldg(a + x) < key;
  return lo + __popc(__ballot_sync(0xffffffffu, pred));
}
__device__ __forceinline__ i64 idiv(i64 x, i64 y, int* err) {
  if (y == 0) { *err = 1; return 0; }
  if (x == (i64)0x8000000000000000ull && y == -1) return x;
  return x / y;
}
__device__ __forceinline__ i64 wadd(i64 a, i64 b) { return (i64)((u64)a + (u64)b); }
__device__ __forceinline__ i64 wsub(i64 a, i64 b) { return (i64)((u64)a - (u64)b); }
__device__ __forceinline__ i64 wmul(i64 a, i64 b) { return (i64)((u64)a * (u64)b); }
__device__ __forceinline__ double wsum_d(double x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ u64 wsum_u(u64 x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
)";

std::string ty(int f) { return f ? "double" : "i64"; }

// `ok`: the row-in-[r0, r1] test of the row being evaluated; integer division
// divides the other rows of the window by 1 so a zero divisor there (a row the
// WHERE dropped, a neighbouring segment, padding) cannot raise (the reference
// divides only the filtered rows, align.cpp:290-305)
std::string binop(const std::string& a, int fa, const std::string& b, int fb, int op, const std::string& ok) {
  if (fa || fb) {
    const char* o = op == RQ_ADD ? "+" : op == RQ_SUB ? "-" : op == RQ_MUL ? "*" : "/";
    return "((double)(" + a + ") " + o + " (double)(" + b + "))";
  }
  switch (op) {
    case RQ_ADD: return "wadd(" + a + ", " + b + ")";
    case RQ_SUB: return "wsub(" + a + ", " + b + ")";
    case RQ_MUL: return "wmul(" + a + ", " + b + ")";
    default: return "idiv(" + a + ", (" + ok + ") ? (" + b + ") : (i64)1, &lerr)";
  }
}

std::string wrap(int logical, const std::string& x) {
  switch (logical) {
    case RQ_I8: return "(i64)(signed char)(" + x + ")";
    case RQ_I16: return "(i64)(short)(" + x + ")";
    case RQ_I32: return "(i64)(int)(" + x + ")";
    default: return x;
  }
}

// the vector type and count of column c's raw loads for the lane's ROWS rows
struct RawLoad {
  const char* vt;  // vector type
  const char* et;  // element pointer type
  int n;           // loads (16-B or 8-B vectors)
};
RawLoad raw_load(int dt) {
  switch (dt) {
    case RQ_I8: return {"uint2", "signed char", 1};
    case RQ_I16: return {"uint4", "short", 1};
    case RQ_I32: return {"int4", "int", 2};
    case RQ_F32: return {"float4", "float", 2};
    case RQ_F64: return {"double2", "double", 4};
    default: return {"longlong2", "i64", 4};
  }
}
std::string wname(int c, int dt, int q) {
  const RawLoad L = raw_load(dt);
  return L.n == 1 ? "w" + std::to_string(c) : "w" + std::to_string(c) + "_" + std::to_string(q);
}

// raw vector loads of column c at row `rowv` into w<c>[_q]<suffix>; with a
// guard, a lane past the window's end loads nothing (zero vectors)
void gen_raw_loads(std::ostringstream& o, int c, const dev::PlainSrc& s, const std::string& rowv,
                   const std::string& suffix, const std::string& guard) {
  const RawLoad L = raw_load(s.dt);
  for (int q = 0; q < L.n; ++q) {
    const std::string ld = std::string("__ldg((const ") + L.vt + "*)((const " + L.et + "*)c" + std::to_string(c) +
                           ".v + " + rowv + ")" + (L.n == 1 ? "" : " + " + std::to_string(q)) + ")";
    o << "    const " << L.vt << " " << wname(c, s.dt, q) << suffix << " = "
      << (guard.empty() ? ld : "(" + guard + ") ? " + ld + " : " + L.vt + "{}") << ";\n";
  }
}

// w<c>[_q] = w<c>[_q]<suffix> (the window's loads under the names the decode uses)
void gen_alias(std::ostringstream& o, int c, const dev::PlainSrc& s, const std::string& suffix) {
  const RawLoad L = raw_load(s.dt);
  for (int q = 0; q < L.n; ++q)
    o << "    const " << L.vt << " " << wname(c, s.dt, q) << " = " << wname(c, s.dt, q) << suffix << ";\n";
}

// decode of column c's loaded vectors into x<c>_<u>
void gen_decode(std::ostringstream& o, int c, const dev::PlainSrc& s) {
  const std::string p = "c" + std::to_string(c);
  auto raw = [&](int u) -> std::string {
    switch (s.dt) {
      case RQ_I8: return "(i64)(signed char)(w" + std::to_string(c) + (u < 4 ? ".x" : ".y") + " >> " +
                         std::to_string(8 * (u % 4)) + ")";
      case RQ_I16: {
        const char* f[] = {".x", ".y", ".z", ".w"};
        return "(i64)(short)(w" + std::to_string(c) + f[u / 2] + " >> " + std::to_string(16 * (u % 2)) + ")";
      }
      case RQ_I32: return "(i64)w" + std::to_string(c) + "_" + std::to_string(u / 4) + "." + "xyzw"[u % 4];
      case RQ_F32: return "(double)w" + std::to_string(c) + "_" + std::to_string(u / 4) + "." + "xyzw"[u % 4];
      default: return std::string("w") + std::to_string(c) + "_" + std::to_string(u / 2) + (u % 2 ? ".y" : ".x");
    }
  };
  const bool fstore = s.dt == RQ_F32 || s.dt == RQ_F64;
  for (int u = 0; u < ROWS; ++u) {
    std::string v = raw(u);
    if (!fstore) {
      if (s.logical != RQ_I64 && s.logical != RQ_F32 && s.logical != RQ_F64) v = wrap(s.logical, v);
      if (s.has_center) {
        v = "wadd(" + v + ", " + p + ".center)";
        if (s.logical != RQ_I64 && s.logical != RQ_F32 && s.logical != RQ_F64) v = wrap(s.logical, v);
      }
      if (s.flt) v = "(double)(" + v + ")";
    }
    o << "    const " << ty(s.flt) << " x" << c << "_" << u << " = " << v << ";\n";
  }
}

// windows of 32 x ROWS rows a short-segment row loop loads before it
// computes (RQ_JIT_UNROLL=2: both windows' loads issued first). Measured
// slower at the 64-register cap — Q6's row kernel 31 -> 35 µs, C5's 34 ->
// 36 µs (profiles/r2b_ab_jit_unroll.txt) — so one window per trip stays.
int window_unroll() {
  static const int u = [] {
    const char* e = std::getenv("RQ_JIT_UNROLL");
    return e && std::atoi(e) == 2 ? 2 : 1;
  }();
  return u;
}

// windows ahead the row loop prefetches into L2 (RQ_JIT_PF, default 1; 0 = off;
// Q1 row kernel 1.20 -> 1.12 ms at 1, 1.14 at 2, 1.17 at 4)
int prefetch_distance() {
  static const int pf = [] {
    const char* e = std::getenv("RQ_JIT_PF");
    return e ? std::atoi(e) : 1;
  }();
  return pf;
}

// software-pipelined segment bounds in the row loop (RQ_JIT_PIPE=0: off, A/B)
bool pipeline_segments() {
  static const bool on = [] {
    const char* e = std::getenv("RQ_JIT_PIPE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// the source of a plan's kernel; literal slots are appended to ki / kf
std::string gen_source(const dev::XgPlan& P, std::vector<int64_t>& ki, std::vector<double>& kf, int pf, int minb) {
  std::ostringstream o;
  o << kPrelude;
  o << "extern \"C\" __global__ void __launch_bounds__(256, " << minb << ") xg_kernel(const XgSegs S, const i64 chunk, u64* gtab, "
       "const i64 G, int* err, const XgCol c0, const XgCol c1, const XgCol c2, const XgCol c3, const XgK K) {\n";
  o << "  constexpr int NE = " << P.ne << ";\n";
  o << "  __shared__ u64 stab[4096];\n";
  o << "  const i64 cells = G * NE;\n  const bool in_smem = cells <= 4096;\n";
  o << "  if (in_smem) { for (i64 i = threadIdx.x; i < cells; i += 256) stab[i] = 0ull; __syncthreads(); }\n";
  o << "  u64* tab = in_smem ? stab : gtab;\n";
  o << "  const int lane = threadIdx.x & 31;\n";
  o << "  const i64 warp = ((i64)blockIdx.x * 256 + threadIdx.x) >> 5;\n";
  o << "  const i64 nwarps = ((i64)gridDim.x * 256) >> 5;\n  int lerr = 0;\n";
  for (int e = 0; e < P.ne; ++e)
    if (P.e[e].rows) o << "  " << (P.e[e].acc_f ? "double" : "u64") << " a" << e << " = 0;\n";
  // (segments, covered rows) from the device when the table was built without a readback;
  // chunk 0: derived from them as the host does (xg_chunk)
  o << "  const i64 nseg_ = S.dims ? ldg64(S.dims, 0) : S.n, ncov_ = S.dims ? ldg64(S.dims, 1) : S.ncov;\n"
       "  i64 chunk_ = chunk;\n"
       "  if (chunk_ <= 0) { chunk_ = (ncov_ + nwarps - 1) / nwarps; chunk_ = (chunk_ + 127) / 128 * 128;"
       " if (chunk_ < 512) chunk_ = 512; }\n";
  o << "  for (i64 c0_ = warp * chunk_; c0_ < ncov_; c0_ += nwarps * chunk_) {\n"
       "    const i64 c1_ = min(c0_ + chunk_, ncov_);\n"
       "    i64 k = S.cstart ? ldg64(S.cstart, c0_ / chunk_) : warp_lb(S.off, nseg_, c0_ + 1) - 1;\n"
       "    i64 c = c0_;\n";
  // short segments (no L2 prefetch): the next segment's bounds are loaded
  // while this one's rows stream, so a segment costs one round trip, not two
  const bool pipe = pf == 0 && pipeline_segments();
  const int unroll = pf == 0 ? window_unroll() : 1;  // long segments: the L2 prefetch instead
  if (pipe)
    o << "    i64 off = ldg64(S.off, k), s = ldg64(S.s, k), e = ldg64(S.e, k), slot = ldg64(S.slot, k);\n"
         "    while (c < c1_) {\n"
         "      const bool more_ = k + 1 < nseg_;\n"
         "      const i64 n_off = more_ ? ldg64(S.off, k + 1) : 0, n_s = more_ ? ldg64(S.s, k + 1) : 0;\n"
         "      const i64 n_e = more_ ? ldg64(S.e, k + 1) : 0, n_slot = more_ ? ldg64(S.slot, k + 1) : -1;\n";
  else
    o << "    while (c < c1_) {\n"
         "      const i64 off = ldg64(S.off, k), s = ldg64(S.s, k), e = ldg64(S.e, k);\n"
         "      const i64 slot = ldg64(S.slot, k);\n";
  for (int j = 0; j < P.ncst; ++j) {
    if (P.cst_f[j])
      o << "      const double k" << j << " = __longlong_as_double((long long)__ldg(S.cst + " << j << " * S.cstride + k));\n";
    else
      o << "      const i64 k" << j << " = (i64)__ldg(S.cst + " << j << " * S.cstride + k);\n";
  }
  o << "      const i64 r0 = s + (c - off);\n"
       "      const i64 r1 = min(e, s + (c1_ - off) - 1);\n"
       "      for (i64 b = r0 & ~(i64)" << (ROWS - 1) << "; b <= r1; b += " << 32 * ROWS * unroll << ") {\n";
  // L2 prefetch of the window PF windows ahead, one 128-B line per lane and
  // column: more bytes in flight per warp without holding them in registers
  if (pf > 0 && P.nc > 0) {
    o << "        { const i64 pb = b + " << pf * 32 * ROWS << ";\n"
         "          if (pb <= r1) {\n"
         "            const i64 pe = min(r1 + 1, pb + " << 32 * ROWS << ");\n";
    for (int c = 0; c < P.nc; ++c) {
      const int w = dt_width(P.col[c].dt);
      o << "            { const i64 lo = (pb * " << w << ") & ~(i64)127, a = lo + (i64)lane * 128;\n"
           "              if (a < pe * " << w << ") asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"((const char*)c" << c
        << ".v + a)); }\n";
    }
    o << "          }\n        }\n";
  }
  // expression values per row, then the accumulation (guarded form for partial windows)
  auto lit = [&](const dev::XgTerm& t) -> std::string {
    if (t.kflt) {
      kf.push_back(t.kf);
      return "K.f[" + std::to_string(kf.size() - 1) + "]";
    }
    ki.push_back(t.ki);
    return "K.i[" + std::to_string(ki.size() - 1) + "]";
  };
  std::vector<std::vector<std::string>> lits(static_cast<size_t>(P.ne));
  for (int e = 0; e < P.ne; ++e) {
    const dev::XgExpr& X = P.e[e];
    if (!X.rows) continue;
    for (int t = 0; t < X.nt; ++t) lits[static_cast<size_t>(e)].push_back(X.t[t].sop >= 0 ? lit(X.t[t]) : "");
  }
  // one window's decode + expressions + accumulation at `row` (loads named w<c>[_q])
  std::ostringstream body;
  for (int c = 0; c < P.nc; ++c) gen_decode(body, c, P.col[c]);
  for (int e = 0; e < P.ne; ++e) {
    const dev::XgExpr& X = P.e[e];
    if (!X.rows) continue;
    for (int u = 0; u < ROWS; ++u) {
      const std::string ok = "row + " + std::to_string(u) + " >= r0 && row + " + std::to_string(u) + " <= r1";
      std::string v;
      int vf = 0;
      for (int t = 0; t < X.nt; ++t) {
        const dev::XgTerm& T = X.t[t];
        std::string x = T.src < dev::XG_COLS ? "x" + std::to_string(T.src) + "_" + std::to_string(u)
                                             : "k" + std::to_string(T.src - dev::XG_COLS);
        int xf = T.flt;
        if (T.sop >= 0) {
          const std::string& k = lits[static_cast<size_t>(e)][static_cast<size_t>(t)];
          x = T.rev ? binop(k, T.kflt, x, xf, T.sop, ok) : binop(x, xf, k, T.kflt, T.sop, ok);
          xf = xf || T.kflt;
        }
        if (t == 0) {
          v = x;
          vf = xf;
        } else {
          v = binop(v, vf, x, xf, X.op[t - 1], ok);
          vf = vf || xf;
        }
      }
      body << "        const " << ty(vf) << " v" << e << "_" << u << " = " << v << ";\n";
    }
  }
  body << "        if (row >= r0 && row + " << ROWS - 1 << " <= r1) {\n";
  for (int e = 0; e < P.ne; ++e) {
    const dev::XgExpr& X = P.e[e];
    if (!X.rows) continue;
    for (int u = 0; u < ROWS; ++u)
      body << "          a" << e << " += " << (X.acc_f ? "(double)" : "(u64)") << "v" << e << "_" << u << ";\n";
  }
  body << "        } else {\n";
  for (int e = 0; e < P.ne; ++e) {
    const dev::XgExpr& X = P.e[e];
    if (!X.rows) continue;
    for (int u = 0; u < ROWS; ++u)
      body << "          if (row + " << u << " >= r0 && row + " << u << " <= r1) a" << e << " += "
           << (X.acc_f ? "(double)" : "(u64)") << "v" << e << "_" << u << ";\n";
  }
  body << "        }\n";
  if (unroll == 1) {
    o << "        const i64 row = b + lane * " << ROWS << ";\n"
         "        if (row > r1) continue;\n";
    for (int c = 0; c < P.nc; ++c) gen_raw_loads(o, c, P.col[c], "row", "", "");
    o << body.str() << "      }\n";
  } else {
    // both windows' loads issued before either is used: two round trips in
    // flight per warp on segments of a few hundred rows
    o << "        const i64 rw0_ = b + lane * " << ROWS << ", rw1_ = rw0_ + " << 32 * ROWS << ";\n";
    for (int c = 0; c < P.nc; ++c) gen_raw_loads(o, c, P.col[c], "rw0_", "_A", "rw0_ <= r1");
    for (int c = 0; c < P.nc; ++c) gen_raw_loads(o, c, P.col[c], "rw1_", "_B", "rw1_ <= r1");
    for (int w = 0; w < 2; ++w) {
      o << "        if (rw" << w << "_ <= r1) {\n        const i64 row = rw" << w << "_;\n";
      for (int c = 0; c < P.nc; ++c) gen_alias(o, c, P.col[c], w ? "_B" : "_A");
      o << body.str() << "        }\n";
    }
    o << "      }\n";
  }
  o << "      c = min(c1_, off + (e - s + 1));\n";
  if (pipe)
    o << "      const i64 next_slot = (c < c1_ && more_) ? n_slot : -1;\n";
  else
    o << "      const i64 next_slot = (c < c1_ && k + 1 < nseg_) ? ldg64(S.slot, k + 1) : -1;\n";
  o << "      if (next_slot != slot) {\n";
  for (int e = 0; e < P.ne; ++e) {
    const dev::XgExpr& X = P.e[e];
    if (!X.rows) continue;
    if (X.acc_f)
      o << "        { const double t = wsum_d(a" << e << ");\n"
           "          if (S.dpart) { if (lane == 0) S.dpart[(c0_ / chunk_) * S.dcells + slot * NE + " << e << "] += t; }\n"
           "          else if (lane == 0 && t != 0.0) atomicAdd((double*)tab + slot * NE + " << e << ", t);\n"
           "          a" << e << " = 0.0; }\n";
    else
      o << "        { const u64 t = wsum_u(a" << e << "); if (lane == 0 && t != 0ull) atomicAdd(tab + slot * NE + " << e
        << ", t); a" << e << " = 0ull; }\n";
  }
  if (pipe) o << "      }\n      ++k;\n      off = n_off; s = n_s; e = n_e; slot = n_slot;\n    }\n  }\n";
  else o << "      }\n      ++k;\n    }\n  }\n";
  o << "  if (lerr) atomicOr(err, 1);\n";
  o << "  if (in_smem) {\n    __syncthreads();\n    for (i64 i = threadIdx.x; i < cells; i += 256) {\n"
       "      const u64 v = stab[i];\n      if (!v) continue;\n      switch ((int)(i % NE)) {\n";
  for (int e = 0; e < P.ne; ++e) {
    if (!P.e[e].rows) continue;
    if (P.e[e].acc_f)
      o << "        case " << e << ": atomicAdd((double*)gtab + i, __longlong_as_double((long long)v)); break;\n";
    else
      o << "        case " << e << ": atomicAdd(gtab + i, v); break;\n";
  }
  o << "        default: break;\n      }\n    }\n  }\n";
  // the last CTA folds the per-chunk f64 partials in a fixed order (same
  // bits every run): chunk-strided sums per thread, then a fixed tree
  o << "  if (S.fticket) {\n"
       "    __shared__ bool last_;\n"
       "    __threadfence();\n    __syncthreads();\n"
       "    if (threadIdx.x == 0) last_ = atomicInc(S.fticket, gridDim.x - 1) == gridDim.x - 1;\n"
       "    __syncthreads();\n"
       "    if (last_) {\n"
       "      __threadfence();\n"
       "      double* red = (double*)stab;\n"
       "      for (i64 cell = 0; cell < S.dcells; ++cell) {\n"
       "        if (!((S.fmask >> (int)(cell % NE)) & 1u)) continue;\n"
       "        double f0 = 0.0, f1 = 0.0;\n"
       "        i64 q = threadIdx.x;\n"
       "        for (; q + 256 < S.fchunks; q += 512) {\n"
       "          f0 += __ldcg(S.dpart + q * S.dcells + cell);\n"
       "          f1 += __ldcg(S.dpart + (q + 256) * S.dcells + cell);\n"
       "        }\n"
       "        if (q < S.fchunks) f0 += __ldcg(S.dpart + q * S.dcells + cell);\n"
       "        red[threadIdx.x] = f0 + f1;\n"
       "        __syncthreads();\n"
       "        for (int w = 128; w > 0; w >>= 1) {\n"
       "          if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];\n"
       "          __syncthreads();\n"
       "        }\n"
       "        if (threadIdx.x == 0) ((double*)gtab)[cell] = red[0];\n"
       "        __syncthreads();\n"
       "      }\n"
       "    }\n"
       "  }\n}\n";
  return o.str();
}

struct Cache {
  std::mutex mu;
  std::unordered_map<std::string, cudaKernel_t> kernels;
  std::unordered_map<std::string, bool> failed;
};
Cache& cache() {
  static Cache c;
  return c;
}

cudaKernel_t compile(const std::string& src) {
  Nvrtc& N = nvrtc();
  if (!N.ok) return nullptr;
  Cache& C = cache();
  std::lock_guard<std::mutex> g(C.mu);
  auto it = C.kernels.find(src);
  if (it != C.kernels.end()) return it->second;
  if (C.failed.count(src)) return nullptr;
  nvrtcProgram prog;
  if (N.create(&prog, src.c_str(), "xg_kernel.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    C.failed[src] = true;
    return nullptr;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--fmad=false"};
  const nvrtcResult r = N.compile(prog, 4, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    N.log_size(prog, &n);
    std::string log(n, '\0');
    N.log(prog, &log[0]);
    std::fprintf(stderr, "runq_b200: K12 kernel compilation failed (interpreted kernel used):\n%s\n", log.c_str());
    N.destroy(&prog);
    C.failed[src] = true;
    // RQ_JIT_STRICT=1 (the GPU test suite): a generator bug fails loudly
    // instead of silently running the interpreted kernel
    const char* strict = std::getenv("RQ_JIT_STRICT");
    if (strict && strict[0] == '1') throw RqError(RQ_CUDA, "K12 kernel compilation failed:\n" + log);
    return nullptr;
  }
  size_t n = 0;
  N.cubin_size(prog, &n);
  std::vector<char> bin(n);
  N.cubin(prog, bin.data());
  N.destroy(&prog);
  cudaLibrary_t lib;
  if (cudaLibraryLoadData(&lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) {
    cudaGetLastError();
    C.failed[src] = true;
    return nullptr;
  }
  cudaKernel_t k;
  if (cudaLibraryGetKernel(&k, lib, "xg_kernel") != cudaSuccess) {
    cudaGetLastError();
    C.failed[src] = true;
    return nullptr;
  }
  C.kernels[src] = k;
  return k;
}

struct XgColArg {
  const void* v;
  int64_t center;
};
struct XgKArg {
  int64_t i[24];
  double f[24];
};

}  // namespace

bool xg_jit_available() { return nvrtc().ok; }

// Launches the generated kernel for plan P; false if it cannot be built
// (NVRTC missing, too many literals, compile failure).
// Compact structural signature of a plan (what the generated source depends
// on): the source is built only on a cache miss.
std::string plan_signature(const dev::XgPlan& P, int minb, int pf) {
  std::string sig;
  auto put = [&](int64_t v) { sig += std::to_string(v); sig += ','; };
  put(minb);
  put(pf);
  put(pipeline_segments() ? 1 : 0);
  put(pf == 0 ? window_unroll() : 1);
  put(P.nc);
  for (int c = 0; c < P.nc; ++c) {
    put(P.col[c].dt);
    put(P.col[c].logical);
    put(P.col[c].has_center);
    put(P.col[c].flt);
  }
  put(P.ncst);
  for (int j = 0; j < P.ncst; ++j) put(P.cst_f[j]);
  put(P.ne);
  for (int e = 0; e < P.ne; ++e) {
    const dev::XgExpr& X = P.e[e];
    put(X.nt);
    put(X.rows);
    put(X.acc_f);
    put(X.op[0]);
    put(X.op[1]);
    for (int t = 0; t < X.nt; ++t) {
      put(X.t[t].src);
      put(X.t[t].flt);
      put(X.t[t].sop);
      put(X.t[t].rev);
      put(X.t[t].kflt);
    }
  }
  return sig;
}

// literal slots in the order gen_source numbers them
void plan_literals(const dev::XgPlan& P, std::vector<int64_t>& ki, std::vector<double>& kf) {
  for (int e = 0; e < P.ne; ++e) {
    const dev::XgExpr& X = P.e[e];
    if (!X.rows) continue;
    for (int t = 0; t < X.nt; ++t) {
      if (X.t[t].sop < 0) continue;
      if (X.t[t].kflt) kf.push_back(X.t[t].kf);
      else ki.push_back(X.t[t].ki);
    }
  }
}

// Row-kernel CTAs per SM, the grid its covered-row chunks are cut for (the
// k-way segment table's chunk-start entries use the same count), always a
// whole number of waves of resident CTAs: plans of short segments run ONE
// wave (Q6 row kernel 36.4 -> 29.5 µs, C5 37.5 -> 33.4 µs; 2 waves of small
// chunks paid a segment-bound start-up per chunk), long-segment plans 4 waves
// of 3 (Q1 1.198 -> 1.181 ms, C3 2.14 -> 2.07 ms against the former 8 = 2.67
// waves; profiles/r2_ab_bps.txt). RQ_XG_BPS overrides.
int xg_row_blocks_per_sm(int64_t avg_len) {
  static const int env = [] {
    const char* e = std::getenv("RQ_XG_BPS");
    return e ? std::atoi(e) : 0;
  }();
  if (env > 0) return env;
  static const int64_t pf_min = [] {
    const char* e = std::getenv("RQ_JIT_PF_MIN");
    return e ? std::atoll(e) : int64_t{2048};
  }();
  if (avg_len >= pf_min) return 12;  // the long-segment kernel keeps 3 CTAs per SM
  const char* mb = std::getenv("RQ_JIT_MINB");
  return mb && std::atoi(mb) > 0 ? std::atoi(mb) : 4;  // = the short-segment kernel's resident CTAs
}

bool xg_jit_launch(const CtxPtr& ctx, const dev::XgPlan& P, const dev::XgSegs& S, int64_t chunk,
                   unsigned long long* tab, int64_t G, int* err, unsigned blocks, int64_t avg_len) {
  std::vector<int64_t> ki;
  std::vector<double> kf;
  plan_literals(P, ki, kf);
  if (ki.size() > 24 || kf.size() > 24) return false;
  const char* mb = std::getenv("RQ_JIT_MINB");
  // the L2 prefetch pays on long segments (Q1: 1.20 -> 1.12 ms, C3's row pass
  // -4%) and costs on plans of many short selected segments (Q6: +20%)
  static const int64_t pf_min = [] {  // segment length from which the prefetch pays (RQ_JIT_PF_MIN)
    const char* e = std::getenv("RQ_JIT_PF_MIN");
    return e ? std::atoll(e) : int64_t{2048};
  }();
  const int pf = avg_len >= pf_min ? prefetch_distance() : 0;
  // resident CTAs per SM: 3 for long segments (Q1: 4 measured 1.48 vs 1.19 ms),
  // 4 for short ones (Q6 row kernel 41 -> 36 µs; profiles/r2_ab_jit_pipe_minb.txt);
  // RQ_JIT_MINB overrides
  const int minb = mb ? std::atoi(mb) : pf ? 3 : 4;
  const std::string sig = plan_signature(P, minb, pf);
  cudaKernel_t k = nullptr;
  {
    static std::mutex mu;
    static std::unordered_map<std::string, cudaKernel_t> by_sig;
    std::lock_guard<std::mutex> g(mu);
    auto it = by_sig.find(sig);
    if (it != by_sig.end()) {
      k = it->second;
    } else {
      std::vector<int64_t> ki2;
      std::vector<double> kf2;
      k = compile(gen_source(P, ki2, kf2, pf, minb));
      by_sig[sig] = k;  // nullptr too: a failed compilation is not retried
    }
  }
  if (!k) return false;
  XgColArg cols[4] = {};
  for (int c = 0; c < P.nc && c < 4; ++c) cols[c] = {P.col[c].v, P.col[c].center};
  XgKArg K{};
  for (size_t i = 0; i < ki.size(); ++i) K.i[i] = ki[i];
  for (size_t i = 0; i < kf.size(); ++i) K.f[i] = kf[i];
  dev::XgSegs s = S;
  int64_t ch = chunk, g = G;
  void* args[] = {&s, &ch, &tab, &g, &err, &cols[0], &cols[1], &cols[2], &cols[3], &K};
  RQ_CUDA_CHECK(cudaLaunchKernel(reinterpret_cast<const void*>(k), dim3(blocks), dim3(256), args, 0, ctx->stream));
  return true;
}

}  // namespace rqb
