// xg_plan.hpp — the K12 expression group-aggregate plan (host-built, passed
// by value to the interpreted row kernel and to the generated one).
#pragma once

#include <stdint.h>

#include <string>

namespace rqb {
namespace dev {

struct PlainSrc {  // bit-width-reduced plain column (decode inline)
  const void* v;
  int dt, logical, has_center, flt;
  int64_t center;
};

constexpr int XG_COLS = 4, XG_CONSTS = 4, XG_EXPRS = 8;

struct XgTerm {
  int src;   // < XG_COLS: plain column; >= XG_COLS: segment constant src - XG_COLS
  int flt;   // source value is f64
  int sop;   // scalar op (RQ_ADD..RQ_DIV) or -1
  int rev;   // scalar on the left (k op x)
  int kflt;  // scalar is f64
  int64_t ki;
  double kf;
};
struct XgExpr {
  int nt;     // 1..3 terms
  int op[2];  // chain ops, left-deep: ((t0 op0 t1) op1 t2)
  XgTerm t[3];
  int acc_f;  // accumulate in f64 (float result); integer results (AVG too) accumulate in int64
  int res_f;  // expression result is f64
  int rows;   // evaluated per row (references a plain column)
};
struct XgPlan {
  int nc;
  PlainSrc col[XG_COLS];
  int ncst;
  int cst_f[XG_CONSTS];
  int ne;
  XgExpr e[XG_EXPRS];
};

struct XgSegs {
  const int64_t* s;
  const int64_t* e;
  const int64_t* off;   // exclusive prefix of segment lengths (covered rows)
  const int64_t* slot;
  const uint64_t* cst;  // [XG_CONSTS][cstride] RLE operand values (i64 / f64 bits)
  int64_t n;            // segments, or the table's capacity when `dims` is set
  int64_t ncov;         // covered rows (unused when `dims` is set)
  // deterministic f64 sums: each chunk (a warp's covered-row range) writes its
  // per-cell partial to dpart[chunk * dcells + cell] (no atomics); a fixed-
  // order fold adds them up. Null: atomic adds (order-dependent last bits).
  double* dpart;
  int64_t dcells;
  // device-resident (segments, covered rows) of a table built without a host
  // readback (the k-way builder); null: n / ncov above
  const int64_t* dims;
  int64_t cstride;  // operand j of segment k at cst[j * cstride + k]
  // k-way tables: the segment holding each row chunk's first covered row
  // (chunk q starts at row q * xg_chunk(ncov, nwarps)); null: searched in off
  const int64_t* cstart;
  // generated row kernel only: the f64 fold of dpart done by the last CTA to
  // finish (ticket wraps back to 0) for the expressions in fmask, instead of a
  // separate k_xg_dfold launch; null: no in-kernel fold
  unsigned* fticket;
  int64_t fchunks;
  unsigned fmask;
};

// rows per warp chunk of the row kernels: at least 512, a multiple of 128,
// and at most `nwarps` chunks (the deterministic fold's partial tables)
__host__ __device__ inline int64_t xg_chunk(int64_t ncov, int64_t nwarps) {
  int64_t c = (ncov + nwarps - 1) / nwarps;
  c = (c + 127) / 128 * 128;
  return c < 512 ? 512 : c;
}

}  // namespace dev
}  // namespace rqb
