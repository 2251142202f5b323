/*
 * runq_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference's hot-path algorithms. See runq_oracle.h for the contract and
 * how this restatement is pinned (golden vectors + live reference library).
 * Never linked into or called by the product path.
 */
#include "runq_oracle.h"

#include <stddef.h>
#include <string.h>

/* runq::DType codes (dtype.hpp:11) */
enum { I8 = 0, I16 = 1, I32 = 2, I64 = 3, F32 = 4, F64 = 5 };
/* runq::compute::BinOp codes (align.hpp:70) */
enum { ADD = 0, SUB = 1, MUL = 2, DIV = 3, LT = 4, LE = 5, EQ = 6, NE = 7, GE = 8, GT = 9 };

static int64_t lower_bound(const int64_t* b, int64_t nb, int64_t x) {
  int64_t lo = 0, hi = nb;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (b[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static int64_t upper_bound(const int64_t* b, int64_t nb, int64_t x) {
  int64_t lo = 0, hi = nb;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (b[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* kernels.cpp:10-19 */
void orq_bucketize(const int64_t* x, int64_t nx, const int64_t* b, int64_t nb, int right,
                   int64_t* out) {
  for (int64_t i = 0; i < nx; ++i)
    out[i] = right ? upper_bound(b, nb, x[i]) : lower_bound(b, nb, x[i]);
}

/* primitives.cpp:15-46: the list with fewer runs drives; for driver run i,
 * the overlapping runs of the other list are [lower_bound(e_other, s_i),
 * upper_bound(s_other, e_i)); fragments in driver order then other order;
 * idx outputs reported per argument. */
int64_t orq_range_intersect(const int64_t* s1, const int64_t* e1, int64_t n1, const int64_t* s2,
                            const int64_t* e2, int64_t n2, int64_t* s, int64_t* e, int64_t* idx1,
                            int64_t* idx2) {
  int swapped = n1 > n2;
  const int64_t *ds = s1, *de = e1, *os = s2, *oe = e2;
  int64_t dn = n1, on = n2;
  if (swapped) {
    ds = s2; de = e2; dn = n2;
    os = s1; oe = e1; on = n1;
  }
  int64_t k = 0;
  for (int64_t i = 0; i < dn; ++i) {
    int64_t jb = lower_bound(oe, on, ds[i]);
    int64_t je = upper_bound(os, on, de[i]);
    for (int64_t j = jb; j < je; ++j) {
      s[k] = ds[i] > os[j] ? ds[i] : os[j];
      e[k] = de[i] < oe[j] ? de[i] : oe[j];
      idx1[k] = swapped ? j : i;
      idx2[k] = swapped ? i : j;
      ++k;
    }
  }
  return k;
}

/* primitives.cpp:48-61: bin = upper_bound(s, p) - 1, keep if p <= e[bin]. */
int64_t orq_idx_in_rle(const int64_t* p, int64_t np, const int64_t* s, const int64_t* e,
                       int64_t nr, int64_t* p_out, int64_t* run_of, int64_t* idx_of) {
  int64_t k = 0;
  for (int64_t i = 0; i < np; ++i) {
    int64_t b = upper_bound(s, nr, p[i]) - 1;
    if (b >= 0 && p[i] <= e[b]) {
      p_out[k] = p[i];
      run_of[k] = b;
      idx_of[k] = i;
      ++k;
    }
  }
  return k;
}

/* primitives.cpp:63-86: per run, the covered position-index range is
 * [lower_bound(p, s_r), upper_bound(p, e_r) - 1]; expand in run order. */
int64_t orq_rle_contain_idx(const int64_t* p, int64_t np, const int64_t* s, const int64_t* e,
                            int64_t nr, int64_t* p_out, int64_t* run_of, int64_t* idx_of) {
  int64_t k = 0;
  for (int64_t r = 0; r < nr; ++r) {
    int64_t lo = lower_bound(p, np, s[r]);
    int64_t hi = upper_bound(p, np, e[r]) - 1;
    for (int64_t q = lo; q <= hi; ++q) {
      p_out[k] = p[q];
      run_of[k] = r;
      idx_of[k] = q;
      ++k;
    }
  }
  return k;
}

/* primitives.cpp:88-100: bin = upper_bound(p2, p1[i]) - 1, keep on equality. */
int64_t orq_idx_in_idx(const int64_t* p1, int64_t n1, const int64_t* p2, int64_t n2,
                       int64_t* p_out, int64_t* idx1, int64_t* idx2) {
  int64_t k = 0;
  for (int64_t i = 0; i < n1; ++i) {
    int64_t b = upper_bound(p2, n2, p1[i]) - 1;
    if (b >= 0 && p1[i] == p2[b]) {
      p_out[k] = p1[i];
      idx1[k] = i;
      idx2[k] = b;
      ++k;
    }
  }
  return k;
}

/* primitives.cpp:349-360 */
int64_t orq_plain_mask_to_rle(const uint8_t* bits, int64_t n, int64_t* s, int64_t* e) {
  int64_t k = 0;
  int prev = 0;
  for (int64_t i = 0; i < n; ++i) {
    int bit = bits[i] != 0;
    if (bit && !prev) s[k] = i;
    if (!bit && prev) e[k++] = i - 1;
    prev = bit;
  }
  if (prev) e[k++] = n - 1;
  return k;
}

/* primitives.cpp:362-368 */
int64_t orq_plain_mask_to_index(const uint8_t* bits, int64_t n, int64_t* p) {
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i)
    if (bits[i]) p[k++] = i;
  return k;
}

/* primitives.cpp:370-379: s' = exclusive cumsum of lengths, e' = s' + l - 1. */
int64_t orq_compact_rle(const int64_t* s, const int64_t* e, int64_t nr, int64_t* s_out,
                        int64_t* e_out) {
  int64_t at = 0;
  for (int64_t i = 0; i < nr; ++i) {
    int64_t l = e[i] - s[i] + 1;
    s_out[i] = at;
    e_out[i] = at + l - 1;
    at += l;
  }
  return at;
}

static int64_t load_int(int dtype, const void* v, int64_t i) {
  switch (dtype) {
    case I8: return ((const int8_t*)v)[i];
    case I16: return ((const int16_t*)v)[i];
    case I32: return ((const int32_t*)v)[i];
    default: return ((const int64_t*)v)[i];
  }
}

static int64_t wrap_to(int dtype, int64_t x) {
  switch (dtype) {
    case I8: return (int8_t)(uint8_t)x;
    case I16: return (int16_t)(uint16_t)x;
    case I32: return (int32_t)(uint32_t)x;
    default: return x;
  }
}

/* column.cpp:283-297: cast storage to the logical type, then
 * x = T(x + center) at the logical width. */
int64_t orq_plain_to_rle_int(int dtype, const void* values, int64_t n, int64_t* s, int64_t* e) {
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (i == 0 || load_int(dtype, values, i) != load_int(dtype, values, i - 1)) {
      if (k > 0) e[k - 1] = i - 1;
      s[k++] = i;
    }
  }
  if (k > 0) e[k - 1] = n - 1;
  return k;
}

void orq_decode_plain_int(int dtype, const void* values, int64_t n, int logical,
                          int has_center, int64_t center, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t x = wrap_to(logical, load_int(dtype, values, i));
    if (has_center) x = wrap_to(logical, (int64_t)((uint64_t)x + (uint64_t)center));
    out[i] = x;
  }
}

static int cmp_i64(int64_t x, int op, int64_t y) {
  switch (op) {
    case LT: return x < y;
    case LE: return x <= y;
    case EQ: return x == y;
    case NE: return x != y;
    case GE: return x >= y;
    default: return x > y;
  }
}

static uint64_t arith_u64(int64_t x, int op, int64_t y) {
  switch (op) {
    case ADD: return (uint64_t)x + (uint64_t)y;
    case SUB: return (uint64_t)x - (uint64_t)y;
    default: return (uint64_t)x * (uint64_t)y;
  }
}

/* align.cpp compare_scalar, `case Encoding::Rle`: per-run flag, keep the
 * passing runs' s/e unmerged. */
int64_t orq_rle_compare_scalar_i64(const int64_t* v, const int64_t* s, const int64_t* e,
                                   int64_t nr, int op, int64_t k, int64_t* s_out,
                                   int64_t* e_out) {
  int64_t m = 0;
  for (int64_t i = 0; i < nr; ++i) {
    if (cmp_i64(v[i], op, k)) {
      s_out[m] = s[i];
      e_out[m] = e[i];
      ++m;
    }
  }
  return m;
}

/* Fragments of the RLE x RLE positional intersection enumerated by a
 * two-pointer walk (same set and order as primitives.cpp:15-46), each
 * contributing (va op vb) * len to the int64 SUM (groupby.cpp:82-89). */
int64_t orq_sum_rle_binop_i64(const int64_t* va, const int64_t* sa, const int64_t* ea,
                              int64_t ra, const int64_t* vb, const int64_t* sb, const int64_t* eb,
                              int64_t rb, int op) {
  uint64_t acc = 0;
  int64_t i = 0, j = 0;
  while (i < ra && j < rb) {
    int64_t lo = sa[i] > sb[j] ? sa[i] : sb[j];
    int64_t hi = ea[i] < eb[j] ? ea[i] : eb[j];
    if (lo <= hi) acc += arith_u64(va[i], op, vb[j]) * (uint64_t)(hi - lo + 1);
    if (ea[i] < eb[j]) ++i;
    else if (eb[j] < ea[i]) ++j;
    else { ++i; ++j; }
  }
  return (int64_t)acc;
}

/* Advances *r to the first run whose end is >= pos; returns the run index
 * if it contains pos, else -1. */
static int64_t run_at(const int64_t* s, const int64_t* e, int64_t nr, int64_t* r, int64_t pos) {
  while (*r < nr && e[*r] < pos) ++*r;
  if (*r < nr && s[*r] <= pos) return *r;
  return -1;
}

int64_t orq_filtered_sum_rle_idx_rle(const int64_t* cv, const int64_t* cs, const int64_t* ce,
                                     int64_t rc, int cmp, int64_t k, const int64_t* av,
                                     const int64_t* as, const int64_t* ae, int64_t ra,
                                     const int64_t* bv, const int64_t* bp, int64_t nb, int op) {
  uint64_t acc = 0;
  int64_t ic = 0, ia = 0;
  for (int64_t q = 0; q < nb; ++q) {
    int64_t pos = bp[q];
    int64_t rcix = run_at(cs, ce, rc, &ic, pos);
    if (rcix < 0 || !cmp_i64(cv[rcix], cmp, k)) continue;
    int64_t raix = run_at(as, ae, ra, &ia, pos);
    if (raix < 0) continue;
    acc += arith_u64(av[raix], op, bv[q]);
  }
  return (int64_t)acc;
}

int64_t orq_filtered_sum_plain_idx_rle(int c_dtype, const void* c_values, int64_t n, int c_logical,
                                       int c_has_center, int64_t c_center, int cmp, int64_t k,
                                       const int64_t* av, const int64_t* as, const int64_t* ae,
                                       int64_t ra, const int64_t* bv, const int64_t* bp,
                                       int64_t nb, int op) {
  uint64_t acc = 0;
  int64_t ia = 0;
  for (int64_t q = 0; q < nb; ++q) {
    int64_t pos = bp[q];
    if (pos < 0 || pos >= n) continue;
    int64_t c = wrap_to(c_logical, load_int(c_dtype, c_values, pos));
    if (c_has_center) c = wrap_to(c_logical, (int64_t)((uint64_t)c + (uint64_t)c_center));
    if (!cmp_i64(c, cmp, k)) continue;
    int64_t raix = run_at(as, ae, ra, &ia, pos);
    if (raix < 0) continue;
    acc += arith_u64(av[raix], op, bv[q]);
  }
  return (int64_t)acc;
}

double orq_sum_f64(const double* x, int64_t n) {
  double sum = 0.0, comp = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double t = sum + x[i];
    if ((sum >= 0 ? sum : -sum) >= (x[i] >= 0 ? x[i] : -x[i])) comp += (sum - t) + x[i];
    else comp += (x[i] - t) + sum;
    sum = t;
  }
  return sum + comp;
}

/* ---------------------------------------------------------------------------
 * Streaming group-by restatement (see runq_oracle.h). Segments: disjoint
 * ascending closed ranges, one group slot each.
 * ------------------------------------------------------------------------- */

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <unistd.h>

static void neumaier_add(double* sum, double* comp, double x) {
  double t = *sum + x;
  if (fabs(*sum) >= fabs(x)) *comp += (*sum - t) + x;
  else *comp += (x - t) + *sum;
  *sum = t;
}

/* groupby.cpp:82-89 with shape weights = fragment lengths (align.cpp:20-70). */
void orq_seg_sum_runs_i64(const int64_t* ss, const int64_t* se, const int64_t* slot, int64_t nseg,
                          const int64_t* v, const int64_t* s, const int64_t* e, int64_t nr,
                          int64_t* out, int64_t* cnt) {
  int64_t i = 0, j = 0;
  while (i < nseg && j < nr) {
    int64_t lo = ss[i] > s[j] ? ss[i] : s[j];
    int64_t hi = se[i] < e[j] ? se[i] : e[j];
    if (lo <= hi) {
      int64_t len = hi - lo + 1;
      out[slot[i]] = (int64_t)((uint64_t)out[slot[i]] + (uint64_t)v[j] * (uint64_t)len);
      if (cnt) cnt[slot[i]] += len;
    }
    if (se[i] < e[j]) ++i;
    else if (e[j] < se[i]) ++j;
    else { ++i; ++j; }
  }
}

/* Points of an Index / RLE+Index / Plain+Index part located in segments by a
 * merge walk (idx_in_rle, primitives.cpp:48-61), weight 1 each. */
void orq_seg_sum_points_i64(const int64_t* ss, const int64_t* se, const int64_t* slot,
                            int64_t nseg, const int64_t* p, const int64_t* v, int64_t np,
                            int64_t shadow, int64_t* out, int64_t* cnt) {
  int64_t i = 0;
  for (int64_t q = 0; q < np && i < nseg; ++q) {
    while (i < nseg && se[i] < p[q]) ++i;
    if (i < nseg && ss[i] <= p[q]) {
      out[slot[i]] = (int64_t)((uint64_t)out[slot[i]] + (uint64_t)v[q] - (uint64_t)shadow);
      if (cnt) cnt[slot[i]] += 1;
    }
  }
}

/* --- a tiny pthread parallel-for: thread t of T takes rows [lo, hi) ------- */

typedef struct Fold {
  const int64_t *ss, *se, *slot;
  int64_t nseg, nslots, row0, n;
  int dtype, logical, has_center;
  int64_t center;
  const void* values;
  const double *x, *seg_scale;
  int d1_dtype, d2_dtype;
  const void *d1, *d2;
  int64_t m1, a1, m2, a2;
  void* part;          /* per-thread slot tables */
  int T;
} Fold;

typedef struct Job {
  Fold* f;
  int t;
  void (*fn)(Fold*, int);
} Job;

static void* job_main(void* p) {
  Job* j = (Job*)p;
  j->fn(j->f, j->t);
  return NULL;
}

static int n_threads(int64_t n) {
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  int T = c > 0 ? (int)c : 1;
  if (T > 64) T = 64;
  if (n < (int64_t)T * 65536) T = (int)(n / 65536) + 1;
  return T;
}

static void par_run(Fold* f, void (*fn)(Fold*, int)) {
  pthread_t th[64];
  Job jobs[64];
  for (int t = 0; t < f->T; ++t) {
    jobs[t].f = f;
    jobs[t].t = t;
    jobs[t].fn = fn;
    if (t > 0) pthread_create(&th[t], NULL, job_main, &jobs[t]);
  }
  fn(f, 0);
  for (int t = 1; t < f->T; ++t) pthread_join(th[t], NULL);
}

static void rows_of(const Fold* f, int t, int64_t* lo, int64_t* hi) {
  *lo = f->row0 + (int64_t)((__int128)f->n * t / f->T);
  *hi = f->row0 + (int64_t)((__int128)f->n * (t + 1) / f->T);
}

/* decode_values(PlainColumn) column.cpp:283-297 per row, Σ per slot. */
static void fold_int(Fold* f, int t) {
  int64_t lo, hi;
  rows_of(f, t, &lo, &hi);
  uint64_t* acc = (uint64_t*)f->part + (size_t)t * (size_t)f->nslots;
  for (int64_t i = lower_bound(f->se, f->nseg, lo); i < f->nseg && f->ss[i] < hi; ++i) {
    int64_t a = f->ss[i] > lo ? f->ss[i] : lo, b = f->se[i] < hi - 1 ? f->se[i] : hi - 1;
    uint64_t sum = 0;
    for (int64_t r = a; r <= b; ++r) {
      int64_t x = wrap_to(f->logical, load_int(f->dtype, f->values, r - f->row0));
      if (f->has_center) x = wrap_to(f->logical, (int64_t)((uint64_t)x + (uint64_t)f->center));
      sum += (uint64_t)x;
    }
    acc[f->slot[i]] += sum;
  }
}

void orq_seg_sum_plain_int(const int64_t* ss, const int64_t* se, const int64_t* slot, int64_t nseg,
                           int64_t nslots, int64_t row0, int64_t n, int dtype, const void* values,
                           int logical, int has_center, int64_t center, int64_t* out) {
  Fold f = {0};
  f.ss = ss; f.se = se; f.slot = slot; f.nseg = nseg; f.nslots = nslots; f.row0 = row0; f.n = n;
  f.dtype = dtype; f.values = values; f.logical = logical; f.has_center = has_center;
  f.center = center; f.T = n_threads(n);
  f.part = calloc((size_t)f.T * (size_t)nslots, sizeof(uint64_t));
  par_run(&f, fold_int);
  const uint64_t* part = (const uint64_t*)f.part;
  for (int t = 0; t < f.T; ++t)
    for (int64_t g = 0; g < nslots; ++g)
      out[g] = (int64_t)((uint64_t)out[g] + part[(size_t)t * (size_t)nslots + (size_t)g]);
  free(f.part);
}

static double factor(int dtype, const void* d, int64_t r, int64_t m, int64_t a) {
  return (double)(int64_t)((uint64_t)m * (uint64_t)load_int(dtype, d, r) + (uint64_t)a);
}

/* arith(x, f1) then arith(·, f2) in f64 (align.cpp:290-334), SUM float
 * (groupby.cpp:91-97) with weight 1 per row, Neumaier per thread. */
static void fold_f64(Fold* f, int t) {
  int64_t lo, hi;
  rows_of(f, t, &lo, &hi);
  double* ps = (double*)f->part + (size_t)t * (size_t)f->nslots * 2;
  for (int64_t i = lower_bound(f->se, f->nseg, lo); i < f->nseg && f->ss[i] < hi; ++i) {
    int64_t a = f->ss[i] > lo ? f->ss[i] : lo, b = f->se[i] < hi - 1 ? f->se[i] : hi - 1;
    double s0 = ps[2 * f->slot[i]], c0 = ps[2 * f->slot[i] + 1];
    for (int64_t r = a; r <= b; ++r) {
      double y = f->x[r - f->row0];
      if (f->d1) y = y * factor(f->d1_dtype, f->d1, r - f->row0, f->m1, f->a1);
      else if (f->seg_scale) y = y * f->seg_scale[i];
      if (f->d2) y = y * factor(f->d2_dtype, f->d2, r - f->row0, f->m2, f->a2);
      neumaier_add(&s0, &c0, y);
    }
    ps[2 * f->slot[i]] = s0;
    ps[2 * f->slot[i] + 1] = c0;
  }
}

void orq_seg_sum_plain_f64(const int64_t* ss, const int64_t* se, const int64_t* slot, int64_t nseg,
                           int64_t nslots, int64_t row0, int64_t n, const double* x,
                           const double* seg_scale, int d1_dtype, const void* d1, int64_t m1,
                           int64_t a1, int d2_dtype, const void* d2, int64_t m2, int64_t a2,
                           double* sum, double* comp) {
  Fold f = {0};
  f.ss = ss; f.se = se; f.slot = slot; f.nseg = nseg; f.nslots = nslots; f.row0 = row0; f.n = n;
  f.x = x; f.seg_scale = seg_scale; f.d1_dtype = d1_dtype; f.d1 = d1; f.m1 = m1; f.a1 = a1;
  f.d2_dtype = d2_dtype; f.d2 = d2; f.m2 = m2; f.a2 = a2; f.T = n_threads(n);
  f.part = calloc((size_t)f.T * (size_t)nslots * 2, sizeof(double));
  par_run(&f, fold_f64);
  const double* part = (const double*)f.part;
  for (int t = 0; t < f.T; ++t)
    for (int64_t g = 0; g < nslots; ++g) {
      const double* ps = part + ((size_t)t * (size_t)nslots + (size_t)g) * 2;
      neumaier_add(&sum[g], &comp[g], ps[0]);
      neumaier_add(&sum[g], &comp[g], ps[1]);
    }
  free(f.part);
}
