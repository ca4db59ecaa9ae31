/*
 * TEST INFRASTRUCTURE ONLY — see hs_oracle.h. Plain-C restatement of the
 * reference hsolve arithmetic (file:line cited per function, relative to
 * /root/reference/proj). Built by oracle/Makefile with -ffp-contract=off.
 */
#include "hs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

enum { ST_OK = 0, ST_CONFIG = 1, ST_NOT_SPD = 2, ST_SINGULAR = 3, ST_NUMERICAL = 4 };

/* ------------------------------------------------------------------ */
/* parallel-for over [0, count) with a fixed worker count               */

typedef void (*body_fn)(size_t i, void* ctx);
typedef struct {
  body_fn fn;
  void* ctx;
  size_t count;
  size_t stride;
  size_t first;
} pf_arg;

static void* pf_worker(void* p) {
  pf_arg* a = (pf_arg*)p;
  for (size_t i = a->first; i < a->count; i += a->stride) a->fn(i, a->ctx);
  return NULL;
}

static void parallel_for(size_t count, int threads, body_fn fn, void* ctx) {
  if (threads <= 1 || count < 2) {
    for (size_t i = 0; i < count; ++i) fn(i, ctx);
    return;
  }
  size_t w = (size_t)threads;
  if (w > count) w = count;
  pthread_t* th = (pthread_t*)malloc(w * sizeof(pthread_t));
  pf_arg* args = (pf_arg*)malloc(w * sizeof(pf_arg));
  for (size_t k = 0; k < w; ++k) {
    args[k] = (pf_arg){fn, ctx, count, w, k};
    pthread_create(&th[k], NULL, pf_worker, &args[k]);
  }
  for (size_t k = 0; k < w; ++k) pthread_join(th[k], NULL);
  free(th);
  free(args);
}

static size_t block_rows_of(size_t n, size_t b) { return (n + b - 1) / b; }
/* blocked_matrix.cpp:8-15 */
static size_t tri(size_t i, size_t j) { return i * (i + 1) / 2 + j; }

/* ------------------------------------------------------------------ */
/* dd.hpp:18-40 — Knuth TwoSum double-double                            */

typedef struct { double hi, lo; } dd_t;

static dd_t two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double err = (a - (s - bb)) + (b - bb);
  dd_t r = {s, err};
  return r;
}
static dd_t dd_add1(dd_t acc, double x) {
  const dd_t t = two_sum(acc.hi, x);
  const double lo = acc.lo + t.lo;
  const double hi = t.hi + lo;
  dd_t r = {hi, lo - (hi - t.hi)};
  return r;
}
static double dd_value(dd_t a) { return a.hi + a.lo; }

/* ------------------------------------------------------------------ */
/* genmat.cpp:16-34 — splitmix64 counter RNG                            */

static uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t hso_rng_at(uint64_t key, uint64_t counter) { return mix(key ^ mix(counter)); }
double hso_uniform01(uint64_t key, uint64_t counter) {
  return (double)(hso_rng_at(key, counter) >> 11) * 0x1.0p-53;
}
double hso_uniform_pm1(uint64_t key, uint64_t counter) {
  return 2.0 * hso_uniform01(key, counter) - 1.0;
}

/* genmat.cpp:38-54 */
static const uint64_t kPointsStream = 0x706f696e74730001ull;
static const uint64_t kRhsStream = 0x7268730000000001ull;

int hso_generate_inputs(size_t n, size_t dim, uint64_t seed, double* out) {
  if (n == 0 || dim == 0) return ST_CONFIG;
  for (size_t i = 0; i < n; ++i) {
    const double t = (double)i * 0.01;
    for (size_t k = 0; k < dim; ++k) {
      double v;
      if (k == 0) {
        v = t;
      } else {
        const double omega = 1.0 + 0.5 * (double)(k - 1);
        const double noise =
            0.05 * hso_uniform_pm1(seed ^ kPointsStream, (uint64_t)i * dim + k);
        v = sin(omega * t) + noise;
      }
      out[i * dim + k] = v;
    }
  }
  return ST_OK;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* genmat.cpp:91-112: upper median (nth_element at size/2) of the distances
 * of a <=512-point stride subsample; 0 -> 1.0. The selected VALUE is unique,
 * so a full sort picks the same element nth_element does. */
double hso_median_pairwise_distance(const double* pts, size_t n, size_t dim) {
  const size_t m = n < 512 ? n : 512;
  if (m < 2) return 1.0;
  const size_t cnt = m * (m - 1) / 2;
  double* d = (double*)malloc(cnt * sizeof(double));
  size_t w = 0;
  for (size_t i = 0; i < m; ++i) {
    const size_t pi = i * n / m;
    for (size_t j = i + 1; j < m; ++j) {
      const size_t pj = j * n / m;
      double d2 = 0.0;
      for (size_t k = 0; k < dim; ++k) {
        const double dd = pts[pi * dim + k] - pts[pj * dim + k];
        d2 += dd * dd;
      }
      d[w++] = sqrt(d2);
    }
  }
  qsort(d, cnt, sizeof(double), cmp_double);
  const double mid = d[cnt / 2];
  free(d);
  return mid == 0.0 ? 1.0 : mid;
}

typedef struct {
  size_t n, b, dim;
  double sf2, sn2, inv2l2;
  const double* pts;
  double* out;
} gen_ctx;

/* genmat.cpp:128-152 — one block row of tiles */
static void gen_row(size_t i, void* p) {
  gen_ctx* g = (gen_ctx*)p;
  const size_t n = g->n, b = g->b, dim = g->dim;
  for (size_t j = 0; j <= i; ++j) {
    double* blk = g->out + tri(i, j) * b * b;
    for (size_t r = 0; r < b; ++r) {
      const size_t pr = i * b + r;
      for (size_t c = 0; c < b; ++c) {
        const size_t q = j * b + c;
        double v;
        if (pr >= n || q >= n) {
          v = (pr == q) ? 1.0 : 0.0;
        } else if (pr == q) {
          v = g->sf2 + g->sn2;
        } else {
          double d2 = 0.0;
          for (size_t k = 0; k < dim; ++k) {
            const double d = g->pts[pr * dim + k] - g->pts[q * dim + k];
            d2 += d * d;
          }
          v = g->sf2 * exp(-d2 * g->inv2l2);
        }
        blk[r * b + c] = v;
      }
    }
  }
}

/* genmat.cpp:114-154 */
int hso_generate_spd(size_t n, size_t b, double sigma_f2, double length_scale,
                     double sigma_n2, size_t dim, uint64_t seed, int threads,
                     double* out_packed) {
  if (!(sigma_f2 > 0.0) || !(sigma_n2 > 0.0)) return ST_CONFIG;
  if (n == 0 || b == 0 || dim == 0) return ST_CONFIG;
  double* pts = (double*)malloc(n * dim * sizeof(double));
  hso_generate_inputs(n, dim, seed, pts);
  const double ell =
      length_scale > 0.0 ? length_scale : hso_median_pairwise_distance(pts, n, dim);
  gen_ctx g = {n, b, dim, sigma_f2, sigma_n2, 1.0 / (2.0 * ell * ell), pts, out_packed};
  parallel_for(block_rows_of(n, b), threads, gen_row, &g);
  free(pts);
  return ST_OK;
}

/* genmat.cpp:156-162 */
void hso_generate_rhs(size_t n, size_t b, uint64_t seed, double* out) {
  const size_t pn = block_rows_of(n, b) * b;
  memset(out, 0, pn * sizeof(double));
  for (size_t i = 0; i < n; ++i) out[i] = hso_uniform_pm1(seed ^ kRhsStream, i);
}

/* ------------------------------------------------------------------ */
/* block_kernels.cpp:59-95 — one output block row                       */

typedef struct {
  size_t b, rows;
  const double* a;
  const double* x;
  double* y;
} symv_ctx;

/* Accumulation-order switch, for measuring the CG iteration envelope only
 * (tests/test_gpu_fullsize.py, tools/cg_envelope.py). 0 = the reference's
 * order: one running sum per output row over ascending j, c
 * (block_kernels.cpp:59-95). 1 = "tile partials": each tile's contribution
 * to a row is summed from 0 over its b columns and then added to the row in
 * ascending j, which is the accumulation class of the GPU SYMV (per-tile
 * partial slots added in a fixed order). Same products, different rounding. */
static int g_symv_order = 0;
void hso_set_symv_order(int order) { g_symv_order = order; }

static void symv_row(size_t row, void* p) {
  symv_ctx* s = (symv_ctx*)p;
  const size_t b = s->b;
  const int tiled = g_symv_order == 1;
  double* out = s->y + row * b;
  for (size_t r = 0; r < b; ++r) out[r] = 0.0;
  for (size_t j = 0; j < s->rows; ++j) {
    const double* xj = s->x + j * b;
    if (j < row) {
      const double* blk = s->a + tri(row, j) * b * b;
      for (size_t r = 0; r < b; ++r) {
        double acc = tiled ? 0.0 : out[r];
        for (size_t c = 0; c < b; ++c) acc += blk[r * b + c] * xj[c];
        out[r] = tiled ? out[r] + acc : acc;
      }
    } else if (j == row) {
      const double* blk = s->a + tri(row, row) * b * b;
      for (size_t r = 0; r < b; ++r) {
        double acc = tiled ? 0.0 : out[r];
        for (size_t c = 0; c < b; ++c) {
          const double v = (c <= r) ? blk[r * b + c] : blk[c * b + r];
          acc += v * xj[c];
        }
        out[r] = tiled ? out[r] + acc : acc;
      }
    } else {
      const double* blk = s->a + tri(j, row) * b * b;
      for (size_t r = 0; r < b; ++r) {
        double acc = tiled ? 0.0 : out[r];
        for (size_t c = 0; c < b; ++c) acc += blk[c * b + r] * xj[c];
        out[r] = tiled ? out[r] + acc : acc;
      }
    }
  }
}

void hso_symv(size_t n, size_t b, const double* a, const double* x, double* y,
              int threads) {
  symv_ctx s = {b, block_rows_of(n, b), a, x, y};
  parallel_for(s.rows, threads, symv_row, &s);
}

/* block_kernels.cpp:102-116 + cg_solver.cpp:189-205 (dot_reduce chain) */
static dd_t dot_rows(size_t rows, size_t b, const double* u, const double* v) {
  dd_t acc = {0.0, 0.0};
  for (size_t i = 0; i < rows; ++i) {
    double part = 0.0;
    for (size_t c = 0; c < b; ++c) part += u[i * b + c] * v[i * b + c];
    acc = dd_add1(acc, part);
  }
  return acc;
}

double hso_dot(size_t n, size_t b, const double* u, const double* v) {
  return dd_value(dot_rows(block_rows_of(n, b), b, u, v));
}

/* ------------------------------------------------------------------ */
/* cg_solver.cpp:223-368 — homogeneous CG                               */

int hso_solve_cg(size_t n, size_t b, const double* a, const double* rhs,
                 double eps, size_t max_iters, size_t recompute_interval,
                 int threads, double* x, double* stats, double* trace,
                 size_t trace_cap, int64_t* err_iter) {
  if (!(eps > 0.0) || b == 0 || n == 0) return ST_CONFIG;
  const size_t rows = block_rows_of(n, b);
  const size_t pn = rows * b;
  double* r = (double*)malloc(pn * sizeof(double));
  double* s = (double*)malloc(pn * sizeof(double));
  double* t = (double*)malloc(pn * sizeof(double));
  memcpy(r, rhs, pn * sizeof(double));
  memcpy(s, rhs, pn * sizeof(double));
  memset(t, 0, pn * sizeof(double));
  memset(x, 0, pn * sizeof(double));
  size_t iterations = 0, recomputations = 0;
  int status = ST_OK;

  const double u0 = dd_value(dot_rows(rows, b, rhs, rhs)); /* :243 */
  if (!isfinite(u0)) {
    status = ST_NUMERICAL;
    if (err_iter) *err_iter = 0;
    goto done;
  }
  const double limit = eps * eps * u0; /* :248 */
  double u = u0;
  if (u > limit) {
    for (size_t iter = 1; iter <= max_iters; ++iter) {
      hso_symv(n, b, a, s, t, threads); /* line 4 */
      const double st = dd_value(dot_rows(rows, b, s, t));
      const double alpha = u / st;
      if (!isfinite(alpha)) {
        status = ST_NUMERICAL;
        if (err_iter) *err_iter = (int64_t)iter;
        goto done;
      }
      for (size_t i = 0; i < pn; ++i) x[i] += alpha * s[i]; /* line 6 */
      const int recompute = recompute_interval > 0 && iter % recompute_interval == 0;
      if (recompute) { /* :277-298 */
        ++recomputations;
        hso_symv(n, b, a, x, t, threads);
        for (size_t i = 0; i < pn; ++i) r[i] = rhs[i] - t[i];
      } else { /* line 7, axpy with -alpha */
        const double na = -alpha;
        for (size_t i = 0; i < pn; ++i) r[i] += na * t[i];
      }
      const double v = u;
      u = dd_value(dot_rows(rows, b, r, r));
      if (!(u >= 0.0) || !isfinite(u)) {
        status = ST_NUMERICAL;
        if (err_iter) *err_iter = (int64_t)iter;
        goto done;
      }
      const double beta = u / v;
      for (size_t i = 0; i < pn; ++i) s[i] = r[i] + beta * s[i]; /* line 11 */
      iterations = iter;
      if (trace && iter - 1 < trace_cap) {
        trace[3 * (iter - 1) + 0] = u;
        trace[3 * (iter - 1) + 1] = alpha;
        trace[3 * (iter - 1) + 2] = beta;
      }
      if (u <= limit) break;
    }
  }
  stats[2] = (u <= limit) ? 1.0 : 0.0;
  /* :360-365 exit diagnostics */
  hso_symv(n, b, a, x, t, threads);
  for (size_t i = 0; i < pn; ++i) r[i] = rhs[i] - t[i];
  stats[4] = sqrt(dd_value(dot_rows(rows, b, r, r)));
done:
  stats[0] = (double)iterations;
  stats[1] = (double)recomputations;
  stats[3] = u0;
  free(r);
  free(s);
  free(t);
  return status;
}

/* ------------------------------------------------------------------ */
/* block_kernels.cpp:9-57                                               */

int hso_potf_block(double* d, size_t b, int64_t* pivot) {
  for (size_t p = 0; p < b; ++p) {
    for (size_t q = 0; q < p; ++q) {
      double acc = d[p * b + q];
      for (size_t k = 0; k < q; ++k) acc -= d[p * b + k] * d[q * b + k];
      d[p * b + q] = acc / d[q * b + q];
    }
    double acc = d[p * b + p];
    for (size_t k = 0; k < p; ++k) acc -= d[p * b + k] * d[p * b + k];
    if (!(acc > 0.0)) {
      if (pivot) *pivot = (int64_t)p;
      return ST_NOT_SPD;
    }
    d[p * b + p] = sqrt(acc);
  }
  return ST_OK;
}

int hso_trsm_block(double* x, const double* l, size_t b, int64_t* index) {
  for (size_t c = 0; c < b; ++c) {
    const double diag = l[c * b + c];
    if (diag == 0.0 || isnan(diag)) {
      if (index) *index = (int64_t)c;
      return ST_SINGULAR;
    }
  }
  for (size_t r = 0; r < b; ++r) {
    double* xr = x + r * b;
    for (size_t c = 0; c < b; ++c) {
      double acc = xr[c];
      for (size_t k = 0; k < c; ++k) acc -= xr[k] * l[c * b + k];
      xr[c] = acc / l[c * b + c];
    }
  }
  return ST_OK;
}

void hso_gemm_update(double* c, const double* p, const double* q, size_t b) {
  for (size_t r = 0; r < b; ++r)
    for (size_t col = 0; col < b; ++col) {
      double acc = 0.0;
      for (size_t k = 0; k < b; ++k) acc += p[r * b + k] * q[col * b + k];
      c[r * b + col] -= acc;
    }
}

void hso_syrk_update(double* c, const double* p, size_t b) {
  for (size_t r = 0; r < b; ++r)
    for (size_t col = 0; col <= r; ++col) {
      double acc = 0.0;
      for (size_t k = 0; k < b; ++k) acc += p[r * b + k] * p[col * b + k];
      c[r * b + col] -= acc;
    }
}

/* ------------------------------------------------------------------ */
/* cholesky_solver.cpp:158-238 — homogeneous right-looking factor       */

typedef struct {
  double* a;
  size_t b, j, rows;
  size_t* pairs; /* (i,k) flattened */
  int status;
} fac_ctx;

static void trsm_task(size_t idx, void* p) {
  fac_ctx* f = (fac_ctx*)p;
  const size_t i = f->j + 1 + idx;
  const size_t bb = f->b * f->b;
  hso_trsm_block(f->a + tri(i, f->j) * bb, f->a + tri(f->j, f->j) * bb, f->b, NULL);
}

static void step3_task(size_t idx, void* p) {
  fac_ctx* f = (fac_ctx*)p;
  const size_t i = f->pairs[2 * idx], k = f->pairs[2 * idx + 1];
  const size_t bb = f->b * f->b;
  if (k == i)
    hso_syrk_update(f->a + tri(i, i) * bb, f->a + tri(i, f->j) * bb, f->b);
  else
    hso_gemm_update(f->a + tri(i, k) * bb, f->a + tri(i, f->j) * bb,
                    f->a + tri(k, f->j) * bb, f->b);
}

int hso_factorize(size_t n, size_t b, double* a, int threads, int64_t* err_row,
                  int64_t* err_pivot) {
  if (n == 0 || b == 0) return ST_CONFIG;
  const size_t rows = block_rows_of(n, b);
  const size_t bb = b * b;
  size_t* pairs = (size_t*)malloc(2 * (rows * (rows + 1) / 2 + 1) * sizeof(size_t));
  fac_ctx f = {a, b, 0, rows, pairs, 0};
  for (size_t j = 0; j < rows; ++j) {
    int64_t piv = 0;
    /* Step 1 (:170-176) */
    if (hso_potf_block(a + tri(j, j) * bb, b, &piv) != ST_OK) {
      if (err_row) *err_row = (int64_t)j;
      if (err_pivot) *err_pivot = piv;
      free(pairs);
      return ST_NOT_SPD;
    }
    f.j = j;
    /* Step 2 (:183-189) */
    parallel_for(rows - j - 1, threads, trsm_task, &f);
    /* Step 3 (:125-156, :199-206) */
    size_t np = 0;
    for (size_t i = j + 1; i < rows; ++i)
      for (size_t k = j + 1; k <= i; ++k) {
        pairs[2 * np] = i;
        pairs[2 * np + 1] = k;
        ++np;
      }
    parallel_for(np, threads, step3_task, &f);
  }
  free(pairs);
  /* check_finite (:222-238) */
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j <= i; ++j) {
      const double* blk = a + tri(i, j) * bb;
      for (size_t r = 0; r < b; ++r) {
        const size_t cols = (i == j) ? r + 1 : b;
        for (size_t c = 0; c < cols; ++c)
          if (!isfinite(blk[r * b + c])) return ST_NUMERICAL;
      }
    }
  return ST_OK;
}

/* block_kernels.cpp:154-189 */
static void gemv_sub(const double* m, const double* x, double* y, size_t b) {
  for (size_t r = 0; r < b; ++r) {
    double acc = 0.0;
    for (size_t c = 0; c < b; ++c) acc += m[r * b + c] * x[c];
    y[r] -= acc;
  }
}
static void gemv_transpose_sub(const double* m, const double* x, double* y, size_t b) {
  for (size_t r = 0; r < b; ++r) {
    double acc = 0.0;
    for (size_t c = 0; c < b; ++c) acc += m[c * b + r] * x[c];
    y[r] -= acc;
  }
}
static int lower_solve(const double* l, double* y, size_t b) {
  for (size_t r = 0; r < b; ++r) {
    const double diag = l[r * b + r];
    if (diag == 0.0 || isnan(diag)) return ST_SINGULAR;
    double acc = y[r];
    for (size_t c = 0; c < r; ++c) acc -= l[r * b + c] * y[c];
    y[r] = acc / diag;
  }
  return ST_OK;
}
static int lower_transpose_solve(const double* l, double* y, size_t b) {
  for (size_t rr = b; rr-- > 0;) {
    const double diag = l[rr * b + rr];
    if (diag == 0.0 || isnan(diag)) return ST_SINGULAR;
    double acc = y[rr];
    for (size_t c = rr + 1; c < b; ++c) acc -= l[c * b + rr] * y[c];
    y[rr] = acc / diag;
  }
  return ST_OK;
}

/* cholesky_solver.cpp:23-31 */
int hso_forward_substitute(size_t n, size_t b, const double* l, const double* rhs,
                           double* y) {
  const size_t rows = block_rows_of(n, b), bb = b * b;
  memcpy(y, rhs, rows * b * sizeof(double));
  for (size_t i = 0; i < rows; ++i) {
    for (size_t j = 0; j < i; ++j) gemv_sub(l + tri(i, j) * bb, y + j * b, y + i * b, b);
    if (lower_solve(l + tri(i, i) * bb, y + i * b, b) != ST_OK) return ST_SINGULAR;
  }
  return ST_OK;
}

/* cholesky_solver.cpp:33-42 */
int hso_back_substitute(size_t n, size_t b, const double* l, const double* y,
                        double* x) {
  const size_t rows = block_rows_of(n, b), bb = b * b;
  memcpy(x, y, rows * b * sizeof(double));
  for (size_t ii = rows; ii-- > 0;) {
    for (size_t j = ii + 1; j < rows; ++j)
      gemv_transpose_sub(l + tri(j, ii) * bb, x + j * b, x + ii * b, b);
    if (lower_transpose_solve(l + tri(ii, ii) * bb, x + ii * b, b) != ST_OK)
      return ST_SINGULAR;
  }
  return ST_OK;
}

/* cholesky_solver.cpp:275-331 */
int hso_solve_spd(size_t n, size_t b, double* a, const double* rhs, int threads,
                  double* x, double* stats, int64_t* err_row, int64_t* err_pivot) {
  const size_t rows = block_rows_of(n, b), pn = rows * b;
  const size_t vals = rows * (rows + 1) / 2 * b * b;
  double* orig = (double*)malloc(vals * sizeof(double));
  memcpy(orig, a, vals * sizeof(double));
  int st = hso_factorize(n, b, a, threads, err_row, err_pivot);
  if (st == ST_OK) {
    double* y = (double*)malloc(pn * sizeof(double));
    st = hso_forward_substitute(n, b, a, rhs, y);
    if (st == ST_OK) st = hso_back_substitute(n, b, a, y, x);
    if (st == ST_OK && stats) {
      hso_symv(n, b, orig, x, y, threads);
      for (size_t i = 0; i < pn; ++i) y[i] = rhs[i] - y[i];
      stats[0] = sqrt(hso_dot(n, b, y, y));
    }
    free(y);
  }
  free(orig);
  return st;
}

/* partition.cpp:11-47 */
size_t hso_partition_for_fraction(double fraction, size_t block_rows) {
  if (!(fraction >= 0.0 && fraction <= 1.0) || block_rows == 0) return (size_t)-1;
  return (size_t)floor(fraction * (double)block_rows + 0.5);
}

size_t hso_cholesky_border(double fraction, size_t column, size_t block_rows) {
  if (!(fraction >= 0.0 && fraction <= 1.0) || column >= block_rows) return (size_t)-1;
  const size_t nn = block_rows, t = nn - 1 - column;
  const double budget = fraction * (double)(t * (t + 1) / 2);
  for (size_t beta = column + 1; beta <= nn; ++beta) {
    const size_t k = beta - column;
    const size_t below = (t * (t + 1) - (k - 1) * k) / 2;
    if ((double)below <= budget) return beta;
  }
  return nn;
}
