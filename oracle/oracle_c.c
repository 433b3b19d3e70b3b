/*
 * TEST INFRASTRUCTURE ONLY -- the parity oracle, never the product.
 *
 * Plain-C, single-threaded restatement of the reference's CPU algorithms for
 * the Q-less tall-skinny QR hot path (reference = /root/reference/proj,
 * namespace skinnyqr).  Every function cites the reference file:line it
 * follows.  Parity is PINNED: tests/test_oracle.py checks this file against
 * (a) the SPEC worked examples the compiled reference honours,
 * (b) golden vectors under tests/golden/ produced by the unmodified reference
 * (tests/golden/make_golden.py, run in the build container), and (c) the
 * compiled reference itself (oracle/_ref/libskinnyqr_ref.so) when present.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this.  The product (paper_2603_20889_b200) never links or calls it.
 *
 * Conventions: column-major FP64, element (i,j) of an m x n matrix with
 * leading dimension ld at a[j*ld + i] (types.hpp:79,94).  Status codes mirror
 * the reference's exception classes (types.hpp:11-77).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#define ORC_OK 0
#define ORC_E_DIMENSION (-1)
#define ORC_E_ARGUMENT (-2)
#define ORC_E_BREAKDOWN (-3)
#define ORC_E_SINGULAR (-4)
#define ORC_E_ZERO_MATRIX (-5)
#define ORC_E_RANK_DEFICIENT (-6)
#define ORC_E_NOCONVERGENCE (-7)

typedef long long i64;

/* ------------------------------------------------------------------------- */
/* counter-based random stream and controlled-spectrum generator              */
/* ------------------------------------------------------------------------- */

/* matgen.cpp:8-13 -- SplitMix64 finaliser over seed + (index+1)*golden. */
uint64_t orc_mix64(uint64_t seed, uint64_t index) {
  uint64_t z = seed + (index + 1u) * 0x9E3779B97F4A7C15ull;
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

/* matgen.cpp:15-17 -- top 53 bits scaled to [0,1). */
double orc_uniform01(uint64_t seed, uint64_t index) {
  return (double)(orc_mix64(seed, index) >> 11) * 0x1.0p-53;
}

/* matgen.cpp:32-59 -- apply H_0 ... H_{nref-1} (last reflector first) to the
 * len x ncols matrix a; reflector jr's vector is drawn from stream positions
 * base + jr*len + i mapped to (-1,1). */
static void random_reflectors(double* a, i64 len, i64 ncols, uint64_t seed, uint64_t base,
                              i64 nref) {
  double* v = (double*)malloc(sizeof(double) * (size_t)len);
  for (i64 jr = nref - 1; jr >= 0; --jr) {
    double vv = 0.0;
    for (i64 i = 0; i < len; ++i) {
      v[i] = 2.0 * orc_uniform01(seed, base + (uint64_t)(jr * len + i)) - 1.0;
      vv += v[i] * v[i];
    }
    if (vv == 0.0) continue;
    const double scale = 2.0 / vv;
    for (i64 j = 0; j < ncols; ++j) {
      double* col = a + j * len;
      double s = 0.0;
      for (i64 i = 0; i < len; ++i) s += v[i] * col[i];
      const double wj = scale * s;
      for (i64 i = 0; i < len; ++i) col[i] -= v[i] * wj;
    }
  }
  free(v);
}

/* matgen.cpp:77-109 -- X = U diag(sigma) V^T, geometric or linear spectrum. */
int orc_generate(i64 m, i64 n, double kappa, int linear_decay, uint64_t seed, double* x) {
  if (n < 1 || m < n) return ORC_E_ARGUMENT;
  if (kappa < 1.0) return ORC_E_ARGUMENT;
  if (n == 1 && kappa != 1.0) return ORC_E_ARGUMENT;
  double* sigma = (double*)malloc(sizeof(double) * (size_t)n);
  if (n == 1) {
    sigma[0] = 1.0;
  } else if (!linear_decay) { /* matgen.cpp:67-69 */
    for (i64 i = 0; i < n; ++i) sigma[i] = pow(kappa, -(double)i / (double)(n - 1));
  } else { /* matgen.cpp:70-75 */
    const double lo = 1.0 / kappa;
    for (i64 i = 0; i < n; ++i) sigma[i] = 1.0 + ((double)i / (double)(n - 1)) * (lo - 1.0);
  }
  double* u = (double*)calloc((size_t)(m * n), sizeof(double));
  for (i64 j = 0; j < n; ++j) u[j * m + j] = 1.0;
  random_reflectors(u, m, n, seed, 0, n);
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < m; ++i) u[j * m + i] *= sigma[j];
  double* v = (double*)calloc((size_t)(n * n), sizeof(double));
  for (i64 j = 0; j < n; ++j) v[j * n + j] = 1.0;
  random_reflectors(v, n, n, seed, 1ull << 63, n); /* matgen.cpp:21-23 */
  memset(x, 0, sizeof(double) * (size_t)(m * n));
  for (i64 j = 0; j < n; ++j)
    for (i64 k = 0; k < n; ++k) {
      const double vjk = v[k * n + j];
      for (i64 i = 0; i < m; ++i) x[j * m + i] += vjk * u[k * m + i];
    }
  free(sigma); free(u); free(v);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* plans (plan.hpp:24-37, plan.cpp:9-32)                                       */
/* ------------------------------------------------------------------------- */

i64 orc_rows_per_block(i64 m, i64 k, i64 b) { return ((m + k * b - 1) / (k * b)) * b; }
i64 orc_block_begin(i64 m, i64 k, i64 b, i64 blk) {
  const i64 s = blk * orc_rows_per_block(m, k, b);
  return s < m ? s : m;
}
i64 orc_block_end(i64 m, i64 k, i64 b, i64 blk) {
  const i64 e = (blk + 1) * orc_rows_per_block(m, k, b);
  return e < m ? e : m;
}
/* plan.cpp:19-32: largest b with (b+n)*n doubles <= 192 KiB, at least 2n. */
i64 orc_default_tsqr_panel_rows(i64 n) {
  if (n < 1 || n > 64) return ORC_E_ARGUMENT;
  const i64 budget = 192 * 1024 / 8;
  const i64 fit = budget / n > n ? budget / n - n : 0;
  return fit > 2 * n ? fit : 2 * n;
}
/* plan.cpp:9-17: 32 KiB panel, at least n rows. */
i64 orc_default_gram_panel_rows(i64 n) {
  const i64 nn = n > 1 ? n : 1;
  const i64 b = 32 * 1024 / (8 * nn);
  return b > n ? b : n;
}

/* ------------------------------------------------------------------------- */
/* validation (types.cpp:40-48), sign normalisation (types.cpp:8-14)           */
/* ------------------------------------------------------------------------- */

static int all_finite(const double* p, i64 count) {
  for (i64 i = 0; i < count; ++i)
    if (!isfinite(p[i])) return 0;
  return 1;
}

int orc_validate(const double* x, i64 m, i64 n) {
  if (n < 1 || m < n) return ORC_E_DIMENSION;
  return all_finite(x, m * n) ? ORC_OK : ORC_E_ARGUMENT;
}

void orc_sign_normalize(double* r, i64 n) {
  for (i64 i = 0; i < n; ++i)
    if (r[i * n + i] < 0.0)
      for (i64 j = i; j < n; ++j) r[j * n + i] = -r[j * n + i];
}

/* ------------------------------------------------------------------------- */
/* trapezoidal Householder on the [W; R] pencil (tsqr.cpp:12-166)               */
/* ------------------------------------------------------------------------- */

typedef struct {
  i64 b, n, ld, active; /* ld = b + n */
  double *pen, *v, *w;
} pencil_t;

static void pencil_init(pencil_t* ws, i64 b, i64 n) {
  ws->b = b; ws->n = n; ws->ld = b + n; ws->active = 0;
  ws->pen = (double*)calloc((size_t)((b + n) * n), sizeof(double));
  ws->v = (double*)calloc((size_t)(b + n), sizeof(double));
  ws->w = (double*)calloc((size_t)(b + n), sizeof(double));
}
static void pencil_free(pencil_t* ws) { free(ws->pen); free(ws->v); free(ws->w); }

/* tsqr.cpp:27-40 -- triangle rows [0,n) -> [p,p+n) (walking down), W on top. */
static void pencil_load(pencil_t* ws, const double* panel, i64 ld, i64 p) {
  for (i64 j = 0; j < ws->n; ++j) {
    double* c = ws->pen + j * ws->ld;
    if (ws->active > 0)
      for (i64 i = ws->n - 1; i >= 0; --i) c[p + i] = c[i];
    memcpy(c, panel + j * ld, sizeof(double) * (size_t)p);
  }
  ws->active = p;
}

static double dotp(const double* a, const double* b, i64 len) {
  double s = 0.0;
  for (i64 i = 0; i < len; ++i) s += a[i] * b[i];
  return s;
}

/* tsqr.cpp:51-71 -- reflector for pencil column `col` over rows [col, col+p];
 * dlarfg convention: sigma = |tail|^2; sigma == 0 -> zero reflector, tau 0;
 * beta = -sign(pivot)*hypot with pivot > 0 -> -norm else +norm;
 * vec = tail/(pivot-beta), vec[col] = 1; column <- (beta, 0...). */
static double reflector(double* column, double* vec, i64 col, i64 p) {
  double* tail = column + col + 1;
  const double sigma = dotp(tail, tail, p);
  if (sigma == 0.0) {
    for (i64 i = 0; i <= p; ++i) vec[col + i] = 0.0;
    return 0.0;
  }
  const double pivot = column[col];
  const double norm = sqrt(pivot * pivot + sigma);
  const double beta = pivot > 0.0 ? -norm : norm;
  const double inv = 1.0 / (pivot - beta);
  vec[col] = 1.0;
  for (i64 i = 0; i < p; ++i) vec[col + 1 + i] = tail[i] * inv;
  column[col] = beta;
  for (i64 i = 0; i < p; ++i) tail[i] = 0.0;
  return (beta - pivot) / beta;
}

/* tsqr.cpp:75-133 -- paired reflectors (i, i+1), joint update of trailing
 * columns x -= a*v + c*w with a = tau_v (v.x), c = tau_w (w.x - a (v.w)). */
static void pencil_factor(pencil_t* ws) {
  const i64 n = ws->n, p = ws->active, ld = ws->ld;
  if (p == 0) return;
  double *v = ws->v, *w = ws->w;
  i64 i = 0;
  for (; i + 1 < n; i += 2) {
    const double tv = reflector(ws->pen + i * ld, v, i, p);
    if (tv != 0.0) { /* tsqr.cpp:90-95 */
      double* nx = ws->pen + (i + 1) * ld + i;
      const double s = tv * dotp(v + i, nx, p + 1);
      for (i64 t = 0; t < p + 1; ++t) nx[t] += -s * v[i + t];
    }
    const double tw = reflector(ws->pen + (i + 1) * ld, w, i + 1, p);
    if (i + 2 < n) { /* tsqr.cpp:99-126 */
      v[i + p + 1] = 0.0;
      w[i] = 0.0;
      const i64 len = p + 2;
      const double vtw = dotp(v + i, w + i, len);
      for (i64 j = i + 2; j < n; ++j) {
        double* xj = ws->pen + j * ld + i;
        double sv = 0.0, sw = 0.0;
        for (i64 t = 0; t < len; ++t) { sv += v[i + t] * xj[t]; sw += w[i + t] * xj[t]; }
        const double a = tv * sv;
        const double c = tw * (sw - a * vtw);
        for (i64 t = 0; t < len; ++t) xj[t] -= a * v[i + t] + c * w[i + t];
      }
    }
  }
  if (i < n) reflector(ws->pen + i * ld, v, i, p); /* tsqr.cpp:128-131 */
}

/* Exposed single step for the SPEC.md:316 example: fresh pencil, one panel. */
int orc_factor_trapezoidal(const double* w, i64 p, i64 n, i64 b, double* pencil_out) {
  if (b < 1 || n < 1 || p < 1 || p > b) return ORC_E_ARGUMENT;
  pencil_t ws; pencil_init(&ws, b, n);
  pencil_load(&ws, w, p, p);
  pencil_factor(&ws);
  memcpy(pencil_out, ws.pen, sizeof(double) * (size_t)((b + n) * n));
  pencil_free(&ws);
  return ORC_OK;
}

/* tsqr.cpp:137-158 -- stream `rows` rows (ld) in b-row panels through the
 * pencil; un-normalised n x n upper triangle out (strict lower = 0). */
static void block_qr_core(const double* x, i64 ld, i64 rows, i64 n, i64 b, double* r) {
  memset(r, 0, sizeof(double) * (size_t)(n * n));
  if (rows <= 0) return;
  pencil_t ws; pencil_init(&ws, b, n);
  for (i64 off = 0; off < rows; off += b) {
    const i64 p = rows - off < b ? rows - off : b;
    pencil_load(&ws, x + off, ld, p);
    pencil_factor(&ws);
  }
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i <= j; ++i) r[j * n + i] = ws.pen[j * ws.ld + i];
  pencil_free(&ws);
}

/* tsqr.cpp:162-166 */
int orc_block_qless_qr(const double* x, i64 m, i64 n, i64 b, double* r) {
  if (b < 1 || n < 1) return ORC_E_ARGUMENT;
  block_qr_core(x, m, m, n, b, r);
  return ORC_OK;
}

/* tsqr.cpp:168-184 -- Y is (k*n) x n, block i's triangle at rows [i*n, i*n+n). */
int orc_tsqr_stage1(const double* x, i64 m, i64 n, i64 k, i64 b, double* y) {
  if (k < 1 || b < 1) return ORC_E_ARGUMENT;
  const i64 ldy = k * n;
  memset(y, 0, sizeof(double) * (size_t)(ldy * n));
  double* r = (double*)malloc(sizeof(double) * (size_t)(n * n));
  for (i64 blk = 0; blk < k; ++blk) {
    const i64 lo = orc_block_begin(m, k, b, blk), hi = orc_block_end(m, k, b, blk);
    block_qr_core(x + lo, m, hi - lo, n, b, r);
    for (i64 j = 0; j < n; ++j)
      for (i64 i = 0; i <= j; ++i) y[j * ldy + blk * n + i] = r[j * n + i];
  }
  free(r);
  return ORC_OK;
}

/* tsqr.cpp:186-197 */
int orc_tsqr_qless(const double* x, i64 m, i64 n, i64 k, i64 b, double* r) {
  const int st = orc_validate(x, m, n);
  if (st) return st;
  if (n > 64) return ORC_E_ARGUMENT;
  if (k < 1 || b < 1) return ORC_E_ARGUMENT;
  double* y = (double*)malloc(sizeof(double) * (size_t)(k * n * n));
  orc_tsqr_stage1(x, m, n, k, b, y);
  block_qr_core(y, k * n, k * n, n, b, r);
  orc_sign_normalize(r, n);
  free(y);
  return ORC_OK;
}

/* tsqr.cpp:199-240 / small.cpp:34-64 -- classical unblocked Householder QR on
 * a full copy; columns whose tail is exactly zero are skipped. */
static void hhqr_inplace(double* work, i64 m, i64 n, double* r) {
  for (i64 j = 0; j < n; ++j) {
    double* cj = work + j * m;
    const i64 tail = m - j - 1;
    const double sigma = dotp(cj + j + 1, cj + j + 1, tail);
    if (sigma == 0.0) continue;
    const double pivot = cj[j];
    const double norm = sqrt(pivot * pivot + sigma);
    const double beta = pivot > 0.0 ? -norm : norm;
    const double tau = (beta - pivot) / beta;
    const double inv = 1.0 / (pivot - beta);
    for (i64 i = j + 1; i < m; ++i) cj[i] *= inv;
    cj[j] = beta;
    for (i64 jj = j + 1; jj < n; ++jj) {
      double* c = work + jj * m;
      const double s = tau * (c[j] + dotp(cj + j + 1, c + j + 1, tail));
      c[j] -= s;
      for (i64 i = j + 1; i < m; ++i) c[i] -= s * cj[i];
    }
  }
  memset(r, 0, sizeof(double) * (size_t)(n * n));
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i <= j && i < m; ++i) r[j * n + i] = work[j * m + i];
  orc_sign_normalize(r, n);
}

int orc_reference_hhqr(const double* x, i64 m, i64 n, double* r) {
  const int st = orc_validate(x, m, n);
  if (st) return st;
  double* work = (double*)malloc(sizeof(double) * (size_t)(m * n));
  memcpy(work, x, sizeof(double) * (size_t)(m * n));
  hhqr_inplace(work, m, n, r);
  free(work);
  return ORC_OK;
}

int orc_hhqr_small(const double* a, i64 m, i64 n, double* r) {
  if (m < n) return ORC_E_DIMENSION;
  double* work = (double*)malloc(sizeof(double) * (size_t)(m * n));
  memcpy(work, a, sizeof(double) * (size_t)(m * n));
  hhqr_inplace(work, m, n, r);
  free(work);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Gram kernels (gram.cpp:23-151; leaf semantics kernels_scalar.cpp:6-49)       */
/* ------------------------------------------------------------------------- */

/* op: 0 plain (syrk_upper), 1 solve (trsm_right_upper then syrk), 2 multiply
 * (gemm_right then syrk).  k blocks of b-row panels; block partials are summed
 * in ascending block order over the upper triangle, then mirrored
 * (gram.cpp:81-92). */
static void blocked_gram(const double* x, i64 m, i64 n, i64 k, i64 b, int op,
                         const double* factor, const double* inv_diag, double* c) {
  memset(c, 0, sizeof(double) * (size_t)(n * n));
  double* local = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* win = (double*)malloc(sizeof(double) * (size_t)(b * n));
  double* wout = (double*)malloc(sizeof(double) * (size_t)(b * n));
  for (i64 blk = 0; blk < k; ++blk) {
    const i64 lo = orc_block_begin(m, k, b, blk), hi = orc_block_end(m, k, b, blk);
    if (lo >= hi) continue;
    memset(local, 0, sizeof(double) * (size_t)(n * n));
    for (i64 off = lo; off < hi; off += b) {
      const i64 p = hi - off < b ? hi - off : b;
      const double* src = x + off;
      i64 lds = m;
      if (op != 0) {
        for (i64 j = 0; j < n; ++j) memcpy(win + j * p, x + off + j * m, sizeof(double) * (size_t)p);
        if (op == 1) { /* kernels_scalar.cpp:19-32: skip exact-zero r_ij, scale by 1/r_jj */
          for (i64 j = 0; j < n; ++j) {
            double* wj = win + j * p;
            for (i64 i = 0; i < j; ++i) {
              const double rij = factor[j * n + i];
              if (rij == 0.0) continue;
              const double* wi = win + i * p;
              for (i64 t = 0; t < p; ++t) wj[t] -= rij * wi[t];
            }
            for (i64 t = 0; t < p; ++t) wj[t] *= inv_diag[j];
          }
          src = win;
        } else { /* kernels_scalar.cpp:34-48 */
          for (i64 j = 0; j < n; ++j) {
            double* oj = wout + j * p;
            for (i64 t = 0; t < p; ++t) oj[t] = 0.0;
            for (i64 i = 0; i < n; ++i) {
              const double bij = factor[j * n + i];
              if (bij == 0.0) continue;
              const double* wi = win + i * p;
              for (i64 t = 0; t < p; ++t) oj[t] += bij * wi[t];
            }
          }
          src = wout;
        }
        lds = p;
      }
      for (i64 j = 0; j < n; ++j) /* kernels_scalar.cpp:6-17 */
        for (i64 i = 0; i <= j; ++i)
          local[j * n + i] += dotp(src + i * lds, src + j * lds, p);
    }
    for (i64 j = 0; j < n; ++j)
      for (i64 i = 0; i <= j; ++i) c[j * n + i] += local[j * n + i];
  }
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < j; ++i) c[i * n + j] = c[j * n + i];
  free(local); free(win); free(wout);
}

/* gram.cpp:113-121 */
int orc_tsmttsm(const double* x, i64 m, i64 n, i64 k, i64 b, double* c) {
  if (k < 1 || b < 1) return ORC_E_ARGUMENT;
  if (!all_finite(x, m * n)) return ORC_E_ARGUMENT;
  blocked_gram(x, m, n, k, b, 0, NULL, NULL, c);
  return ORC_OK;
}

/* gram.cpp:106-111 */
double orc_trsm_diag_tolerance(const double* r, i64 n) {
  double mx = 0.0;
  for (i64 j = 0; j < n; ++j) mx = fmax(mx, fabs(r[j * n + j]));
  return (double)n * DBL_EPSILON * mx;
}

/* gram.cpp:123-140 */
int orc_tsmRttsmR(const double* x, i64 m, i64 n, const double* r, i64 k, i64 b, double* c,
                  i64* err_index) {
  if (k < 1 || b < 1) return ORC_E_ARGUMENT;
  const double dtol = orc_trsm_diag_tolerance(r, n);
  double* inv = (double*)malloc(sizeof(double) * (size_t)n);
  for (i64 j = 0; j < n; ++j) {
    if (fabs(r[j * n + j]) <= dtol) {
      if (err_index) *err_index = j;
      free(inv);
      return ORC_E_SINGULAR;
    }
    inv[j] = 1.0 / r[j * n + j];
  }
  blocked_gram(x, m, n, k, b, 1, r, inv, c);
  free(inv);
  return ORC_OK;
}

/* gram.cpp:142-151 */
int orc_tsmmttsmm(const double* x, i64 m, i64 n, const double* bm, i64 k, i64 b, double* c) {
  if (k < 1 || b < 1) return ORC_E_ARGUMENT;
  if (!all_finite(bm, n * n)) return ORC_E_ARGUMENT;
  blocked_gram(x, m, n, k, b, 2, bm, NULL, c);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* n x n factorisations (gram_qr.cpp:36-121, small.cpp:9-32)                    */
/* ------------------------------------------------------------------------- */

/* gram_qr.cpp:36-58 -- left-looking upper Cholesky; breakdown when the pivot
 * is <= n*eps*max|c_jj|. */
int orc_cholesky(const double* c, i64 n, double* r, i64* err_index) {
  memset(r, 0, sizeof(double) * (size_t)(n * n));
  double cmax = 0.0;
  for (i64 j = 0; j < n; ++j) cmax = fmax(cmax, fabs(c[j * n + j]));
  const double tol = (double)n * DBL_EPSILON * cmax;
  for (i64 j = 0; j < n; ++j) {
    for (i64 i = 0; i < j; ++i) {
      double s = c[j * n + i];
      for (i64 t = 0; t < i; ++t) s -= r[i * n + t] * r[j * n + t];
      r[j * n + i] = s / r[i * n + i];
    }
    double d = c[j * n + j];
    for (i64 t = 0; t < j; ++t) d -= r[j * n + t] * r[j * n + t];
    if (d <= tol) {
      if (err_index) *err_index = j;
      return ORC_E_BREAKDOWN;
    }
    r[j * n + j] = sqrt(d);
  }
  return ORC_OK;
}

static double offdiag_norm(const double* a, i64 n) { /* gram_qr.cpp:17-23 */
  double s = 0.0;
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < j; ++i) s += a[j * n + i] * a[j * n + i];
  return sqrt(2.0 * s);
}

/* gram_qr.cpp:60-121 -- cyclic-by-row Jacobi, threshold 10*n*eps*|C|_F, at
 * most 30 sweeps, eigenpairs stable-sorted descending. */
int orc_eigh_small(const double* c, i64 n, double* values, double* vectors) {
  if (n > 128) return ORC_E_ARGUMENT;
  double* a = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* u = (double*)calloc((size_t)(n * n), sizeof(double));
  memcpy(a, c, sizeof(double) * (size_t)(n * n));
  for (i64 j = 0; j < n; ++j) u[j * n + j] = 1.0;
  double fro = 0.0;
  for (i64 t = 0; t < n * n; ++t) fro += c[t] * c[t];
  const double thr = 10.0 * (double)n * DBL_EPSILON * sqrt(fro);
  int converged = offdiag_norm(a, n) <= thr;
  for (int sweep = 0; sweep < 30 && !converged; ++sweep) {
    for (i64 p = 0; p + 1 < n; ++p)
      for (i64 q = p + 1; q < n; ++q) {
        const double apq = a[q * n + p];
        if (apq == 0.0) continue;
        const double app = a[p * n + p], aqq = a[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = t * cs;
        a[p * n + p] = app - t * apq;
        a[q * n + q] = aqq + t * apq;
        a[q * n + p] = 0.0;
        a[p * n + q] = 0.0;
        for (i64 i = 0; i < n; ++i) {
          if (i == p || i == q) continue;
          const double aip = a[p * n + i], aiq = a[q * n + i];
          a[p * n + i] = cs * aip - sn * aiq;
          a[q * n + i] = sn * aip + cs * aiq;
          a[i * n + p] = a[p * n + i];
          a[i * n + q] = a[q * n + i];
        }
        for (i64 i = 0; i < n; ++i) {
          const double uip = u[p * n + i], uiq = u[q * n + i];
          u[p * n + i] = cs * uip - sn * uiq;
          u[q * n + i] = sn * uip + cs * uiq;
        }
      }
    converged = offdiag_norm(a, n) <= thr;
  }
  if (!converged) { free(a); free(u); return ORC_E_NOCONVERGENCE; }
  /* stable descending order by insertion (gram_qr.cpp:107-110) */
  i64* perm = (i64*)malloc(sizeof(i64) * (size_t)n);
  for (i64 j = 0; j < n; ++j) perm[j] = j;
  for (i64 j = 1; j < n; ++j) {
    const i64 pj = perm[j];
    i64 t = j;
    while (t > 0 && a[perm[t - 1] * n + perm[t - 1]] < a[pj * n + pj]) { perm[t] = perm[t - 1]; --t; }
    perm[t] = pj;
  }
  for (i64 j = 0; j < n; ++j) {
    values[j] = a[perm[j] * n + perm[j]];
    memcpy(vectors + j * n, u + perm[j] * n, sizeof(double) * (size_t)n);
  }
  free(a); free(u); free(perm);
  return ORC_OK;
}

/* small.cpp:9-20 */
void orc_triangular_multiply(const double* a, const double* b, i64 n, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(n * n));
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i <= j; ++i) {
      double s = 0.0;
      for (i64 t = i; t <= j; ++t) s += a[t * n + i] * b[j * n + t];
      out[j * n + i] = s;
    }
}

/* small.cpp:22-32 (square case) */
void orc_small_multiply(const double* a, const double* b, i64 n, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(n * n));
  for (i64 j = 0; j < n; ++j)
    for (i64 t = 0; t < n; ++t) {
      const double btj = b[j * n + t];
      if (btj == 0.0) continue;
      for (i64 i = 0; i < n; ++i) out[j * n + i] += a[t * n + i] * btj;
    }
}

/* ------------------------------------------------------------------------- */
/* drivers (gram_qr.cpp:123-221, lstsq.cpp:13-61)                               */
/* ------------------------------------------------------------------------- */

/* gram_qr.cpp:123-131 */
int orc_cholqr2(const double* x, i64 m, i64 n, i64 k, i64 b, double* r, i64* err_index) {
  int st = orc_validate(x, m, n);
  if (st) return st;
  double* c = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* r1 = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* r2 = (double*)malloc(sizeof(double) * (size_t)(n * n));
  st = orc_tsmttsm(x, m, n, k, b, c);
  if (!st) st = orc_cholesky(c, n, r1, err_index);
  if (!st) st = orc_tsmRttsmR(x, m, n, r1, k, b, c, err_index);
  if (!st) st = orc_cholesky(c, n, r2, err_index);
  if (!st) orc_triangular_multiply(r2, r1, n, r);
  free(c); free(r1); free(r2);
  return st;
}

/* gram_qr.cpp:133-176 */
int orc_svqb_pass(const double* c, i64 n, double* bmat, double* z, double* sigma, i64* rank_out) {
  double* ds = (double*)malloc(sizeof(double) * (size_t)n);
  double* dsi = (double*)malloc(sizeof(double) * (size_t)n);
  double* cs = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* val = (double*)malloc(sizeof(double) * (size_t)n);
  double* vec = (double*)malloc(sizeof(double) * (size_t)(n * n));
  int st = ORC_OK;
  for (i64 j = 0; j < n; ++j) {
    const double d = c[j * n + j];
    ds[j] = d > 0.0 ? 1.0 / sqrt(d) : 1.0;
    dsi[j] = d > 0.0 ? sqrt(d) : 1.0;
  }
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < n; ++i) cs[j * n + i] = c[j * n + i] * ds[i] * ds[j];
  st = orc_eigh_small(cs, n, val, vec);
  if (!st && !(val[0] > 0.0)) st = ORC_E_ZERO_MATRIX;
  i64 rank = 0;
  if (!st) {
    const double tol = 10.0 * (double)n * DBL_EPSILON;
    while (rank < n && val[rank] >= tol * val[0]) ++rank;
    if (rank == 0) st = ORC_E_ZERO_MATRIX;
  }
  if (!st) {
    memset(bmat, 0, sizeof(double) * (size_t)(n * n));
    memset(z, 0, sizeof(double) * (size_t)(n * n));
    for (i64 j = 0; j < rank; ++j) {
      const double inv_sqrt = 1.0 / sqrt(val[j]);
      const double sqrt_l = sqrt(val[j]);
      for (i64 i = 0; i < n; ++i) {
        bmat[j * n + i] = ds[i] * vec[j * n + i] * inv_sqrt;
        z[i * n + j] = sqrt_l * vec[j * n + i] * dsi[i];
      }
    }
    st = orc_eigh_small(c, n, val, vec); /* gram_qr.cpp:171-174: sigma from unscaled C */
    if (!st)
      for (i64 j = 0; j < n; ++j) sigma[j] = sqrt(fmax(val[j], 0.0));
    *rank_out = rank;
  }
  free(ds); free(dsi); free(cs); free(val); free(vec);
  return st;
}

/* gram_qr.cpp:178-191 */
int orc_svqb2(const double* x, i64 m, i64 n, i64 k, i64 b, double* transform, double* z,
              double* sigma, i64* rank) {
  int st = orc_validate(x, m, n);
  if (st) return st;
  const size_t sq = sizeof(double) * (size_t)(n * n);
  double* c = (double*)malloc(sq);
  double *b1 = (double*)malloc(sq), *z1 = (double*)malloc(sq);
  double *b2 = (double*)malloc(sq), *z2 = (double*)malloc(sq);
  double* s2 = (double*)malloc(sizeof(double) * (size_t)n);
  i64 rank1 = 0;
  st = orc_tsmttsm(x, m, n, k, b, c);
  if (!st) st = orc_svqb_pass(c, n, b1, z1, sigma, &rank1);
  if (!st) st = orc_tsmmttsmm(x, m, n, b1, k, b, c);
  if (!st) st = orc_svqb_pass(c, n, b2, z2, s2, rank);
  if (!st) {
    orc_small_multiply(b1, b2, n, transform);
    orc_small_multiply(z2, z1, n, z);
  }
  free(c); free(b1); free(z1); free(b2); free(z2); free(s2);
  return st;
}

/* gram_qr.cpp:193-221 -- Q = X R^{-1}, column-oriented substitution with the
 * reciprocal diagonal, exact-zero r_ij skipped. */
int orc_reconstruct_q(const double* x, i64 m, i64 n, const double* r, double* q, i64* err_index) {
  const double dtol = orc_trsm_diag_tolerance(r, n);
  for (i64 j = 0; j < n; ++j)
    if (fabs(r[j * n + j]) <= dtol) {
      if (err_index) *err_index = j;
      return ORC_E_SINGULAR;
    }
  memcpy(q, x, sizeof(double) * (size_t)(m * n));
  for (i64 j = 0; j < n; ++j) {
    double* qj = q + j * m;
    for (i64 i = 0; i < j; ++i) {
      const double rij = r[j * n + i];
      if (rij == 0.0) continue;
      const double* qi = q + i * m;
      for (i64 t = 0; t < m; ++t) qj[t] -= rij * qi[t];
    }
    const double d = 1.0 / r[j * n + j];
    for (i64 t = 0; t < m; ++t) qj[t] *= d;
  }
  return ORC_OK;
}

/* lstsq.cpp:13-61 -- method 0 tsqr, 1 cholqr2, 2 svqb2; plans are the
 * reference defaults with k = `threads` (max_threads() there). */
int orc_solve_lstsq(const double* a, i64 m, i64 n, const double* rhs, int method, i64 threads,
                    double* x_out, double* residual, i64* err_index) {
  if (m < n + 1) return ORC_E_DIMENSION;
  int st = orc_validate(a, m, n);
  if (st) return st;
  if (!all_finite(rhs, m)) return ORC_E_ARGUMENT;
  const i64 ne = n + 1;
  double* ext = (double*)malloc(sizeof(double) * (size_t)(m * ne));
  memcpy(ext, a, sizeof(double) * (size_t)(m * n));
  memcpy(ext + m * n, rhs, sizeof(double) * (size_t)m);
  double* r = (double*)calloc((size_t)(ne * ne), sizeof(double));
  if (method == 0) {
    const i64 b = orc_default_tsqr_panel_rows(ne);
    st = b < 0 ? (int)b : orc_tsqr_qless(ext, m, ne, threads, b, r);
  } else if (method == 1) {
    st = orc_cholqr2(ext, m, ne, threads, orc_default_gram_panel_rows(ne), r, err_index);
  } else {
    const size_t sq = sizeof(double) * (size_t)(ne * ne);
    double *tr = (double*)malloc(sq), *z = (double*)malloc(sq);
    double* sg = (double*)malloc(sizeof(double) * (size_t)ne);
    i64 rank = 0;
    st = orc_svqb2(ext, m, ne, threads, orc_default_gram_panel_rows(ne), tr, z, sg, &rank);
    if (!st) st = orc_hhqr_small(z, ne, ne, r); /* lstsq.cpp:37-39 */
    free(tr); free(z); free(sg);
  }
  if (!st) {
    double mx = 0.0;
    for (i64 j = 0; j < n; ++j) mx = fmax(mx, fabs(r[j * ne + j]));
    const double dtol = (double)n * DBL_EPSILON * mx;
    for (i64 ii = n - 1; ii >= 0 && !st; --ii) {
      if (fabs(r[ii * ne + ii]) <= dtol) {
        if (err_index) *err_index = ii;
        st = ORC_E_RANK_DEFICIENT;
        break;
      }
      double s = r[n * ne + ii];
      for (i64 j = ii + 1; j < n; ++j) s -= r[j * ne + ii] * x_out[j];
      x_out[ii] = s / r[ii * ne + ii];
    }
    if (!st) *residual = fabs(r[n * ne + n]);
  }
  free(ext); free(r);
  return st;
}
