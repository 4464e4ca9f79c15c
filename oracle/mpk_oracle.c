/*
 * mpk_oracle.c -- CPU restatement of the reference mpkrylov hot path.
 *
 * TEST INFRASTRUCTURE ONLY (parity checker + bench.py CPU baseline).
 * Nothing in paper_2504_14498_b200/ links or calls this file.
 *
 * Restates, operation for operation, the reference at
 * /root/reference/pkg/src/mpkrylov (file:line cited per function).  Build
 * with -O2 -ffp-contract=off (no FMA contraction, no fast-math) so every
 * binary64 operation rounds exactly as CPython / numba do.  Pinned against
 * reference-generated golden vectors (tests/golden/, tests/test_oracle_golden.py).
 */
#include "mpk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define BUF 32

#include <pthread.h>

/* Row-parallel helper for the embarrassingly parallel kernels (SpMV rows,
 * axpy elements): results are bit-identical to the serial loop because
 * each output element is computed by exactly the reference's sequence. */
static int g_threads = 1;
static __thread int tl_serial = 0;
void orc_set_threads(int t) { g_threads = t < 1 ? 1 : t; }

typedef void (*range_fn)(void *arg, int64_t lo, int64_t hi);
typedef struct {
  range_fn f;
  void *arg;
  int64_t lo, hi;
} par_job_t;
static void *par_tramp(void *p) {
  par_job_t *j = (par_job_t *)p;
  tl_serial = 1;
  j->f(j->arg, j->lo, j->hi);
  return NULL;
}
static void par_for(int64_t n, range_fn f, void *arg) {
  int t = g_threads, i;
  if (tl_serial || t <= 1 || n < 16384) {
    f(arg, 0, n);
    return;
  }
  if (t > 64) t = 64;
  pthread_t th[64];
  par_job_t jobs[64];
  for (i = 0; i < t; ++i) {
    jobs[i].f = f;
    jobs[i].arg = arg;
    jobs[i].lo = n * i / t;
    jobs[i].hi = n * (i + 1) / t;
    if (i > 0) pthread_create(&th[i], NULL, par_tramp, &jobs[i]);
  }
  f(arg, jobs[0].lo, jobs[0].hi);
  for (i = 1; i < t; ++i) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------------ */
/* EFTs: _mccore.py:19-24 (two_sum), :34-51 (Dekker split / two_prod)  */
/* ------------------------------------------------------------------ */
void orc_two_sum(double a, double b, double *s, double *e) {
  double q = a + b;
  double bb = q - a;
  *e = (a - (q - bb)) + (b - bb);
  *s = q;
}

void orc_two_prod(double a, double b, double *p, double *e) {
  double pp = a * b;
  double t = 134217729.0 * a;
  double ah = t - (t - a);
  double al = a - ah;
  t = 134217729.0 * b;
  double bh = t - (t - b);
  double bl = b - bh;
  *e = ((ah * bh - pp) + ah * bl + al * bh) + al * bl;
  *p = pp;
}

/* renorm_terms _mccore.py:90-116, twin _kernels.py:24-81 */
void orc_renorm(const double *terms, int m, double *out, int k) {
  int i;
  if (m == 0) {
    for (i = 0; i < k; ++i) out[i] = 0.0;
    return;
  }
  for (i = 0; i < m; ++i) {
    if (!isfinite(terms[i])) {
      double s = 0.0;
      int j;
      for (j = 0; j < m; ++j) s += terms[j];
      out[0] = s;
      for (j = 1; j < k; ++j) out[j] = 0.0;
      return;
    }
  }
  double ext[BUF], e[BUF];
  int cnt = m;
  for (i = 0; i < m; ++i) ext[i] = terms[i];
  int passes = 0;
  for (;;) {
    /* _distill :54-79 -- VecSum bottom-up */
    double s = ext[cnt - 1];
    for (i = cnt - 2; i >= 0; --i) {
      double q, err;
      orc_two_sum(ext[i], s, &q, &err);
      e[i + 1] = err;
      s = q;
    }
    e[0] = s;
    /* zero-eliminating extraction */
    int n2 = 0;
    double eps = e[0];
    for (i = 1; i < cnt; ++i) {
      double q, enew;
      orc_two_sum(eps, e[i], &q, &enew);
      if (enew != 0.0) {
        ext[n2++] = q;
        eps = enew;
      } else {
        eps = q;
      }
    }
    ext[n2++] = eps;
    cnt = n2;
    passes += 1;
    /* _is_strict :82-87 */
    int ok = 1;
    for (i = 0; i < cnt - 1; ++i) {
      if (ext[i] + ext[i + 1] != ext[i]) {
        ok = 0;
        break;
      }
    }
    if (ok || passes >= 8) break;
  }
  for (i = 0; i < k; ++i) out[i] = (i < cnt) ? ext[i] + 0.0 : 0.0;
}

/* mc_add _mccore.py:129-155 (magnitude merge, ties prefer x) */
void orc_add(const double *x, const double *y, double *out, int k) {
  if (k == 1) {
    out[0] = x[0] + y[0];
    return;
  }
  double buf[8];
  int i = 0, j = 0, t = 0;
  while (i < k && j < k) {
    if (fabs(x[i]) >= fabs(y[j]))
      buf[t++] = x[i++];
    else
      buf[t++] = y[j++];
  }
  while (i < k) buf[t++] = x[i++];
  while (j < k) buf[t++] = y[j++];
  orc_renorm(buf, 2 * k, out, k);
}

/* mc_sub _mccore.py:158-159 = add of the negation (twin _sub1 :115-141) */
void orc_sub(const double *x, const double *y, double *out, int k) {
  double ny[4];
  int i;
  for (i = 0; i < k; ++i) ny[i] = -y[i];
  orc_add(x, ny, out, k);
}

/* mc_mul _mccore.py:162-186 (level scheme; last level plain products) */
void orc_mul(const double *x, const double *y, double *out, int k) {
  if (k == 1) {
    out[0] = x[0] * y[0];
    return;
  }
  double terms[BUF];
  double carry[4], nxt[4];
  int nt = 0, nc = 0, lvl, i;
  for (lvl = 0; lvl < k; ++lvl) {
    int nn = 0;
    if (lvl < k - 1) {
      for (i = 0; i <= lvl; ++i) {
        double p, e;
        orc_two_prod(x[i], y[lvl - i], &p, &e);
        terms[nt++] = p;
        nxt[nn++] = e;
      }
    } else {
      for (i = 0; i <= lvl; ++i) terms[nt++] = x[i] * y[lvl - i];
    }
    for (i = 0; i < nc; ++i) terms[nt++] = carry[i];
    for (i = 0; i < nn; ++i) carry[i] = nxt[i];
    nc = nn;
  }
  orc_renorm(terms, nt, out, k);
}

static int is_zero_k(const double *x, int k) {
  int i;
  for (i = 0; i < k; ++i)
    if (x[i] != 0.0) return 0;
  return 1;
}

static int is_finite_k(const double *x, int k) {
  int i;
  for (i = 0; i < k; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

/* _div_by_zero _mccore.py:216-219 */
static double div_by_zero(double x0, double y0) {
  if (x0 == 0.0) return NAN;
  return copysign(INFINITY, x0) * copysign(1.0, y0);
}

/* mc_div _mccore.py:222-237 (Newton reciprocal) */
void orc_div(const double *x, const double *y, double *out, int k) {
  int i, it;
  if (k == 1) {
    out[0] = (y[0] == 0.0) ? div_by_zero(x[0], y[0]) : x[0] / y[0];
    return;
  }
  if (y[0] == 0.0 && is_zero_k(y, k)) {
    out[0] = div_by_zero(x[0], y[0]);
    for (i = 1; i < k; ++i) out[i] = 0.0;
    return;
  }
  double one[4] = {1.0, 0.0, 0.0, 0.0};
  double w[4] = {0.0, 0.0, 0.0, 0.0};
  double t1[4], t2[4], t3[4];
  w[0] = 1.0 / y[0];
  int iters = (k == 2) ? 1 : 2;
  for (it = 0; it < iters; ++it) {
    orc_mul(y, w, t1, k);
    orc_sub(one, t1, t2, k);
    orc_mul(w, t2, t3, k);
    orc_add(w, t3, t1, k);
    memcpy(w, t1, sizeof(double) * k);
  }
  double q[4], r[4];
  orc_mul(x, w, q, k);
  orc_mul(q, y, t1, k);
  orc_sub(x, t1, r, k);
  orc_mul(r, w, t2, k);
  orc_add(q, t2, out, k);
}

/* mc_sqrt _mccore.py:245-266 (Newton rsqrt) */
int orc_sqrt(const double *x, double *out, int k) {
  int i, it;
  if (x[0] < 0.0) return -1;
  if (x[0] == 0.0 && is_zero_k(x, k)) {
    for (i = 0; i < k; ++i) out[i] = 0.0;
    return 0;
  }
  if (k == 1) {
    out[0] = sqrt(x[0]);
    return 0;
  }
  double one[4] = {1.0, 0.0, 0.0, 0.0};
  double z[4] = {0.0, 0.0, 0.0, 0.0};
  double t[4], a[4], b[4];
  z[0] = 1.0 / sqrt(x[0]);
  int iters = (k == 2) ? 1 : 2;
  for (it = 0; it < iters; ++it) {
    orc_mul(z, z, a, k);
    orc_mul(x, a, b, k);
    orc_sub(one, b, t, k);
    orc_mul(z, t, a, k);
    for (i = 0; i < k; ++i) a[i] = a[i] * 0.5;
    orc_add(z, a, b, k);
    memcpy(z, b, sizeof(double) * k);
  }
  double r[4];
  orc_mul(x, z, r, k);
  orc_mul(r, r, a, k);
  orc_sub(x, a, t, k);
  for (i = 0; i < k; ++i) b[i] = z[i] * 0.5;
  orc_mul(t, b, a, k);
  orc_add(r, a, out, k);
  return 0;
}

/* mc_cmp _mccore.py:283-290 */
int orc_cmp(const double *x, const double *y, int k) {
  double d[4];
  orc_sub(x, y, d, k);
  if (d[0] > 0.0) return 1;
  if (d[0] < 0.0) return -1;
  return 0;
}

/* cx_mul _mccore.py:322-325 (twin _cmul1 _kernels.py:206-214) */
void orc_cx_mul(const double *ar, const double *ai, const double *br,
                const double *bi, double *outr, double *outi, int k) {
  double t1[4], t2[4], r[4], im[4];
  orc_mul(ar, br, t1, k);
  orc_mul(ai, bi, t2, k);
  orc_sub(t1, t2, r, k);
  orc_mul(ar, bi, t1, k);
  orc_mul(ai, br, t2, k);
  orc_add(t1, t2, im, k);
  memcpy(outr, r, sizeof(double) * k);
  memcpy(outi, im, sizeof(double) * k);
}

/* cx_div _mccore.py:328-347 (Smith) */
void orc_cx_div(const double *ar, const double *ai, const double *br,
                const double *bi, double *outr, double *outi, int k) {
  double t[4], d[4], u[4], v[4], re[4], im[4];
  int i;
  if (fabs(br[0]) >= fabs(bi[0])) {
    if (is_zero_k(br, k) && is_zero_k(bi, k)) {
      outr[0] = div_by_zero(ar[0], 0.0);
      outi[0] = div_by_zero(ai[0], 0.0);
      for (i = 1; i < k; ++i) outr[i] = outi[i] = 0.0;
      return;
    }
    orc_div(bi, br, t, k);
    orc_mul(bi, t, u, k);
    orc_add(br, u, d, k);
    orc_mul(ai, t, u, k);
    orc_add(ar, u, v, k);
    orc_div(v, d, re, k);
    orc_mul(ar, t, u, k);
    orc_sub(ai, u, v, k);
    orc_div(v, d, im, k);
  } else {
    orc_div(br, bi, t, k);
    orc_mul(br, t, u, k);
    orc_add(u, bi, d, k);
    orc_mul(ar, t, u, k);
    orc_add(u, ai, v, k);
    orc_div(v, d, re, k);
    orc_mul(ai, t, u, k);
    orc_sub(u, ar, v, k);
    orc_div(v, d, im, k);
  }
  memcpy(outr, re, sizeof(double) * k);
  memcpy(outi, im, sizeof(double) * k);
}

/* CPython 3.12 complex division (_Py_c_quot), used by the k=1 complex ILU
 * (ilu.py:217, :381 via Python `complex.__truediv__`). */
void orc_py_cdiv(double ar, double ai, double br, double bi, double *qr,
                 double *qi) {
  double abr = br < 0 ? -br : br;
  double abi = bi < 0 ? -bi : bi;
  if (abr >= abi) {
    if (abr == 0.0) {
      *qr = *qi = 0.0; /* Python raises ZeroDivisionError; unreachable */
    } else {
      double ratio = bi / br;
      double denom = br + bi * ratio;
      *qr = (ar + ai * ratio) / denom;
      *qi = (ai - ar * ratio) / denom;
    }
  } else if (abi >= abr) {
    double ratio = br / bi;
    double denom = br * ratio + bi;
    *qr = (ar * ratio + ai) / denom;
    *qi = (ai * ratio - ar) / denom;
  } else {
    *qr = *qi = NAN;
  }
}

/* CPython complex product: (ar*br - ai*bi, ar*bi + ai*br) */
static inline void py_cmul(double ar, double ai, double br, double bi,
                           double *pr, double *pi) {
  *pr = ar * br - ai * bi;
  *pi = ar * bi + ai * br;
}

/* batched element-wise helpers (_kernels.py:558-588 + div/sqrt) */
void orc_ew_add(int64_t n, const double *a, const double *b, double *out,
                int k) {
  int64_t i;
  for (i = 0; i < n; ++i) orc_add(a + i * k, b + i * k, out + i * k, k);
}
void orc_ew_mul(int64_t n, const double *a, const double *b, double *out,
                int k) {
  int64_t i;
  for (i = 0; i < n; ++i) orc_mul(a + i * k, b + i * k, out + i * k, k);
}
void orc_ew_div(int64_t n, const double *a, const double *b, double *out,
                int k) {
  int64_t i;
  for (i = 0; i < n; ++i) orc_div(a + i * k, b + i * k, out + i * k, k);
}
void orc_ew_sqrt(int64_t n, const double *a, double *out, int k) {
  int64_t i;
  for (i = 0; i < n; ++i) orc_sqrt(a + i * k, out + i * k, k);
}
void orc_ew_renorm(int64_t n, int m, const double *a, double *out, int k) {
  int64_t i;
  for (i = 0; i < n; ++i) orc_renorm(a + i * m, m, out + i * k, k);
}

/* ------------------------------------------------------------------ */
/* sparse / vector kernels                                             */
/* ------------------------------------------------------------------ */

/* spmv_real_mixed _kernels.py:243-263, spmv_cx_mixed :326-353 */
typedef struct {
  const int64_t *rp, *ci;
  const double *av_re, *av_im, *x_re, *x_im;
  double *y_re, *y_im;
  int k;
} spmv_args_t;

static void spmv_rows(void *pa, int64_t lo, int64_t hi) {
  spmv_args_t *a = (spmv_args_t *)pa;
  const int64_t *rp = a->rp, *ci = a->ci;
  const double *av_re = a->av_re, *av_im = a->av_im;
  int k = a->k;
  int64_t i;
  for (i = lo; i < hi; ++i) {
    double acc[4] = {0, 0, 0, 0}, acci[4] = {0, 0, 0, 0};
    double aw[4] = {0, 0, 0, 0}, awi[4] = {0, 0, 0, 0};
    double tmp[4], pr[4], pi[4];
    int64_t p;
    int c;
    for (p = rp[i]; p < rp[i + 1]; ++p) {
      int64_t j = ci[p];
      aw[0] = av_re[p];
      if (!av_im) {
        orc_mul(aw, a->x_re + j * k, tmp, k);
        orc_add(acc, tmp, acc, k);
      } else {
        awi[0] = av_im[p];
        orc_cx_mul(aw, awi, a->x_re + j * k, a->x_im + j * k, pr, pi, k);
        orc_add(acc, pr, acc, k);
        orc_add(acci, pi, acci, k);
      }
    }
    for (c = 0; c < k; ++c) {
      a->y_re[i * k + c] = acc[c];
      if (av_im) a->y_im[i * k + c] = acci[c];
    }
  }
}

void orc_spmv_mixed(int64_t n, const int64_t *rp, const int64_t *ci,
                    const double *av_re, const double *av_im, int k,
                    const double *x_re, const double *x_im, double *y_re,
                    double *y_im) {
  spmv_args_t a = {rp, ci, av_re, av_im, x_re, x_im, y_re, y_im, k};
  par_for(n, spmv_rows, &a);
}

/* spmv_adjoint_real_mixed _kernels.py:281-297, _cx_mixed :379-400 */
void orc_spmv_adjoint_mixed(int64_t n, const int64_t *rp, const int64_t *ci,
                            const double *av_re, const double *av_im, int k,
                            const double *x_re, const double *x_im,
                            double *y_re, double *y_im) {
  int64_t i, p;
  double aw[4] = {0, 0, 0, 0}, awi[4] = {0, 0, 0, 0};
  double tmp[4], pr[4], pi[4];
  memset(y_re, 0, sizeof(double) * n * k);
  if (av_im) memset(y_im, 0, sizeof(double) * n * k);
  for (i = 0; i < n; ++i) {
    for (p = rp[i]; p < rp[i + 1]; ++p) {
      int64_t j = ci[p];
      aw[0] = av_re[p];
      if (!av_im) {
        orc_mul(aw, x_re + i * k, tmp, k);
        orc_add(y_re + j * k, tmp, y_re + j * k, k);
      } else {
        awi[0] = -av_im[p];
        orc_cx_mul(aw, awi, x_re + i * k, x_im + i * k, pr, pi, k);
        orc_add(y_re + j * k, pr, y_re + j * k, k);
        orc_add(y_im + j * k, pi, y_im + j * k, k);
      }
    }
  }
}

/* dot_real _kernels.py:487-499, hdot_cx :502-522 (sequential ascending) */
void orc_hdot(int64_t n, int k, const double *x_re, const double *x_im,
              const double *y_re, const double *y_im, double *out_re,
              double *out_im) {
  double acc[4] = {0, 0, 0, 0}, acci[4] = {0, 0, 0, 0};
  double tmp[4], pr[4], pi[4], conj[4];
  int64_t i;
  int c;
  for (i = 0; i < n; ++i) {
    if (!x_im) {
      orc_mul(x_re + i * k, y_re + i * k, tmp, k);
      orc_add(acc, tmp, acc, k);
    } else {
      for (c = 0; c < k; ++c) conj[c] = -x_im[i * k + c];
      orc_cx_mul(x_re + i * k, conj, y_re + i * k, y_im + i * k, pr, pi, k);
      orc_add(acc, pr, acc, k);
      orc_add(acci, pi, acci, k);
    }
  }
  for (c = 0; c < k; ++c) {
    out_re[c] = acc[c];
    if (out_im) out_im[c] = acci[c];
  }
}

/* norm2 sparse.py:532-539 -> sumsq_real/cx _kernels.py:525-552 + mc_sqrt */
void orc_norm2(int64_t n, int k, const double *x_re, const double *x_im,
               double *out) {
  double acc[4] = {0, 0, 0, 0}, tmp[4];
  int64_t i;
  for (i = 0; i < n; ++i) {
    orc_mul(x_re + i * k, x_re + i * k, tmp, k);
    orc_add(acc, tmp, acc, k);
    if (x_im) {
      orc_mul(x_im + i * k, x_im + i * k, tmp, k);
      orc_add(acc, tmp, acc, k);
    }
  }
  if (orc_sqrt(acc, out, k) != 0) {
    int c;
    for (c = 0; c < k; ++c) out[c] = NAN;
  }
}

/* axpy_real _kernels.py:408-418, axpy_cx :421-434: out = y + alpha*x */
typedef struct {
  int k;
  const double *a_re, *a_im, *x_re, *x_im, *y_re, *y_im;
  double *o_re, *o_im;
} axpy_args_t;

static void axpy_rows(void *pa, int64_t lo, int64_t hi) {
  axpy_args_t *a = (axpy_args_t *)pa;
  int k = a->k;
  int64_t i;
  for (i = lo; i < hi; ++i) {
    double tmp[4], pr[4], pi[4], zr[4] = {0, 0, 0, 0};
    if (!a->x_im) {
      orc_mul(a->a_re, a->x_re + i * k, tmp, k);
      orc_add(a->y_re + i * k, tmp, a->o_re + i * k, k);
    } else {
      orc_cx_mul(a->a_re, a->a_im ? a->a_im : zr, a->x_re + i * k,
                 a->x_im + i * k, pr, pi, k);
      orc_add(a->y_re + i * k, pr, a->o_re + i * k, k);
      orc_add(a->y_im + i * k, pi, a->o_im + i * k, k);
    }
  }
}

void orc_axpy(int64_t n, int k, const double *a_re, const double *a_im,
              const double *x_re, const double *x_im, const double *y_re,
              const double *y_im, double *o_re, double *o_im) {
  axpy_args_t a = {k, a_re, a_im, x_re, x_im, y_re, y_im, o_re, o_im};
  par_for(n, axpy_rows, &a);
}

/* ------------------------------------------------------------------ */
/* ILU(0) in binary64: ilu.py:172-276 (factorization), :322-371 sweeps */
/* ------------------------------------------------------------------ */

int orc_ilu0_factor(int64_t n, const int64_t *rp, const int64_t *ci,
                    const int64_t *dp, const double *a_re, const double *a_im,
                    double *lu_re, double *lu_im, int64_t *bad_row,
                    int *structural) {
  int64_t i, nnz = rp[n];
  int cx = a_im != NULL;
  /* _structural_check ilu.py:172-175 */
  for (i = 0; i < n; ++i) {
    if (dp[i] < 0) {
      *bad_row = i;
      *structural = 1;
      return 1;
    }
  }
  memcpy(lu_re, a_re, sizeof(double) * nnz);
  if (cx) memcpy(lu_im, a_im, sizeof(double) * nnz);
  /* row-wise IKJ ilu.py:234-252 */
  for (i = 0; i < n; ++i) {
    int64_t lo = rp[i], hi = rp[i + 1], d = dp[i];
    int64_t t;
    for (t = lo; t < d; ++t) {
      int64_t kc = ci[t];
      int64_t uk = dp[kc];
      double lr, li = 0.0;
      if (!cx) {
        lr = lu_re[t] / lu_re[uk];
      } else {
        orc_py_cdiv(lu_re[t], lu_im[t], lu_re[uk], lu_im[uk], &lr, &li);
      }
      lu_re[t] = lr;
      if (cx) lu_im[t] = li;
      /* eliminate with row kc's upper part (ascending s); merge-find ptr */
      int64_t s, q = lo;
      for (s = uk + 1; s < rp[kc + 1]; ++s) {
        int64_t col = ci[s];
        while (q < hi && ci[q] < col) ++q;
        if (q < hi && ci[q] == col) {
          if (!cx) {
            lu_re[q] = lu_re[q] - lr * lu_re[s];
          } else {
            double pr, pi;
            py_cmul(lr, li, lu_re[s], lu_im[s], &pr, &pi);
            lu_re[q] = lu_re[q] - pr;
            lu_im[q] = lu_im[q] - pi;
          }
        }
      }
    }
    /* is_zero ilu.py:251-252 */
    if (lu_re[d] == 0 && (!cx || lu_im[d] == 0)) {
      *bad_row = i;
      *structural = 0;
      return 1;
    }
  }
  for (i = 0; i < nnz; ++i) {
    if (!isfinite(lu_re[i]) || (cx && !isfinite(lu_im[i]))) return 2;
  }
  return 0;
}

/* ilu0_apply ilu.py:410-420 (k=1): _sweep_forward :322-331 then
 * _sweep_backward :334-343; adjoint ilu.py:423-433 via :346-371. */
int orc_ilu0_apply_f64(int64_t n, const int64_t *rp, const int64_t *ci,
                       const int64_t *dp, const double *lu_re,
                       const double *lu_im, const double *r_re,
                       const double *r_im, double *z_re, double *z_im,
                       int adjoint) {
  int cx = lu_im != NULL;
  int64_t i, p;
  double *yr = (double *)malloc(sizeof(double) * (n ? n : 1));
  double *yi = cx ? (double *)malloc(sizeof(double) * (n ? n : 1)) : NULL;
  if (!adjoint) {
    for (i = 0; i < n; ++i) {
      double ar = r_re[i], ai = cx ? r_im[i] : 0.0;
      for (p = rp[i]; p < dp[i]; ++p) {
        int64_t j = ci[p];
        if (!cx) {
          ar = ar - lu_re[p] * yr[j];
        } else {
          double pr, pi;
          py_cmul(lu_re[p], lu_im[p], yr[j], yi[j], &pr, &pi);
          ar = ar - pr;
          ai = ai - pi;
        }
      }
      yr[i] = ar;
      if (cx) yi[i] = ai;
    }
    for (i = n - 1; i >= 0; --i) {
      double ar = yr[i], ai = cx ? yi[i] : 0.0;
      for (p = dp[i] + 1; p < rp[i + 1]; ++p) {
        int64_t j = ci[p];
        if (!cx) {
          ar = ar - lu_re[p] * z_re[j];
        } else {
          double pr, pi;
          py_cmul(lu_re[p], lu_im[p], z_re[j], z_im[j], &pr, &pi);
          ar = ar - pr;
          ai = ai - pi;
        }
      }
      if (!cx) {
        z_re[i] = ar / lu_re[dp[i]];
      } else {
        orc_py_cdiv(ar, ai, lu_re[dp[i]], lu_im[dp[i]], &z_re[i], &z_im[i]);
      }
    }
  } else {
    /* U^H y = r by ascending row scatter (conj values, conj diagonal) */
    double *acr = z_re, *aci = z_im; /* reuse z as the scatter target */
    memcpy(acr, r_re, sizeof(double) * n);
    if (cx) memcpy(aci, r_im, sizeof(double) * n);
    for (i = 0; i < n; ++i) {
      int64_t d = dp[i];
      if (!cx) {
        yr[i] = acr[i] / lu_re[d];
      } else {
        orc_py_cdiv(acr[i], aci[i], lu_re[d], -lu_im[d], &yr[i], &yi[i]);
      }
      for (p = d + 1; p < rp[i + 1]; ++p) {
        int64_t c = ci[p];
        if (!cx) {
          acr[c] = acr[c] - lu_re[p] * yr[i];
        } else {
          double pr, pi;
          py_cmul(lu_re[p], -lu_im[p], yr[i], yi[i], &pr, &pi);
          acr[c] = acr[c] - pr;
          aci[c] = aci[c] - pi;
        }
      }
    }
    /* L^H z = y by descending row scatter */
    memcpy(acr, yr, sizeof(double) * n);
    if (cx) memcpy(aci, yi, sizeof(double) * n);
    for (i = n - 1; i >= 0; --i) {
      double zr = acr[i], zi = cx ? aci[i] : 0.0;
      for (p = rp[i]; p < dp[i]; ++p) {
        int64_t c = ci[p];
        if (!cx) {
          acr[c] = acr[c] - lu_re[p] * zr;
        } else {
          double pr, pi;
          py_cmul(lu_re[p], -lu_im[p], zr, zi, &pr, &pi);
          acr[c] = acr[c] - pr;
          aci[c] = aci[c] - pi;
        }
      }
    }
  }
  free(yr);
  free(yi);
  /* _finite_or_raise ilu.py:403-407 */
  for (i = 0; i < n; ++i) {
    if (!isfinite(z_re[i]) || (cx && !isfinite(z_im[i]))) return 2;
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* solver context (solvers.py:105-149)                                 */
/* ------------------------------------------------------------------ */

typedef struct {
  double re[4], im[4];
} sc_t;

typedef struct {
  double *re, *im;
} vec_t;

typedef struct {
  int64_t n;
  int k, cx;
  const int64_t *rp, *ci;
  int64_t *dp;
  const double *a_re, *a_im;
  int use_ilu;
  double *lu_re, *lu_im;
  double *w_re, *w_im, *w2_re, *w2_im; /* binary64 scratch */
  double *hist;
  int64_t hist_cap, hist_len;
  int sweep_err;
} ctx_t;

static vec_t vnew(ctx_t *c) {
  vec_t v;
  v.re = (double *)calloc((size_t)(c->n * c->k) + 1, sizeof(double));
  v.im = c->cx ? (double *)calloc((size_t)(c->n * c->k) + 1, sizeof(double))
               : NULL;
  return v;
}
static void vfree(vec_t *v) {
  free(v->re);
  free(v->im);
  v->re = v->im = NULL;
}
static void vcopy(ctx_t *c, vec_t *dst, const vec_t *src) {
  memcpy(dst->re, src->re, sizeof(double) * c->n * c->k);
  if (c->cx) memcpy(dst->im, src->im, sizeof(double) * c->n * c->k);
}

/* scalar ops (multicomponent.py MCFloat / MCComplex operators) */
static sc_t sc_zero(void) {
  sc_t s;
  memset(&s, 0, sizeof(s));
  return s;
}
static sc_t sc_sub(ctx_t *c, sc_t a, sc_t b) {
  sc_t r = sc_zero();
  orc_sub(a.re, b.re, r.re, c->k);
  if (c->cx) orc_sub(a.im, b.im, r.im, c->k);
  return r;
}
static sc_t sc_mul(ctx_t *c, sc_t a, sc_t b) {
  sc_t r = sc_zero();
  if (!c->cx)
    orc_mul(a.re, b.re, r.re, c->k);
  else
    orc_cx_mul(a.re, a.im, b.re, b.im, r.re, r.im, c->k);
  return r;
}
static sc_t sc_div(ctx_t *c, sc_t a, sc_t b) {
  sc_t r = sc_zero();
  if (!c->cx)
    orc_div(a.re, b.re, r.re, c->k);
  else
    orc_cx_div(a.re, a.im, b.re, b.im, r.re, r.im, c->k);
  return r;
}
static sc_t sc_neg(ctx_t *c, sc_t a) {
  int i;
  for (i = 0; i < c->k; ++i) {
    a.re[i] = -a.re[i];
    a.im[i] = -a.im[i];
  }
  return a;
}
static sc_t sc_conj(ctx_t *c, sc_t a) {
  int i;
  if (c->cx)
    for (i = 0; i < c->k; ++i) a.im[i] = -a.im[i];
  return a;
}
static int sc_is_zero(ctx_t *c, sc_t a) {
  return is_zero_k(a.re, c->k) && (!c->cx || is_zero_k(a.im, c->k));
}

/* vector ops (sparse.py:509-600) */
static sc_t v_hdot(ctx_t *c, const vec_t *x, const vec_t *y) {
  sc_t r = sc_zero();
  orc_hdot(c->n, c->k, x->re, x->im, y->re, y->im, r.re, c->cx ? r.im : NULL);
  return r;
}
static sc_t v_norm2(ctx_t *c, const vec_t *x, int record) {
  sc_t r = sc_zero();
  orc_norm2(c->n, c->k, x->re, x->im, r.re);
  if (record && c->hist && c->hist_len < c->hist_cap) {
    memcpy(c->hist + c->hist_len * c->k, r.re, sizeof(double) * c->k);
  }
  if (record) c->hist_len++;
  return r;
}
/* out = y + alpha*x (out may alias y or x elementwise) */
static void v_axpy(ctx_t *c, sc_t a, const vec_t *x, const vec_t *y,
                   vec_t *out) {
  orc_axpy(c->n, c->k, a.re, a.im, x->re, x->im, y->re, y->im, out->re,
           out->im);
}
/* scale _kernels.py:437-464 */
static void v_scale(ctx_t *c, sc_t a, const vec_t *x, vec_t *out) {
  int64_t i;
  int k = c->k;
  for (i = 0; i < c->n; ++i) {
    if (!c->cx) {
      double tmp[4];
      orc_mul(a.re, x->re + i * k, tmp, k);
      memcpy(out->re + i * k, tmp, sizeof(double) * k);
    } else {
      double pr[4], pi[4];
      orc_cx_mul(a.re, a.im, x->re + i * k, x->im + i * k, pr, pi, k);
      memcpy(out->re + i * k, pr, sizeof(double) * k);
      memcpy(out->im + i * k, pi, sizeof(double) * k);
    }
  }
}
static void v_sub(ctx_t *c, const vec_t *x, const vec_t *y, vec_t *out) {
  int64_t i;
  int k = c->k;
  for (i = 0; i < c->n; ++i) {
    double t[4];
    orc_sub(x->re + i * k, y->re + i * k, t, k);
    memcpy(out->re + i * k, t, sizeof(double) * k);
  }
  if (c->cx)
    for (i = 0; i < c->n; ++i) {
      double t[4];
      orc_sub(x->im + i * k, y->im + i * k, t, k);
      memcpy(out->im + i * k, t, sizeof(double) * k);
    }
}
static void v_add(ctx_t *c, const vec_t *x, const vec_t *y, vec_t *out) {
  int64_t i;
  int k = c->k;
  for (i = 0; i < c->n; ++i) {
    double t[4];
    orc_add(x->re + i * k, y->re + i * k, t, k);
    memcpy(out->re + i * k, t, sizeof(double) * k);
  }
  if (c->cx)
    for (i = 0; i < c->n; ++i) {
      double t[4];
      orc_add(x->im + i * k, y->im + i * k, t, k);
      memcpy(out->im + i * k, t, sizeof(double) * k);
    }
}
static void v_matvec(ctx_t *c, const vec_t *x, vec_t *out) {
  orc_spmv_mixed(c->n, c->rp, c->ci, c->a_re, c->a_im, c->k, x->re, x->im,
                 out->re, out->im);
}
static void v_matvec_adj(ctx_t *c, const vec_t *x, vec_t *out) {
  orc_spmv_adjoint_mixed(c->n, c->rp, c->ci, c->a_re, c->a_im, c->k, x->re,
                         x->im, out->re, out->im);
}

/* ilu0_apply_mixed ilu.py:448-458: promote . f64 apply . demote.
 * Complex demotion is numpy's `re + 1j*im` (sparse.py:392), applied to r
 * and again to z before _promote_exact (ilu.py:436-445). */
static void v_precond(ctx_t *c, const vec_t *r, vec_t *out, int adjoint) {
  int64_t i, n = c->n;
  int k = c->k;
  if (!c->use_ilu) {
    if (out != r) vcopy(c, out, r);
    return;
  }
  for (i = 0; i < n; ++i) {
    if (!c->cx) {
      c->w_re[i] = r->re[i * k];
    } else {
      double re0 = r->re[i * k], im0 = r->im[i * k];
      c->w_re[i] = re0 + (0.0 * im0 - 0.0);
      c->w_im[i] = 0.0 + im0;
    }
  }
  int st = orc_ilu0_apply_f64(n, c->rp, c->ci, c->dp, c->lu_re, c->lu_im,
                              c->w_re, c->w_im, c->w2_re, c->w2_im, adjoint);
  if (st != 0) c->sweep_err = 1;
  memset(out->re, 0, sizeof(double) * n * k);
  if (c->cx) memset(out->im, 0, sizeof(double) * n * k);
  for (i = 0; i < n; ++i) {
    if (!c->cx) {
      out->re[i * k] = c->w2_re[i];
    } else {
      double re0 = c->w2_re[i], im0 = c->w2_im[i];
      out->re[i * k] = re0 + (0.0 * im0 - 0.0);
      out->im[i * k] = 0.0 + im0;
    }
  }
}

static int nrm_lt(ctx_t *c, sc_t a, sc_t b) {
  return orc_cmp(a.re, b.re, c->k) < 0;
}

typedef struct {
  int64_t it;
  int conv;
  int bd;
  int have_nrm;
  sc_t nrm, nrm0;
} res_t;

static res_t mkres(int64_t it, int conv, int bd, int have, sc_t nrm,
                   sc_t nrm0) {
  res_t r;
  r.it = it;
  r.conv = conv;
  r.bd = bd;
  r.have_nrm = have;
  r.nrm = nrm;
  r.nrm0 = nrm0;
  return r;
}

/* _Ctx.threshold solvers.py:146-149 */
static sc_t threshold(ctx_t *c, sc_t nrm0, double er, double ea) {
  sc_t e_r = sc_zero(), e_a = sc_zero(), t = sc_zero(), r = sc_zero();
  e_r.re[0] = er;
  e_a.re[0] = ea;
  orc_mul(e_r.re, nrm0.re, t.re, c->k);
  orc_add(t.re, e_a.re, r.re, c->k);
  return r;
}

#define SWEEP_CHECK()                      \
  do {                                     \
    if (c->sweep_err) {                    \
      res = mkres(0, 0, ORC_BD_NUMERIC_SWEEP, 0, nrm, nrm0); \
      goto done;                           \
    }                                      \
  } while (0)

/* bicg solvers.py:183-226 */
static res_t run_bicg(ctx_t *c, const vec_t *b, vec_t *x, double er,
                      double ea, int64_t max_iter) {
  res_t res;
  vec_t r = vnew(c), rt = vnew(c), z = vnew(c), zt = vnew(c), p = vnew(c),
        pt = vnew(c), q = vnew(c), qt = vnew(c), tmp = vnew(c);
  sc_t nrm = sc_zero(), nrm0, thr, rho, sigma, alpha, beta, rho_new;
  int have = 0;
  int64_t it;
  v_matvec(c, x, &tmp);
  v_sub(c, b, &tmp, &r);
  vcopy(c, &rt, &r);
  nrm0 = v_norm2(c, &r, 1);
  thr = threshold(c, nrm0, er, ea);
  if (nrm_lt(c, nrm0, thr)) {
    res = mkres(0, 1, 0, 1, nrm0, nrm0);
    goto done;
  }
  v_precond(c, &r, &z, 0);
  SWEEP_CHECK();
  v_precond(c, &rt, &zt, 1);
  SWEEP_CHECK();
  vcopy(c, &p, &z);
  vcopy(c, &pt, &zt);
  rho = v_hdot(c, &zt, &r);
  for (it = 1; it <= max_iter; ++it) {
    v_matvec(c, &p, &q);
    v_matvec_adj(c, &pt, &qt);
    sigma = v_hdot(c, &pt, &q);
    if (sc_is_zero(c, sigma)) {
      res = mkres(it, 0, ORC_BD_SIGMA_ZERO, have, nrm, nrm0);
      goto done;
    }
    if (sc_is_zero(c, rho)) {
      res = mkres(it, 0, ORC_BD_RHO_ZERO, have, nrm, nrm0);
      goto done;
    }
    alpha = sc_div(c, rho, sigma);
    v_axpy(c, alpha, &p, x, x);
    v_axpy(c, sc_neg(c, alpha), &q, &r, &r);
    v_axpy(c, sc_neg(c, sc_conj(c, alpha)), &qt, &rt, &rt);
    nrm = v_norm2(c, &r, 1);
    have = 1;
    if (!is_finite_k(nrm.re, c->k)) {
      res = mkres(it, 0, ORC_BD_NONFINITE_RESIDUAL, 1, nrm, nrm0);
      goto done;
    }
    if (nrm_lt(c, nrm, thr)) {
      res = mkres(it, 1, 0, 1, nrm, nrm0);
      goto done;
    }
    v_precond(c, &r, &z, 0);
    SWEEP_CHECK();
    v_precond(c, &rt, &zt, 1);
    SWEEP_CHECK();
    rho_new = v_hdot(c, &zt, &r);
    beta = sc_div(c, rho_new, rho);
    v_axpy(c, beta, &p, &z, &p);
    v_axpy(c, sc_conj(c, beta), &pt, &zt, &pt);
    rho = rho_new;
  }
  res = mkres(max_iter, 0, 0, have, nrm, nrm0);
done:
  vfree(&r); vfree(&rt); vfree(&z); vfree(&zt); vfree(&p); vfree(&pt);
  vfree(&q); vfree(&qt); vfree(&tmp);
  return res;
}

/* cgs solvers.py:229-272 */
static res_t run_cgs(ctx_t *c, const vec_t *b, vec_t *x, double er, double ea,
                     int64_t max_iter) {
  res_t res;
  vec_t r = vnew(c), rt0 = vnew(c), u = vnew(c), p = vnew(c), q = vnew(c),
        phat = vnew(c), v = vnew(c), uhat = vnew(c), qhat = vnew(c),
        tmp = vnew(c);
  sc_t nrm = sc_zero(), nrm0, thr, rho, rho_old = sc_zero(), sigma, alpha,
       beta;
  int have = 0;
  int64_t it;
  v_matvec(c, x, &tmp);
  v_sub(c, b, &tmp, &r);
  vcopy(c, &rt0, &r);
  nrm0 = v_norm2(c, &r, 1);
  thr = threshold(c, nrm0, er, ea);
  if (nrm_lt(c, nrm0, thr)) {
    res = mkres(0, 1, 0, 1, nrm0, nrm0);
    goto done;
  }
  for (it = 1; it <= max_iter; ++it) {
    rho = v_hdot(c, &rt0, &r);
    if (sc_is_zero(c, rho)) {
      res = mkres(it, 0, ORC_BD_RHO_ZERO, have, nrm, nrm0);
      goto done;
    }
    if (it == 1) {
      vcopy(c, &u, &r);
      vcopy(c, &p, &u);
    } else {
      beta = sc_div(c, rho, rho_old);
      v_axpy(c, beta, &q, &r, &u);
      v_axpy(c, beta, &p, &q, &tmp);
      v_axpy(c, beta, &tmp, &u, &p);
    }
    v_precond(c, &p, &phat, 0);
    SWEEP_CHECK();
    v_matvec(c, &phat, &v);
    sigma = v_hdot(c, &rt0, &v);
    if (sc_is_zero(c, sigma)) {
      res = mkres(it, 0, ORC_BD_SIGMA_ZERO, have, nrm, nrm0);
      goto done;
    }
    alpha = sc_div(c, rho, sigma);
    v_axpy(c, sc_neg(c, alpha), &v, &u, &q);
    v_add(c, &u, &q, &tmp);
    v_precond(c, &tmp, &uhat, 0);
    SWEEP_CHECK();
    v_axpy(c, alpha, &uhat, x, x);
    v_matvec(c, &uhat, &qhat);
    v_axpy(c, sc_neg(c, alpha), &qhat, &r, &r);
    rho_old = rho;
    nrm = v_norm2(c, &r, 1);
    have = 1;
    if (!is_finite_k(nrm.re, c->k)) {
      res = mkres(it, 0, ORC_BD_NONFINITE_RESIDUAL, 1, nrm, nrm0);
      goto done;
    }
    if (nrm_lt(c, nrm, thr)) {
      res = mkres(it, 1, 0, 1, nrm, nrm0);
      goto done;
    }
  }
  res = mkres(max_iter, 0, 0, have, nrm, nrm0);
done:
  vfree(&r); vfree(&rt0); vfree(&u); vfree(&p); vfree(&q); vfree(&phat);
  vfree(&v); vfree(&uhat); vfree(&qhat); vfree(&tmp);
  return res;
}

/* bicgstab solvers.py:275-328 */
static res_t run_bicgstab(ctx_t *c, const vec_t *b, vec_t *x, double er,
                          double ea, int64_t max_iter) {
  res_t res;
  vec_t r = vnew(c), rt0 = vnew(c), p = vnew(c), v = vnew(c), phat = vnew(c),
        s = vnew(c), shat = vnew(c), t = vnew(c), tmp = vnew(c);
  sc_t nrm = sc_zero(), nrm0, thr, rho, rho_old = sc_zero(),
       alpha = sc_zero(), omega = sc_zero(), sigma, beta, tt, ts;
  int have = 0;
  int64_t it;
  v_matvec(c, x, &tmp);
  v_sub(c, b, &tmp, &r);
  vcopy(c, &rt0, &r);
  nrm0 = v_norm2(c, &r, 1);
  thr = threshold(c, nrm0, er, ea);
  if (nrm_lt(c, nrm0, thr)) {
    res = mkres(0, 1, 0, 1, nrm0, nrm0);
    goto done;
  }
  for (it = 1; it <= max_iter; ++it) {
    rho = v_hdot(c, &rt0, &r);
    if (sc_is_zero(c, rho)) {
      res = mkres(it, 0, ORC_BD_RHO_ZERO, have, nrm, nrm0);
      goto done;
    }
    if (it == 1) {
      vcopy(c, &p, &r);
    } else {
      if (sc_is_zero(c, omega)) {
        res = mkres(it, 0, ORC_BD_OMEGA_ZERO, have, nrm, nrm0);
        goto done;
      }
      beta = sc_mul(c, sc_div(c, rho, rho_old), sc_div(c, alpha, omega));
      v_axpy(c, sc_neg(c, omega), &v, &p, &tmp);
      v_axpy(c, beta, &tmp, &r, &p);
    }
    v_precond(c, &p, &phat, 0);
    SWEEP_CHECK();
    v_matvec(c, &phat, &v);
    sigma = v_hdot(c, &rt0, &v);
    if (sc_is_zero(c, sigma)) {
      res = mkres(it, 0, ORC_BD_SIGMA_ZERO, have, nrm, nrm0);
      goto done;
    }
    alpha = sc_div(c, rho, sigma);
    v_axpy(c, sc_neg(c, alpha), &v, &r, &s);
    nrm = v_norm2(c, &s, 1);
    have = 1;
    if (!is_finite_k(nrm.re, c->k)) {
      res = mkres(it, 0, ORC_BD_NONFINITE_RESIDUAL, 1, nrm, nrm0);
      goto done;
    }
    if (nrm_lt(c, nrm, thr)) {
      v_axpy(c, alpha, &phat, x, x);
      res = mkres(it, 1, 0, 1, nrm, nrm0);
      goto done;
    }
    v_precond(c, &s, &shat, 0);
    SWEEP_CHECK();
    v_matvec(c, &shat, &t);
    tt = v_hdot(c, &t, &t);
    if (sc_is_zero(c, tt)) {
      res = mkres(it, 0, ORC_BD_OMEGA_ZERO, 1, nrm, nrm0);
      goto done;
    }
    ts = v_hdot(c, &t, &s);
    omega = sc_div(c, ts, tt);
    v_axpy(c, alpha, &phat, x, &tmp);
    v_axpy(c, omega, &shat, &tmp, x);
    v_axpy(c, sc_neg(c, omega), &t, &s, &r);
    rho_old = rho;
    nrm = v_norm2(c, &r, 1);
    if (!is_finite_k(nrm.re, c->k)) {
      res = mkres(it, 0, ORC_BD_NONFINITE_RESIDUAL, 1, nrm, nrm0);
      goto done;
    }
    if (nrm_lt(c, nrm, thr)) {
      res = mkres(it, 1, 0, 1, nrm, nrm0);
      goto done;
    }
  }
  res = mkres(max_iter, 0, 0, have, nrm, nrm0);
done:
  vfree(&r); vfree(&rt0); vfree(&p); vfree(&v); vfree(&phat); vfree(&s);
  vfree(&shat); vfree(&t); vfree(&tmp);
  return res;
}

/* gpbicg solvers.py:331-412 (x = M^-1 yhat at exit, :357-359) */
static res_t run_gpbicg(ctx_t *c, const vec_t *b, vec_t *x, double er,
                        double ea, int64_t max_iter) {
  res_t res;
  vec_t yhat = vnew(c), r = vnew(c), rt0 = vnew(c), t_prev = vnew(c),
        w = vnew(c), u = vnew(c), z = vnew(c), p = vnew(c), Bp = vnew(c),
        y = vnew(c), t = vnew(c), Bt = vnew(c), tmp = vnew(c),
        tmp2 = vnew(c), zero = vnew(c);
  sc_t nrm = sc_zero(), nrm0, thr, rho, beta = sc_zero(), sigma, alpha,
       btbt, btt, zeta, eta, yy, ybt, bty, yt, delta, rho_new;
  int have = 0;
  int64_t it;
  v_matvec(c, &zero, &tmp);
  v_sub(c, b, &tmp, &r);
  vcopy(c, &rt0, &r);
  nrm0 = v_norm2(c, &r, 1);
  thr = threshold(c, nrm0, er, ea);
  if (nrm_lt(c, nrm0, thr)) {
    /* report x = yhat (zeros), not M^-1 applied (solvers.py:346-347) */
    vcopy(c, x, &yhat);
    res = mkres(0, 1, 0, 1, nrm0, nrm0);
    goto done_nofinish;
  }
  rho = v_hdot(c, &rt0, &r);
  for (it = 1; it <= max_iter; ++it) {
    if (it == 1) {
      vcopy(c, &p, &r);
    } else {
      v_sub(c, &p, &u, &tmp);
      v_axpy(c, beta, &tmp, &r, &p);
    }
    v_precond(c, &p, &tmp, 0);
    SWEEP_CHECK();
    v_matvec(c, &tmp, &Bp);
    sigma = v_hdot(c, &rt0, &Bp);
    if (sc_is_zero(c, sigma)) {
      res = mkres(it, 0, ORC_BD_SIGMA_ZERO, have, nrm, nrm0);
      goto finish;
    }
    if (sc_is_zero(c, rho)) {
      res = mkres(it, 0, ORC_BD_RHO_ZERO, have, nrm, nrm0);
      goto finish;
    }
    alpha = sc_div(c, rho, sigma);
    v_sub(c, &Bp, &w, &tmp);
    v_sub(c, &t_prev, &r, &tmp2);
    v_axpy(c, alpha, &tmp, &tmp2, &y);
    v_axpy(c, sc_neg(c, alpha), &Bp, &r, &t);
    v_precond(c, &t, &tmp, 0);
    SWEEP_CHECK();
    v_matvec(c, &tmp, &Bt);
    btbt = v_hdot(c, &Bt, &Bt);
    btt = v_hdot(c, &Bt, &t);
    if (it == 1) {
      if (sc_is_zero(c, btbt)) {
        res = mkres(it, 0, ORC_BD_BREAKDOWN_LS, have, nrm, nrm0);
        goto finish;
      }
      zeta = sc_div(c, btt, btbt);
      eta = sc_zero();
    } else {
      yy = v_hdot(c, &y, &y);
      ybt = v_hdot(c, &y, &Bt);
      bty = v_hdot(c, &Bt, &y);
      yt = v_hdot(c, &y, &t);
      delta = sc_sub(c, sc_mul(c, yy, btbt), sc_mul(c, ybt, bty));
      if (sc_is_zero(c, delta)) {
        res = mkres(it, 0, ORC_BD_BREAKDOWN_LS, have, nrm, nrm0);
        goto finish;
      }
      eta = sc_div(c, sc_sub(c, sc_mul(c, btbt, yt), sc_mul(c, ybt, btt)),
                   delta);
      zeta = sc_div(c, sc_sub(c, sc_mul(c, yy, btt), sc_mul(c, bty, yt)),
                    delta);
    }
    if (it > 1) {
      /* u = axpy(zeta, Bp, scale(eta, axpy(beta, u, t_prev - r))) */
      v_sub(c, &t_prev, &r, &tmp);
      v_axpy(c, beta, &u, &tmp, &tmp2);
      v_scale(c, eta, &tmp2, &tmp);
      v_axpy(c, zeta, &Bp, &tmp, &u);
    } else {
      v_scale(c, zeta, &Bp, &u);
    }
    /* z = axpy(-alpha, u, axpy(zeta, r, scale(eta, z))) */
    v_scale(c, eta, &z, &tmp);
    v_axpy(c, zeta, &r, &tmp, &tmp2);
    v_axpy(c, sc_neg(c, alpha), &u, &tmp2, &z);
    /* yhat = yhat + axpy(alpha, p, z) */
    v_axpy(c, alpha, &p, &z, &tmp);
    v_add(c, &yhat, &tmp, &yhat);
    /* r = axpy(-eta, y, axpy(-zeta, Bt, t)) */
    v_axpy(c, sc_neg(c, zeta), &Bt, &t, &tmp);
    v_axpy(c, sc_neg(c, eta), &y, &tmp, &r);
    nrm = v_norm2(c, &r, 1);
    have = 1;
    if (!is_finite_k(nrm.re, c->k)) {
      res = mkres(it, 0, ORC_BD_NONFINITE_RESIDUAL, 1, nrm, nrm0);
      goto finish;
    }
    if (nrm_lt(c, nrm, thr)) {
      res = mkres(it, 1, 0, 1, nrm, nrm0);
      goto finish;
    }
    rho_new = v_hdot(c, &rt0, &r);
    if (sc_is_zero(c, zeta)) {
      res = mkres(it, 0, ORC_BD_ZETA_ZERO, 1, nrm, nrm0);
      goto finish;
    }
    if (sc_is_zero(c, rho)) {
      res = mkres(it, 0, ORC_BD_RHO_ZERO, 1, nrm, nrm0);
      goto finish;
    }
    beta = sc_mul(c, sc_div(c, alpha, zeta), sc_div(c, rho_new, rho));
    v_axpy(c, beta, &Bp, &Bt, &w);
    rho = rho_new;
    vcopy(c, &t_prev, &t);
  }
  res = mkres(max_iter, 0, 0, have, nrm, nrm0);
finish:
  v_precond(c, &yhat, x, 0);
  if (c->sweep_err) res = mkres(0, 0, ORC_BD_NUMERIC_SWEEP, 0, nrm, nrm0);
  goto done_nofinish;
done:
done_nofinish:
  vfree(&yhat); vfree(&r); vfree(&rt0); vfree(&t_prev); vfree(&w);
  vfree(&u); vfree(&z); vfree(&p); vfree(&Bp); vfree(&y); vfree(&t);
  vfree(&Bt); vfree(&tmp); vfree(&tmp2); vfree(&zero);
  return res;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* solve solvers.py:418-453 */
int orc_solve(int64_t n, const int64_t *rp, const int64_t *ci,
              const double *a_re, const double *a_im, int method, int k,
              double eps_rel, double eps_abs, int64_t max_iter,
              int precond_ilu, const double *b_re, const double *b_im,
              double *x_re, double *x_im, double *hist, int64_t hist_cap,
              orc_report_t *rep) {
  ctx_t c;
  int64_t i, nnz = rp[n];
  memset(&c, 0, sizeof(c));
  memset(rep, 0, sizeof(*rep));
  rep->final_recursive_relres = NAN;
  rep->true_relres = NAN;
  c.n = n;
  c.k = k;
  c.cx = a_im != NULL;
  c.rp = rp;
  c.ci = ci;
  c.a_re = a_re;
  c.a_im = a_im;
  c.hist = hist;
  c.hist_cap = hist_cap;
  c.use_ilu = precond_ilu;
  /* CsrMatrix._find_diagonals sparse.py:235-243 */
  c.dp = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
  for (i = 0; i < n; ++i) {
    int64_t p;
    c.dp[i] = -1;
    for (p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i) c.dp[i] = p;
  }
  double t0 = now_s();
  if (precond_ilu) {
    c.lu_re = (double *)malloc(sizeof(double) * (nnz + 1));
    c.lu_im = c.cx ? (double *)malloc(sizeof(double) * (nnz + 1)) : NULL;
    int st = orc_ilu0_factor(n, rp, ci, c.dp, a_re, a_im, c.lu_re, c.lu_im,
                             &rep->bad_row, &rep->structural);
    if (st != 0) {
      rep->breakdown = (st == 1) ? ORC_BD_SINGULAR_PIVOT : ORC_BD_NUMERIC_FACTOR;
      rep->factor_seconds = now_s() - t0;
      free(c.dp);
      free(c.lu_re);
      free(c.lu_im);
      return 0;
    }
    c.w_re = (double *)malloc(sizeof(double) * (n + 1));
    c.w2_re = (double *)malloc(sizeof(double) * (n + 1));
    if (c.cx) {
      c.w_im = (double *)malloc(sizeof(double) * (n + 1));
      c.w2_im = (double *)malloc(sizeof(double) * (n + 1));
    }
  }
  double t1 = now_s();
  rep->factor_seconds = t1 - t0;
  vec_t b, x;
  b.re = (double *)b_re;
  b.im = (double *)b_im;
  x.re = x_re;
  x.im = x_im;
  memset(x_re, 0, sizeof(double) * n * k);
  if (c.cx) memset(x_im, 0, sizeof(double) * n * k);
  res_t res;
  switch (method) {
    case ORC_BICG: res = run_bicg(&c, &b, &x, eps_rel, eps_abs, max_iter); break;
    case ORC_CGS: res = run_cgs(&c, &b, &x, eps_rel, eps_abs, max_iter); break;
    case ORC_BICGSTAB:
      res = run_bicgstab(&c, &b, &x, eps_rel, eps_abs, max_iter);
      break;
    default: res = run_gpbicg(&c, &b, &x, eps_rel, eps_abs, max_iter); break;
  }
  rep->loop_seconds = now_s() - t1;
  rep->hist_len = c.hist_len;
  if (res.bd == ORC_BD_NUMERIC_SWEEP) {
    rep->iterations = 0;
    rep->converged = 0;
    rep->breakdown = ORC_BD_NUMERIC_SWEEP;
    rep->has_x = 0;
  } else {
    rep->iterations = res.it;
    rep->converged = res.conv;
    rep->breakdown = res.bd;
    rep->has_x = 1;
    /* _report solvers.py:165-180 */
    if (res.have_nrm && !is_zero_k(res.nrm0.re, k)) {
      double q[4];
      orc_div(res.nrm.re, res.nrm0.re, q, k);
      rep->final_recursive_relres = q[0];
    }
    /* true residual solvers.py:446-450 (spmv on promoted A == mixed) */
    vec_t ax = vnew(&c), resid = vnew(&c);
    v_matvec(&c, &x, &ax);
    v_sub(&c, &b, &ax, &resid);
    sc_t nb = v_norm2(&c, &b, 0);
    if (!is_zero_k(nb.re, k)) {
      sc_t nr = v_norm2(&c, &resid, 0);
      double q[4];
      orc_div(nr.re, nb.re, q, k);
      rep->true_relres = q[0];
    }
    vfree(&ax);
    vfree(&resid);
  }
  free(c.dp);
  free(c.lu_re);
  free(c.lu_im);
  free(c.w_re);
  free(c.w_im);
  free(c.w2_re);
  free(c.w2_im);
  return 0;
}

typedef struct {
  int nsys;
  const int64_t *n;
  const int64_t *const *rp;
  const int64_t *const *ci;
  const double *const *a_re;
  int method, k;
  double eps_rel, eps_abs;
  int64_t max_iter;
  const double *const *b_re;
  double *const *x_re;
  orc_report_t *reps;
  int next;
  pthread_mutex_t mu;
} batch_t;

static void *batch_worker(void *p) {
  batch_t *b = (batch_t *)p;
  tl_serial = 1;
  for (;;) {
    pthread_mutex_lock(&b->mu);
    int s = b->next++;
    pthread_mutex_unlock(&b->mu);
    if (s >= b->nsys) break;
    orc_solve(b->n[s], b->rp[s], b->ci[s], b->a_re[s], NULL, b->method, b->k,
              b->eps_rel, b->eps_abs, b->max_iter, 1, b->b_re[s], NULL,
              b->x_re[s], NULL, NULL, 0, &b->reps[s]);
  }
  return NULL;
}

int orc_solve_batch(int nsys, const int64_t *n, const int64_t *const *rp,
                    const int64_t *const *ci, const double *const *a_re,
                    int method, int k, double eps_rel, double eps_abs,
                    int64_t max_iter, const double *const *b_re,
                    double *const *x_re, orc_report_t *reps, int nthreads) {
  batch_t b = {nsys, n, rp, ci, a_re, method, k, eps_rel, eps_abs, max_iter,
               b_re, x_re, reps, 0, PTHREAD_MUTEX_INITIALIZER};
  int t = nthreads < 1 ? 1 : (nthreads > 256 ? 256 : nthreads), i;
  pthread_t th[256];
  for (i = 1; i < t; ++i) pthread_create(&th[i], NULL, batch_worker, &b);
  batch_worker(&b);
  tl_serial = 0;
  for (i = 1; i < t; ++i) pthread_join(th[i], NULL);
  return 0;
}
