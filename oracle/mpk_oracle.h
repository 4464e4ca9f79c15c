/*
 * mpk_oracle.h -- CPU restatement of the reference mpkrylov hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 kernels and the timed CPU baseline in bench.py --impl reference.
 * The product path (paper_2504_14498_b200/) never links or calls it.
 *
 * Every function restates the reference Python/numba code operation for
 * operation (same evaluation order, no FMA contraction: build with
 * -ffp-contract=off), citing /root/reference/pkg/src/mpkrylov/<file>:<line>.
 * Pinned against reference-generated golden vectors in tests/golden/.
 *
 * Layouts follow the reference: an MC vector is a C-contiguous (n, k)
 * float64 array (most significant component first), complex vectors are a
 * pair of such arrays (re, im).  CSR indices are int64 as in sparse.py.
 */
#ifndef MPK_ORACLE_H
#define MPK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- MC core (_mccore.py / _kernels.py twins) ---- */
void orc_two_sum(double a, double b, double *s, double *e);
void orc_two_prod(double a, double b, double *p, double *e);
void orc_renorm(const double *terms, int m, double *out, int k);
void orc_add(const double *x, const double *y, double *out, int k);
void orc_sub(const double *x, const double *y, double *out, int k);
void orc_mul(const double *x, const double *y, double *out, int k);
void orc_div(const double *x, const double *y, double *out, int k);
int orc_sqrt(const double *x, double *out, int k); /* -1 on negative */
int orc_cmp(const double *x, const double *y, int k);
void orc_cx_mul(const double *ar, const double *ai, const double *br,
                const double *bi, double *outr, double *outi, int k);
void orc_cx_div(const double *ar, const double *ai, const double *br,
                const double *bi, double *outr, double *outi, int k);
/* CPython complex ops (k = 1 complex ILU arithmetic). */
void orc_py_cdiv(double ar, double ai, double br, double bi, double *qr,
                 double *qi);

/* batched element-wise ops on (n,k) arrays (tests) */
void orc_ew_add(int64_t n, const double *a, const double *b, double *out, int k);
void orc_ew_mul(int64_t n, const double *a, const double *b, double *out, int k);
void orc_ew_div(int64_t n, const double *a, const double *b, double *out, int k);
void orc_ew_sqrt(int64_t n, const double *a, double *out, int k);
void orc_ew_renorm(int64_t n, int m, const double *a, double *out, int k);

/* ---- sparse kernels (sparse.py / _kernels.py) ---- */
void orc_spmv_mixed(int64_t n, const int64_t *rp, const int64_t *ci,
                    const double *av_re, const double *av_im, int k,
                    const double *x_re, const double *x_im, double *y_re,
                    double *y_im);
void orc_spmv_adjoint_mixed(int64_t n, const int64_t *rp, const int64_t *ci,
                            const double *av_re, const double *av_im, int k,
                            const double *x_re, const double *x_im,
                            double *y_re, double *y_im);
void orc_hdot(int64_t n, int k, const double *x_re, const double *x_im,
              const double *y_re, const double *y_im, double *out_re,
              double *out_im);
void orc_norm2(int64_t n, int k, const double *x_re, const double *x_im,
               double *out);
void orc_axpy(int64_t n, int k, const double *a_re, const double *a_im,
              const double *x_re, const double *x_im, const double *y_re,
              const double *y_im, double *o_re, double *o_im);

/* ---- ILU(0) in binary64 (ilu.py) ----
 * status: 0 ok, 1 singular pivot (bad_row, structural), 2 numeric breakdown */
int orc_ilu0_factor(int64_t n, const int64_t *rp, const int64_t *ci,
                    const int64_t *dp, const double *a_re, const double *a_im,
                    double *lu_re, double *lu_im, int64_t *bad_row,
                    int *structural);
/* z = U^-1 L^-1 r on binary64 vectors (complex: split re/im arrays) */
int orc_ilu0_apply_f64(int64_t n, const int64_t *rp, const int64_t *ci,
                       const int64_t *dp, const double *lu_re,
                       const double *lu_im, const double *r_re,
                       const double *r_im, double *z_re, double *z_im,
                       int adjoint);

/* ---- solvers (solvers.py) ---- */
enum {
  ORC_BD_NONE = 0,
  ORC_BD_SIGMA_ZERO = 1,
  ORC_BD_RHO_ZERO = 2,
  ORC_BD_OMEGA_ZERO = 3,
  ORC_BD_NONFINITE_RESIDUAL = 4,
  ORC_BD_BREAKDOWN_LS = 5,
  ORC_BD_ZETA_ZERO = 6,
  ORC_BD_SINGULAR_PIVOT = 7,
  ORC_BD_NUMERIC_FACTOR = 8,
  ORC_BD_NUMERIC_SWEEP = 9
};
enum { ORC_BICG = 0, ORC_CGS = 1, ORC_BICGSTAB = 2, ORC_GPBICG = 3 };

typedef struct {
  int64_t iterations;
  int32_t converged;
  int32_t breakdown;
  int64_t bad_row;
  int32_t structural;
  int32_t has_x;
  double final_recursive_relres;
  double true_relres;
  int64_t hist_len;
  double factor_seconds;
  double loop_seconds;
} orc_report_t;

/* solve(): build binary64 ILU(0), run the method with mixed SpMV, compute
 * the true residual.  hist receives the norm2 sequence (k doubles each). */
int orc_solve(int64_t n, const int64_t *rp, const int64_t *ci,
              const double *a_re, const double *a_im, int method, int k,
              double eps_rel, double eps_abs, int64_t max_iter,
              int precond_ilu, const double *b_re, const double *b_im,
              double *x_re, double *x_im, double *hist, int64_t hist_cap,
              orc_report_t *rep);

void orc_set_threads(int t);

/* independent systems solved on nthreads host threads (cfg5 CPU arm) */
int orc_solve_batch(int nsys, const int64_t *n, const int64_t *const *rp,
                    const int64_t *const *ci, const double *const *a_re,
                    int method, int k, double eps_rel, double eps_abs,
                    int64_t max_iter, const double *const *b_re,
                    double *const *x_re, orc_report_t *reps, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
