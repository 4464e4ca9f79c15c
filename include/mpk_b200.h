/*
 * mpk_b200.h -- C ABI of the B200 (sm_100a) mpkrylov hot path.
 *
 * Drop-in boundary for the reference package mpkrylov
 * (/root/reference/pkg/src/mpkrylov).  The reference is pure Python+numba
 * with no FFI of its own; each entry point below replaces one Python
 * function on the hot path (cited per function), takes plain pointers and
 * sizes, and uses the reference's array layouts: CSR row_ptr/col_idx int64
 * (sparse.py:192-233), values float64; MC vectors C-contiguous (n, k)
 * float64 with the most significant component first, complex vectors as a
 * (re, im) pair of such arrays (sparse.py:341-404, _kernels.py:8-10).
 * All pointers are HOST pointers unless the name says _dev.
 *
 * Status codes: 0 ok, 1 singular pivot, 2 numeric breakdown, 3 invalid
 * argument, 4 CUDA error.  mpk_last_error() returns a thread-local message.
 * The Python binding (paper_2504_14498_b200/_lib.py) maps them to the
 * reference exceptions (ValueError, SingularPivotError,
 * NumericBreakdownError) and breakdown strings (solvers.py:207-407).
 */
#ifndef MPK_B200_H
#define MPK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPK_OK 0
#define MPK_SINGULAR_PIVOT 1
#define MPK_NUMERIC_BREAKDOWN 2
#define MPK_INVALID 3
#define MPK_CUDA_ERROR 4

/* methods: solvers.py:57 METHODS order is bicg, cgs, bicgstab, gpbicg */
#define MPK_BICG 0
#define MPK_CGS 1
#define MPK_BICGSTAB 2
#define MPK_GPBICG 3

/* breakdown codes (solvers.py string in comment) */
#define MPK_BD_NONE 0              /* None */
#define MPK_BD_SIGMA_ZERO 1        /* "sigma_zero" */
#define MPK_BD_RHO_ZERO 2          /* "rho_zero" */
#define MPK_BD_OMEGA_ZERO 3        /* "omega_zero" */
#define MPK_BD_NONFINITE 4         /* "nonfinite_residual" */
#define MPK_BD_BREAKDOWN_LS 5      /* "breakdown_ls" */
#define MPK_BD_ZETA_ZERO 6         /* "zeta_zero" */
#define MPK_BD_SINGULAR_PIVOT 7    /* SingularPivotError (ilu.py:60-66) */
#define MPK_BD_NUMERIC_FACTOR 8    /* NumericBreakdownError, factors */
#define MPK_BD_NUMERIC_SWEEP 9     /* NumericBreakdownError, sweep */

typedef struct mpk_ctx mpk_ctx;
typedef struct mpk_matrix mpk_matrix;

typedef struct {
  int64_t iterations;
  int32_t converged;
  int32_t breakdown;      /* MPK_BD_* */
  int64_t bad_row;        /* SingularPivotError.k */
  int32_t structural;     /* SingularPivotError(structural=True) */
  int32_t has_x;
  double final_recursive_relres; /* SolveReport, solvers.py:88-102 */
  double true_relres;
  int64_t hist_len;       /* number of norm2 calls in the method */
  double factor_ms;       /* device time of the ILU(0) factorization */
  double solve_ms;        /* device time of the Krylov loop */
  double total_ms;        /* host wall time of the whole call */
  int64_t launches;       /* kernels executed by the call */
} mpk_report;

const char *mpk_last_error(void);
int mpk_version(void);

/* One CUDA device + stream.  Reentrant per context. */
int mpk_ctx_create(int device, mpk_ctx **out);
void mpk_ctx_destroy(mpk_ctx *ctx);
int mpk_ctx_synchronize(mpk_ctx *ctx);
/* the context's cudaStream_t (for event timing by the caller) */
void *mpk_ctx_stream(mpk_ctx *ctx);
/* Context options.  MPK_OPT_REDUCTION selects how dot products / norms are
 * reduced in mpk_hdot, mpk_norm2 and the solvers: MPK_REDUCE_TREE (default,
 * fixed-shape parallel tree) or MPK_REDUCE_SEQUENTIAL (the reference's
 * ascending accumulation, _kernels.py:487-552, bit-identical to it and
 * slow: one dependent chain of n MC additions per reduction). */
#define MPK_OPT_REDUCTION 1
#define MPK_REDUCE_TREE 0
#define MPK_REDUCE_SEQUENTIAL 1
/* MPK_OPT_PRECOND: the preconditioner of the solvers (SolverConfig.precond,
 * solvers.py:64-85, _Ctx.apply solvers.py:128-136): MPK_PRECOND_ILU0_MIXED
 * (default; binary64 ILU(0) applied to the demoted vector) or
 * MPK_PRECOND_NONE (M = I: no factorization, the methods run on the MC
 * vectors themselves, SpMV on MC inputs) */
#define MPK_OPT_PRECOND 2
#define MPK_PRECOND_NONE 0
#define MPK_PRECOND_ILU0_MIXED 1
/* MPK_PRECOND_ILU0_FULL: ILU(0) at the working precision (ilu.py:279-281;
 * factors and sweeps in k-component arithmetic with the _mcfast fused
 * a - b*c and diagonal solvers, _mcfast.py:80-439); all four methods,
 * real and complex */
#define MPK_PRECOND_ILU0_FULL 2
int mpk_ctx_set_option(mpk_ctx *ctx, int option, int64_t value);
/* Per-call form of MPK_OPT_PRECOND (SolverConfig.precond is an argument of
 * every solve() in the reference, solvers.py:418-425): the calling thread's
 * next solves use `value` instead of the context's setting; value < 0
 * clears the override.  Thread-local, so concurrent solves on one context
 * never see each other's preconditioner. */
int mpk_thread_set_option(int option, int64_t value);
/* MPK_OPT_SPMV (per-thread only): SolverConfig.spmv_mode (solvers.py:64-85,
 * _Ctx.matvec :126-134).  MPK_SPMV_FULL makes the solvers multiply with the
 * matrix's working-precision values when mpk_csr_set_mc_values attached
 * them; for binary64-valued matrices both modes are the same computation. */
#define MPK_OPT_SPMV 3
#define MPK_SPMV_MIXED 0
#define MPK_SPMV_FULL 1

/* CsrMatrix.demoted() upload (sparse.py:192-249): binary64 values, val_im
 * NULL for the real field.  Columns must be strictly increasing per row. */
int mpk_csr_upload(mpk_ctx *ctx, int64_t n, int64_t nnz,
                   const int64_t *row_ptr, const int64_t *col_idx,
                   const double *val_re, const double *val_im,
                   mpk_matrix **out);
void mpk_csr_free(mpk_matrix *m);
/* New binary64 values on the uploaded pattern (numeric phase; the pattern
 * analysis -- level sets, sweep matrices, solver plans -- is kept). */
int mpk_csr_set_values(mpk_matrix *m, const double *val_re,
                       const double *val_im);
/* CsrMatrix values at working precision (sparse.py:192-249: val_re / val_im
 * of shape (nnz, k), row-major).  Attaches all k components of every entry
 * for spmv_mode "full" (mpk_spmv_full, MPK_OPT_SPMV) and for the
 * working-precision ILU(0) of an MC-valued matrix (ilu.py:279-281); k = 0
 * detaches them.  The binary64 values of mpk_csr_upload stay the demoted
 * matrix (CsrMatrix.demoted, sparse.py:251-258) that ILU(0)-mixed factors. */
int mpk_csr_set_mc_values(mpk_matrix *m, int k, const double *val_re,
                          const double *val_im);

/* ilu0_factorize_demoted (ilu.py:284-286 -> _factorize_tuples :178-276).
 * Returns MPK_SINGULAR_PIVOT with *bad_row / *structural, or
 * MPK_NUMERIC_BREAKDOWN for non-finite factors. */
int mpk_ilu0_factor(mpk_matrix *m, int64_t *bad_row, int32_t *structural);
/* ilu0_factorize (ilu.py:279-281) of the uploaded binary64 matrix promoted
 * to k = 2..4 components; factors downloadable as (nnz,k) (complex:
 * (nnz,2k) rows re[k] | im[k]) and applicable to (n,k) vectors (complex:
 * the (n,k) re block followed by the (n,k) im block) */
int mpk_ilu0_factor_full(mpk_matrix *m, int k, int64_t *bad_row, int32_t *structural);
int mpk_ilu0_download_full(mpk_matrix *m, int k, double *lu);
int mpk_ilu0_apply_full(mpk_matrix *m, int k, const double *r, double *z);
/* adjoint != 0: ilu0_apply_adjoint (ilu.py:423-433) */
int mpk_ilu0_apply_full_ex(mpk_matrix *m, int k, const double *r, double *z, int adjoint);
/* IluFactors.val_re / val_im as (nnz,) arrays (bitwise parity tests) */
int mpk_ilu0_download(mpk_matrix *m, double *lu_re, double *lu_im);
/* ilu0_apply on binary64 vectors (ilu.py:410-433): z = U^-1 L^-1 r, or the
 * adjoint (LU)^-H r.  Complex: separate re/im arrays of length n. */
int mpk_ilu0_apply_f64(mpk_matrix *m, const double *r_re, const double *r_im,
                       double *z_re, double *z_im, int adjoint);
/* ilu0_apply_mixed / _adjoint_mixed (ilu.py:448-470) on (n,k) MC vectors */
int mpk_ilu0_apply_mixed(mpk_matrix *m, int k, const double *r_re,
                         const double *r_im, double *z_re, double *z_im,
                         int adjoint);

/* spmv_mixed / spmv_adjoint_mixed (sparse.py:465-496) on (n,k) vectors */
int mpk_spmv_mixed(mpk_matrix *m, int k, const double *x_re,
                   const double *x_im, double *y_re, double *y_im,
                   int adjoint);

/* spmv / spmv_adjoint (sparse.py:414-451 -> _kernels.py:224-240, 266-278,
 * 300-323, 356-376): the matrix at working precision (MC x MC products).
 * Without attached MC values the matrix is binary64-valued and the mixed
 * kernels compute the same result bit for bit. */
int mpk_spmv_full(mpk_matrix *m, int k, const double *x_re, const double *x_im,
                  double *y_re, double *y_im, int adjoint);

/* hdot (sparse.py:509-517): out_re/out_im k doubles.  norm2 (:532-539).
 * Device reduction order is a fixed tree. */
int mpk_hdot(mpk_ctx *ctx, int64_t n, int k, const double *x_re,
             const double *x_im, const double *y_re, const double *y_im,
             double *out_re, double *out_im);
int mpk_norm2(mpk_ctx *ctx, int64_t n, int k, const double *x_re,
              const double *x_im, double *out);
/* axpy (sparse.py:542-560): out = y + alpha*x; alpha_im NULL for real */
int mpk_axpy(mpk_ctx *ctx, int64_t n, int k, const double *alpha_re,
             const double *alpha_im, const double *x_re, const double *x_im,
             const double *y_re, const double *y_im, double *out_re,
             double *out_im);

/* Element-wise MC scalar arithmetic on the device (twin tests of
 * _mccore.py): op 0 add, 1 sub, 2 mul, 3 div, 4 sqrt(a), 5 complex mul,
 * 6 complex div, 7 renorm of 7 terms (a is (n,7)), 8 mul((a0,0..), b),
 * 9 mul(a, (b0,0..)), 10 mul((a0,0..),(b0,0..)), 11 fused a - b*c of the
 * working-precision ILU(0) sweeps (_mcfast.rmulsubK, c passed in a_im),
 * 12 fused product (_mcfast.rmulK).  Arrays (n,k). */
int mpk_mc_elementwise(mpk_ctx *ctx, int op, int k, int64_t n,
                       const double *a_re, const double *a_im,
                       const double *b_re, const double *b_im, double *o_re,
                       double *o_im);
/* Host-side MC scalar arithmetic (MCFloat/MCComplex operators,
 * multicomponent.py:184-231): same op codes, one element, no GPU.  Host-only
 * codes 13 two_sum(a0, b0) and 14 two_prod(a0, b0) write (s, e) to o_re[0..1]
 * (the two_sum / two_prod exports, _mccore.py:19-51). */
int mpk_mc_host(int op, int k, const double *a_re, const double *a_im,
                const double *b_re, const double *b_im, double *o_re,
                double *o_im);

/* solve() (solvers.py:418-453) with precond ILU0_MIXED and spmv_mode
 * "mixed": factorization + method + true residual.  x_re/x_im receive the
 * solution (n,k); hist receives the norm2 sequence (k doubles per entry,
 * at most hist_cap entries; rep->hist_len counts all).  max_iter < 0 means
 * the reference default 3n. */
int mpk_solve(mpk_matrix *m, int method, int k, double eps_rel,
              double eps_abs, int64_t max_iter, const double *b_re,
              const double *b_im, double *x_re, double *x_im, double *hist,
              int64_t hist_cap, mpk_report *rep);

/* Same, with b and x already resident in HBM in the device PLANAR layout
 * (component c of element i at p[c*ld + i], ld = mpk_plane_ld(n); complex:
 * k real planes then k imaginary planes).  hist_dev is device memory. */
int64_t mpk_plane_ld(int64_t n);
int mpk_solve_dev(mpk_matrix *m, int method, int k, double eps_rel,
                  double eps_abs, int64_t max_iter, const double *b_dev,
                  double *x_dev, double *hist_dev, int64_t hist_cap,
                  mpk_report *rep);
/* (n,k) host <-> planar device conversion helpers */
int mpk_to_planar(mpk_ctx *ctx, int64_t n, int k, const double *re,
                  const double *im, double *dev);
int mpk_from_planar(mpk_ctx *ctx, int64_t n, int k, const double *dev,
                    double *re, double *im, int cx);

/* Kernel probe for the roofline: average device time (CUDA events on the
 * context stream) of one ILU(0)-mixed apply (forward + backward sweep
 * kernel) of a k-component input, over reps launches.  Needs factors. */
int mpk_bench_apply(mpk_matrix *m, int k, int reps, double *ms_avg);

/* Kernel probe for the SpMV roofline: average device time of one mixed
 * SpMV y = A x (binary64 A, x an exactly promoted binary64 "F" vector -- an
 * ILU(0)-mixed output, as BiCGSTAB/CGS/GPBiCG multiply -- y k-component),
 * the kernel behind spmv_mixed (sparse.py:465-480, _kernels.py:243-263). */
int mpk_bench_spmv(mpk_matrix *m, int k, int reps, double *ms_avg);

/* Sweep plan of an uploaded pattern: info[0..1] = DAG levels of the forward
 * (L) and backward (U) phases; info[2] = plan kept by the upload-time
 * autotuning (0 sync-free global, 1 single-CTA, 2 cluster, 3 ring,
 * 4 lane-chunk wavefront, 5 shuffle wavefront); for plan 5, info[3..11] =
 * line length, forward lag, groups, forward steps per group, backward lag,
 * backward steps, warps per CTA, forward / backward record bytes per chunk.
 * (Diagnostics for the bench's critical-path roofline; no reference
 * counterpart.) */
int mpk_sweep_info(mpk_matrix *m, int64_t *info, int ninfo);

/* A batch of independent solves run concurrently, one native thread per
 * job, each on its matrix's own context/stream (the reference harness runs
 * cells in a thread pool, bench.py:179-216).  device_resident = 0: b/x are
 * host (n,k) arrays as in mpk_solve, and val_re/val_im (optional) are new
 * matrix values copied in first (mpk_csr_set_values); device_resident = 1:
 * b/x are planar device buffers as in mpk_solve_dev. */
typedef struct {
  mpk_matrix *m;
  int32_t method, k;
  double eps_rel, eps_abs;
  int64_t max_iter;
  const double *b_re, *b_im;
  double *x_re, *x_im;
  const double *val_re, *val_im;
  double *hist;
  int64_t hist_cap;
  mpk_report rep; /* out */
  int32_t rc;     /* out */
} mpk_job;
int mpk_run_jobs(mpk_job *jobs, int njobs, int device_resident);

/* Independent systems (cfg5 batch): matrices[i] already uploaded, each
 * solved on its own stream of the context's device.  b/x host (n_i,k). */
int mpk_solve_batch(int nsys, mpk_matrix **ms, int method, int k,
                    double eps_rel, double eps_abs, int64_t max_iter,
                    const double *const *b_re, double *const *x_re,
                    mpk_report *reps);

/* Row-block sharded solve (BASELINE cfg4 at 1/2/4/8 GPUs).
 * The reference has no multi-process path (solvers.py is single-threaded);
 * this is the B200 extension of solve() (solvers.py:418-453) for one system
 * over W GPUs.  Every rank uploads and factors the whole matrix and runs the
 * ILU(0) sweeps in full (the triangular solve does not shard); SpMV rows,
 * vector updates and reduction partials run on the rank's block of
 * ceil(n/W) rows (W*ceil(n/W) <= mpk_plane_ld(n)).  Exchanges: in-place
 * all-gathers of the reduction block partials and of the sweep inputs'
 * head planes; the finalize folds all partials in one fixed order, so
 * every rank takes the same decisions.  b_dev/x_dev/hist_dev as in
 * mpk_solve_dev (x complete on every rank on return).  BiCGSTAB, tree
 * reductions. */
typedef struct mpk_comm mpk_comm;
/* ncclUniqueId (128 bytes) for rank 0 to broadcast (torch.distributed) */
int mpk_comm_unique_id(void *id128);
/* NCCL communicator over W processes (one GPU each) */
int mpk_comm_create(int device, int rank, int world, const void *id128,
                    mpk_comm **out);
/* W virtual ranks in ONE process on one device (tests): out[0..W-1]; each
 * rank's solve must run on its own host thread (device copies + events,
 * host barrier between the ranks' enqueues; no cross-rank kernel waits) */
int mpk_comm_create_local(int world, mpk_comm **out);
void mpk_comm_destroy(mpk_comm *c);
int mpk_comm_rank(const mpk_comm *c);
int mpk_comm_world(const mpk_comm *c);
int mpk_solve_dev_sharded(mpk_matrix *m, mpk_comm *comm, int method, int k,
                          double eps_rel, double eps_abs, int64_t max_iter,
                          const double *b_dev, double *x_dev, double *hist_dev,
                          int64_t hist_cap, mpk_report *rep);

#ifdef __cplusplus
}
#endif
#endif
