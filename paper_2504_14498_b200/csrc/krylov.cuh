// krylov.cuh -- device-side solver state and host-side solver object.
#pragma once

#include <map>
#include <memory>
#include <vector>

#include "common.cuh"
#include "ilu.cuh"
#include "shard.cuh"
#include "ilu_mc.cuh"

namespace mpk {

enum Method { kBiCG = 0, kCGS = 1, kBiCGSTAB = 2, kGPBiCG = 3 };

enum Breakdown {
  kBdNone = 0,
  kBdSigmaZero = 1,
  kBdRhoZero = 2,
  kBdOmegaZero = 3,
  kBdNonfinite = 4,
  kBdLs = 5,
  kBdZetaZero = 6,
  kBdSingularPivot = 7,
  kBdNumericFactor = 8,
  kBdNumericSweep = 9
};

// All MC scalars of the four methods live here, on the device; the host
// never sees them during the iteration (no per-iteration sync).
struct State {
  Sc rho, rho_old, alpha, omega, beta, sigma, nrm, nrm0, thr, zeta, eta;
  long long it, max_iter, iterations, hist_len, hist_cap;
  long long body_runs;  // executions of the captured iteration graph
  int pending;          // end-of-iteration test deferred to the next body
  int done, converged, breakdown, half_exit, have_nrm, sweep_err;
  double eps_rel, eps_abs;
  double relres, true_relres;
  // BiCGSTAB x update deferred beside the next sweep (krylov_impl.cuh
  // xu_kernel): iteration whose update is pending / applied, block counter
  long long xu_it, xu_done;
  int xu_cnt, xu_pad;
};

// Cached per-(method, K, field) solver workspace + graph (krylov_impl.cuh)
struct PlanBase {
  virtual ~PlanBase() {}
};

// Device matrix: binary64 CSR (int32 indices) + ILU(0) factors + the
// transposed gather structures used by the adjoint paths (BiCG).
struct DMat {
  std::map<int, std::unique_ptr<PlanBase>> plans;
  int n;
  long long nnz;
  bool cx;
  int *rp = nullptr, *ci = nullptr, *dp = nullptr;
  double *val = nullptr;  // real [nnz] or double2 [nnz]
  double *lu = nullptr;   // factors, same layout
  // MC-valued matrix (spmv_mode 'full', sparse.py:414-451): all K
  // components of every entry, planar (component c of entry p at
  // mcv[c * mcv_ld + p]; complex: K imaginary planes after the real ones);
  // null for binary64-valued matrices, whose full SpMV is the mixed one
  double *mcv = nullptr;
  int mcv_k = 0;
  long long mcv_ld = 0;
  bool factored = false;
  // A^T gather (ascending source row) for spmv_adjoint
  int *at_rp = nullptr, *at_ci = nullptr, *at_perm = nullptr;
  double *at_val = nullptr;
  // U^T (ascending rows) and L^T (descending rows) for the adjoint sweeps
  int *ut_rp = nullptr, *ut_ci = nullptr, *ut_perm = nullptr;
  int *lt_rp = nullptr, *lt_ci = nullptr, *lt_perm = nullptr;
  double *ut_val = nullptr, *lt_val = nullptr;
  bool adj_ready = false;
  long long h_adj_sizes[2] = {0, 0};
  // sweep scratch
  double *sw_y = nullptr, *sw_y2 = nullptr;
  // level orders (host-computed once per pattern): plain L / U sweeps and
  // the adjoint U^H / L^H sweeps
  int *ord_f = nullptr, *ord_b = nullptr, *ord_fa = nullptr, *ord_ba = nullptr;
  int *lev_f = nullptr, *lev_b = nullptr, *lev_fa = nullptr, *lev_ba = nullptr;
  int levels_f = 0, levels_b = 0, levels_fa = 0, levels_ba = 0;
  // sweep-pipelined SpMV (units.cu pspmv_kernel; large stencil patterns
  // whose sweeps run on the shuffle-wavefront plan): 32-row chunks sorted by
  // the backward-DAG level at which their inputs are complete, claim /
  // started counters and per-chunk done flags
  int *pipe_order = nullptr;
  int *pipe_last = nullptr;   // per chunk: the column whose z value comes last
  int pipe_nchunks = 0;
  int *pipe_state = nullptr;  // [0] claimed chunks, [1] backward CTAs running
  int *pipe_flag = nullptr;   // [pipe_nchunks]
  // factorization ticket order of deep DAGs (FactorArgs::ordp), else null
  int *ord_fp = nullptr;
  int nt_fp = 0;
  // level-ordered sweep matrices (single-CTA path, small n)
  SweepMats smat, smat_adj;
  bool smat_built = false, smat_adj_built = false;
  // working-precision ILU(0) (precond 'ilu0', ilu_mc.cu): [nnz][K] factors,
  // [n][K] reciprocal diagonals, planar K-component sweep scratch
  double *lu_mc = nullptr, *rcp_mc = nullptr, *sw_mc = nullptr, *sw_mc2 = nullptr;
  int lu_mc_k = 0;
  bool mc_factored = false;
  int *tick = nullptr;  // 4 ints: [0..1] sweep A, [2..3] sweep B
  int *err = nullptr;
  // host copies of the pattern (for building transposes)
  std::vector<int> h_rp, h_ci, h_dp;
};

// ILU(0)-mixed apply dispatch: the ring sweep (one SM, vector in shared
// memory) or the cluster sweep when its plan exists, else the prefetched
// single-CTA sweep over the level-ordered sweep matrices, else the sync-free
// multi-CTA kernel.
inline void do_sweep(const DMat &A, const SweepArgs &a, bool adjoint,
                     cudaStream_t st) {
  const bool mats = adjoint ? A.smat_adj_built : A.smat_built;
  const CSweep &cs = adjoint ? A.smat_adj.cs : A.smat.cs;
  const RSweep &rs = adjoint ? A.smat_adj.rs : A.smat.rs;
  if (!adjoint && A.smat.ss.on)
    launch_ssweep(a, A.smat.ss, st);
  else if (!adjoint && A.smat.wf.on)
    launch_wsweep(a, A.smat.wf, A.cx, st);
  else if (rs.nchunks > 0)
    launch_rsweep(a, rs, A.cx, adjoint, st);
  else if (cs.C > 0)
    launch_csweep(a, cs, A.cx, adjoint, st);
  else if (mats)
    launch_sweep_mats(a, adjoint ? A.smat_adj : A.smat, A.cx, adjoint, st);
  else
    launch_sweep(a, A.cx, adjoint, st);
}

struct SolveParams {
  int method, k;
  double eps_rel, eps_abs;
  long long max_iter;
  int precond_ilu;  // 1: ILU(0)-mixed, 0: identity, 2: working-precision ILU(0)
  long long hist_cap;
  int reduce_seq;   // 1: sequential-order (bit-identical twin) reductions
  int full_a = 0;   // 1: SpMV on the matrix's MC values (DMat::mcv)
  Exchange *ex = nullptr;  // row-block sharded solve (shard.cuh), else null
};

struct SolveOut {
  long long iterations;
  int converged, breakdown, half_exit;
  double relres, true_relres;
  long long hist_len;
  float factor_ms, loop_ms;
  long long launches;  // kernels executed by this solve
};

// Solve with the right-hand side already on the device (planar MC layout,
// K [x2] planes of ld doubles).  x_out: planar MC, hist_out: device
// [hist_cap * k] doubles.  Factorization must have been done (if ILU).
int run_solve(DMat &A, const SolveParams &p, const double *d_b, double *d_x,
              double *d_hist, SolveOut *out, cudaStream_t st, char *errbuf);

// unit kernels used by the C-ABI (parity tests)
int unit_spmv(DMat &A, int k, bool adjoint, bool x_is_f, const double *d_x,
              double *d_y, cudaStream_t st);
constexpr int kPipeRow = 12;  // longest row a pipeline plan accepts
// y (planar MC, K planes of ld) = A z for the chunks whose inputs the running
// backward sweep has already produced (z: F vector, sentinel until written);
// see units.cu.  Launches nothing and returns false when the matrix has no
// pipeline plan.
void launch_pipe_reset(DMat &A, cudaStream_t st);
void launch_pipe_delay(cudaStream_t st);
constexpr size_t kPipeSmem = 88 * 1024;  // keeps side kernels off the sweep CTAs' SMs
bool launch_pspmv(DMat &A, int k, const double *z, double *y, const int *done,
                  cudaStream_t st);
int unit_spmv_full(DMat &A, int k, bool adjoint, bool x_is_f, const double *d_x,
                   double *d_y, const int *done, cudaStream_t st);
int unit_reduce(int k, bool cx, int op, long long n, const double *d_x,
                const double *d_y, double *h_out, cudaStream_t st, int seq);
int unit_axpy(int k, bool cx, long long n, const double *alpha_re,
              const double *alpha_im, const double *d_x, const double *d_y,
              double *d_out, cudaStream_t st);
int unit_mc(int op, int k, const double *a_re, const double *a_im,
            const double *b_re, const double *b_im, double *o_re,
            double *o_im, int n, cudaStream_t st);

void ensure_adjoint(DMat &A, cudaStream_t st);

inline long long plane_ld(long long n) { return (n + 31) / 32 * 32; }

}  // namespace mpk
