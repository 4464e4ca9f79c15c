// ilu_mc.cuh -- working-precision ILU(0) (precond 'ilu0'), see ilu_mc.cu.
#pragma once

#include "common.cuh"

namespace mpk {

struct FactorMcArgs {
  int n;
  int cx;          // complex field: values are flat (re[K], im[K])
  const int *rp, *ci, *dp;
  double *lu;      // [nnz][K]: in A promoted, out the factors (in place)
  int *rowflag;    // per-row completion flags (zeroed)
  int *tick;       // [0] ticket, [1] exit counter
  int *bad_row;    // atomicMin of zero-pivot rows (init INT_MAX)
  int *nonfinite;  // set if any factor is non-finite
  const int *ord;  // tickets -> rows in level order of the L DAG (or null)
};
struct SweepMcArgs {
  int n;
  int cx;
  long long ld;          // plane stride of in / y / z
  const int *rp, *ci, *dp;
  const double *lu;      // [nnz][K] factors
  const double *rcp;     // real [n][K] mc_div(1, U_ii); complex [2n][2K+1]
                         // Smith diagonals (plain, then adjoint)
  const double *in;      // planar K-component input
  double *y, *z;         // planar scratch / output (plane 0 sentinel-reset here)
  int *tick;
  int *err;
  const int *done;
  // adjoint (BiCG, ilu.py:346-371): gathers over U^T (ascending source
  // rows) and L^T (descending), values at lu[perm[q]]
  int adjoint;
  const int *ut_rp, *ut_ci, *ut_perm, *lt_rp, *lt_ci, *lt_perm;
  // tickets -> rows in level order of the phase's DAG (null: natural order);
  // a warp's 32 rows then rarely depend on each other
  const int *ord_f, *ord_b;
};
void launch_factor_mc(const FactorMcArgs &a, int k, cudaStream_t st);
void launch_recip_mc(int n, const int *dp, const double *lu, double *rcp, int k, bool cx,
                     cudaStream_t st);
void launch_sweep_mc(const SweepMcArgs &a, int k, cudaStream_t st);

}  // namespace mpk
