// ilu.cuh -- binary64 ILU(0) factorization and triangular sweeps on sm_100a.
//
// Reference: ilu.py:178-276 (_factorize_tuples, k=1), :322-343 (sweeps),
// :346-371 (adjoint sweeps), :448-470 (mixed apply = promote . f64 . demote).
//
// Bit-exactness: each row is processed by ONE thread in exactly the
// reference's per-row order (ascending L columns; ascending U columns;
// final division), with explicit _rn intrinsics (no FMA contraction).
// Parallelism comes from the DAG: rows are claimed in dependency-compatible
// order through an atomic ticket (forward rows ascending, backward rows
// descending), and a row waits only on rows with smaller tickets, which are
// held by resident warps -> deadlock-free without a level barrier
// ("sync-free" scheduling; critical path = level depth).
// Readiness is signalled by the value itself: outputs are pre-filled with a
// signalling-NaN sentinel and read with L1-bypassing volatile loads.
#pragma once

#include "common.cuh"

namespace mpk {

struct SweepArgs {
  int n;
  // level schedule: rows sorted by level (a topological order of the sweep
  // DAG), lev_f[L]..lev_f[L+1] = rows of forward level L (ord_f), same for
  // the backward phase.  Used by the single-CTA shared-memory kernel.
  const int *ord_f, *ord_b, *lev_f, *lev_b;
  int nlev_f, nlev_b;
  const int *rp, *ci, *dp;
  const double *lu;  // real: [nnz]; complex: double2 [nnz]
  // adjoint gather structures (BiCG): U^T rows ascending, L^T descending
  const int *ut_rp, *ut_ci;
  const double *ut_val;  // real [nnzU] / complex double2
  const int *lt_rp, *lt_ci;
  const double *lt_val;
  // input: head plane(s) of an MC vector (complex: re plane, im plane)
  const double *in_re, *in_im;
  // scratch y (sentinel-filled) and output z (F vector, sentinel-filled)
  double *y, *z;
  int *tick;       // [0] ticket, [1] exit counter
  int *err;        // set to 1 on a non-finite z (NumericBreakdownError)
  const int *done; // solver done flag (skip when set), may be null
};

// Level-ordered copy of one sweep phase ("sweep matrix"): position r in
// level order holds row row[r] whose entries are col/val[ptr[r]..ptr[r+1])
// in the reference's per-row order; dval[r] is the divisor (backward plain
// / forward adjoint phases).  Values are gathered from the factors (src,
// dsrc) after every factorization.
struct SweepPhase {
  int nlev = 0;
  int maxw = 0;         // widest level (rows)
  int *lev = nullptr;   // nlev+1 level pointers into [0, n]
  int4 *desc = nullptr; // n: {row, first entry, entry count, 0} per position
  int *col = nullptr;   // entries, level order, reference order per row
  int *src = nullptr;   // entry -> index into lu
  double *val = nullptr;
  int *dsrc = nullptr;  // n, -1 if no divisor
  double *dval = nullptr;
  long long nent = 0;
};

// Cluster sweep plan: both phases of one apply split over the C CTAs of a
// thread-block cluster (one SM each).  Row i's value lives in the shared
// memory of the CTA that computes it in the forward phase ("owner", slot s);
// every reference to it is a packed address pk = owner << 24 | s read with
// ld.shared::cluster (DSMEM).  Per (level, CTA) the row descriptors and
// entries are contiguous ("segments"), staged into shared memory by bulk
// async copies two levels ahead; levels are separated by a cluster barrier.
struct __align__(16) CDesc {
  int init;   // pk of the initial value (forward: rhs in own slot; backward: y_i)
  int out;    // pk the result is stored to (row's owner slot)
  int e0;     // first entry, relative to the segment
  int cnt;    // entries
  int row;    // global row (z output, rhs)
  int hasdiv; // divide by d at the end
  int pad0, pad1;
  double dr, di;  // divisor (gathered from the factors)
};
struct __align__(16) CEntR {
  double v;
  int pk;
  int pad;
};
struct __align__(16) CEntC {
  double vr, vi;
  int pk;
  int pad[3];
};
struct CSweep {
  int C = 0, T = 0;   // cluster size, threads per CTA (0: no plan)
  int nl = 0, nf = 0; // levels (forward + backward), forward levels
  int4 *seg = nullptr;        // [nl][C] {desc_off, ndesc, ent_off, nent}
  CDesc *desc = nullptr;
  int *dsrc = nullptr;        // per descriptor: lu index of divisor or -1
  void *ent = nullptr;        // CEntR / CEntC
  int *esrc = nullptr;        // per entry: lu index
  int *slot_row = nullptr;    // [C][..] global row held in each slot
  int *slot_off = nullptr;    // C+1 offsets into slot_row
  long long ndesc = 0, nent = 0;
  int maxslots = 0, maxdesc = 0, maxent = 0;
  size_t smem = 0;            // dynamic shared memory per CTA
};

struct SweepMats {
  SweepPhase fwd, bwd;
  bool conj = false;  // adjoint: values are conjugated at use
  CSweep cs;          // cluster plan (cs.C > 0 when built)
};
// cluster sweep over a plan (values gathered); cfg: env MPK_CSWEEP_C
void launch_csweep(const SweepArgs &a, const CSweep &p, bool cx, bool adjoint,
                   cudaStream_t st);
void gather_csweep(const double *lu, const CSweep &p, bool cx, cudaStream_t st);
size_t csweep_smem_limit();

void launch_sweep(const SweepArgs &a, bool cx, bool adjoint,
                  cudaStream_t st);
// single-CTA prefetched sweep over prepared sweep matrices (small n)
void launch_sweep_mats(const SweepArgs &a, const SweepMats &m, bool cx,
                       bool adjoint, cudaStream_t st);
bool sweep_uses_smem(int n, bool cx);
void launch_sweep_reset(double *y, double *z, int n, bool cx,
                        const int *done, cudaStream_t st);

struct FactorArgs {
  int n;
  const int *rp, *ci, *dp;
  double *lu;      // in: A values, out: factors (in place)
  int *rowflag;    // per-row completion flags (zeroed)
  const int *ord;  // level order of the L DAG (single-CTA path)
  const int *lev;  // level pointers into ord
  int nlev;
  int *tick;       // [0] ticket, [1] exit counter
  int *bad_row;    // atomicMin of zero-pivot rows (init INT_MAX)
  int *nonfinite;  // set if any factor is non-finite
};
void launch_factor(const FactorArgs &a, bool cx, cudaStream_t st);

}  // namespace mpk
