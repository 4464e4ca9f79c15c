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
#include "wf.cuh"

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
  // sweep-pipelined SpMV (units.cu pspmv_kernel): every CTA of the backward
  // phase counts itself in here once it is running (null: unused)
  int *started = nullptr;
};

// Host-side hook of the pipelined SpMV: when set, a sweep plan that runs its
// two phases as two launches records this event between them (the consumer
// kernel is released when the forward phase is done, next to the backward
// launch).  Null: no event.  Only the shuffle-wavefront plan honours it.
inline thread_local cudaEvent_t tl_sweep_mid = nullptr;
// ... and makes its second launch wait for this event (work on a side stream
// that must be done before the backward phase writes the output vector).
inline thread_local cudaEvent_t tl_sweep_wait = nullptr;

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
// thread-block cluster (one SM each); levels are separated by a cluster
// barrier.  Two layouts of the vector:
//  * replicated (repl = 1, when it fits): every CTA holds the whole vector
//    in its shared memory; values are read locally and every result is
//    written to the own copy and pushed to each peer (st.shared::cluster);
//  * distributed (repl = 0): row i lives in the shared memory of the CTA
//    that computes it in the forward phase ("owner", slot s) and is read
//    with ld.shared::cluster through the packed address pk = owner<<24 | s.
// Per (level, CTA) the work is one "segment" of a byte stream, staged into
// shared memory by one bulk async copy (TMA) nbuf-1 levels ahead:
//   CSDesc[nd] | int32 ref[ne] (16-B padded) | value[ne] (f64 or double2)
// with ne = sum(cnt + hasdiv): a row's divisor is the value after its
// entries.  ref / CSDesc.row are row indices (repl) or pks (distributed).
struct __align__(16) CSDesc {
  int row;     // repl: row index; distributed: pk of the row's slot
  int e0;      // first entry, relative to the segment
  int cnt;     // entries (the divisor, if any, follows them)
  int hasdiv;  // bit 0: divisor present; bits 1..: the row's position k in
               // its CTA's compute order of the phase (dataflow mode)
};
struct CSweep {
  int C = 0, T = 0;   // cluster size, threads per CTA (0: no plan)
  int nl = 0, nf = 0; // levels (forward + backward), forward levels
  int repl = 0;       // replicated vector (see above)
  int nbuf = 3;       // staging buffers (levels in flight + 1)
  int4 *seg = nullptr;        // [nl][C] {byte offset / 16, bytes, nd, ne}
  unsigned char *stream = nullptr;
  long long *eoff = nullptr;  // per value slot: double index in the stream
  int *esrc = nullptr;        // per value slot: lu index
  long long nval = 0;
  int *slot_row = nullptr;    // distributed: [C][..] global row of each slot
  int *slot_off = nullptr;    // C+1 offsets into slot_row
  int maxslots = 0;           // vector slots per CTA
  int maxseg = 0;             // largest segment (bytes)
  size_t smem = 0;            // dynamic shared memory per CTA
  // dataflow mode (dflow = 1, replicated vector): no barrier per level --
  // a value's arrival in the local copy (it replaces a signalling-NaN
  // sentinel) is the readiness signal; three cluster barriers per apply
  // (start, forward/backward switch, end).  Initial values of each CTA's
  // rows live in a local array indexed by the row's compute position k:
  // the forward right-hand side, then y_i for the backward phase.
  int dflow = 0;
  int ninit = 0;              // max rows per CTA and phase
  int *brow = nullptr;        // [C][..] backward rows in compute order
  int *boff = nullptr;        // C+1 offsets into brow
};

// Ring sweep plan: one CTA holds the whole vector in shared memory; both
// phases' rows (level order) and entries are laid out as a byte stream of
// "chunks" (a chunk = consecutive rows of one level: RDesc[nrows] | col
// int32[nent] | val f64-or-double2[nent], 16-byte aligned) that a producer
// warp streams through a ring of shared-memory slots with bulk async copies
// (TMA), while the consumer warps process the previous chunks.  Levels are
// separated by a named barrier of the consumer warps only.
struct __align__(16) RDesc {
  int row;     // global row
  int e0;      // first entry, relative to the chunk
  int cnt;     // entries
  int hasdiv;  // divide by d at the end
  double dr, di;
};
struct RChunk {  // device + host metadata of one chunk
  long long off; // byte offset in the stream
  int bytes;     // multiple of 16
  int nrows, nent;
  int level_end; // last chunk of its level: barrier after it
  int fwd;       // forward phase
  int pad;
};
struct RSweep {
  int nchunks = 0, S = 0, slot = 0;  // chunks, ring slots, slot bytes
  int T = 0;                         // threads (consumers + 1 producer warp)
  unsigned char *stream = nullptr;   // device byte stream
  RChunk *chunks = nullptr;          // device chunk table
  long long *eoff = nullptr;         // per entry: double index of its value
  int *esrc = nullptr;               // per entry: lu index
  long long nent = 0;
  long long *doff = nullptr;         // per row desc: double index of dr
  int *dsrc = nullptr;               // per row desc: lu index (-1: none)
  long long ndesc = 0;
  size_t smem = 0;
};

struct SweepMats {
  SweepPhase fwd, bwd;
  bool conj = false;  // adjoint: values are conjugated at use
  CSweep cs;          // cluster plan (cs.C > 0 when built)
  RSweep rs;          // ring plan (rs.nchunks > 0 when built)
  WSweep wf;          // lane-chunk wavefront plan (wf.on when kept; wf.cu)
  SSweep ss;          // shuffle-wavefront plan (ss.on when kept; swf.cu)
};
// wavefront plan (wf.cuh): analysis at upload, values gathered per factorization
bool build_wsweep(WSweep &w, int n, bool cx, const int *rp, const int *ci,
                  const int *dp, int nlev_f, int nlev_b, cudaStream_t st);
void gather_wsweep(const double *lu, const WSweep &w, bool cx, cudaStream_t st);
void launch_wsweep(const SweepArgs &a, const WSweep &w, bool cx, cudaStream_t st);
void free_wsweep(WSweep &w);
// shuffle-wavefront plan (swf.cu): stencil-structured real sweeps
bool build_ssweep(SSweep &w, int n, bool cx, const int *rp, const int *ci, const int *dp,
                  cudaStream_t st);
void gather_ssweep(const double *lu, const SSweep &w, cudaStream_t st);
void launch_ssweep(const SweepArgs &a, const SSweep &w, cudaStream_t st);
void free_ssweep(SSweep &w);
int ssweep_bwd_ctas(const SSweep &w);
void launch_rsweep(const SweepArgs &a, const RSweep &p, bool cx, bool adjoint,
                   cudaStream_t st);
void gather_rsweep(const double *lu, const RSweep &p, bool cx, cudaStream_t st);
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
  // ticket order of the multi-CTA kernel for deep DAGs: the level order with
  // every level padded (-1) to a multiple of 32 tickets, so that the 32 rows
  // a warp claims always belong to ONE level and never wait on each other
  const int *ordp = nullptr;
  int nt = 0;      // padded ticket count
  // Publication by value (real matrices whose rows all fit factor_row_local):
  // a copy of the factors, sentinel-filled before the launch, into which a
  // finished row writes its diagonal and upper part with plain relaxed
  // stores; consumers poll the values they need (as the sweeps do), so no
  // flag, no release fence and no separate fetch sit between two DAG levels.
  double *pub = nullptr;
  int *tick;       // [0] ticket, [1] exit counter
  int *bad_row;    // atomicMin of zero-pivot rows (init INT_MAX)
  int *nonfinite;  // set if any factor is non-finite
};
void launch_factor(const FactorArgs &a, bool cx, cudaStream_t st);
void launch_fill_sentinel(double *p, long long n, cudaStream_t st);

}  // namespace mpk
