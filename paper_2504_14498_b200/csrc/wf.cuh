// wf.cuh -- lane-chunk wavefront ("WF") plan for the binary64 ILU(0) sweeps.
//
// Reference: ilu.py:322-343 (_sweep_forward / _sweep_backward).  Per-row
// arithmetic is the reference's (ascending entries, final division), so
// results are bitwise those of every other sweep path; only the schedule
// differs.
//
// Idea.  For matrices whose sweep DAG is "banded" -- every dependency of the
// row at phase position p lies at most D positions back (a natural-order
// grid stencil: D = grid line + 1) -- the phase order is cut into chunks of
// Lc consecutive positions (one grid line), and chunk l is processed by
// "lane" l strictly in order, with lane l skewed `lag` steps behind lane
// l-1 (position x of lane l runs at step x + lag*l).  The host analysis
// picks Lc and the smallest lag for which every dependency is produced at an
// earlier step.  32 consecutive lanes form a group, run by ONE warp in
// lockstep (a __syncwarp per step): dependencies inside the group come from
// a per-warp shared-memory ring of the last H steps' outputs (no L2 round
// trip on the critical path), older or cross-group ones from global memory
// with sentinel polling (groups are claimed in order through a ticket, so a
// warp only waits on lower-ticket warps that are resident: deadlock-free).
// The critical path is then ~ (groups x 32 x lag + S) warp steps of a few
// dependent FP64 ops each, instead of one device-wide synchronisation per
// DAG level (cfg4: 6142 levels per phase).
//
// The per-(group, step) entries are pre-laid out as fixed-size records
//   int32 off[EM][32] | int32 col[EM][32] | value[EM][32] | divisor[32]
// (off: shared-memory source of the value -- ring, stage or zero slot;
// col: global row of a staged value), T records + a fetch table (the
// chunk's staged values spread over the 32 lanes) per chunk, streamed into
// shared memory by one bulk async copy (TMA) per chunk, NB in flight.
#pragma once

#include "common.cuh"

namespace mpk {

constexpr int kWfEM = 4;        // entry slots per row (rows with more: no plan)
constexpr int kWfH = 16;        // ring depth (steps)
constexpr int kWfT = 8;         // steps per bulk copy
constexpr int kWfNB = 4;        // copies in flight (buffers)
constexpr int kWfSkip = 0x7fffffff;

struct WPhase {
  int fwd = 1;          // forward: positions = rows ascending; backward: descending
  int Lc = 0, lag = 0;  // chunk length (positions per lane), skew per lane
  int nlanes = 0, ngroups = 0;
  int S = 0;            // steps per group, padded to a multiple of kWfT
  int recsz = 0;        // bytes per step record
  int kmax = 0;         // fetch-table rounds per chunk (32 items each)
  int chunkb = 0;       // bytes per chunk: T records + fetch table
  int rhs16 = 0;        // lane rows 16-byte aligned per chunk (vector rhs copies)
  unsigned char *rec = nullptr;  // [ngroups][S/T] chunks
  int *esrc = nullptr;  // per value slot ((g*S+s)*EM+e)*32+j: lu index or -1
  int *dsrc = nullptr;  // per divisor slot (g*S+s)*32+j: lu index or -1
  long long nslots = 0, ndslots = 0;
  long long cost = 0;   // modelled critical path (warp steps)
};

struct WSweep {
  int on = 0;
  WPhase f, b;
  int wpb = 0;          // warps per CTA
  size_t smem = 0;      // dynamic shared memory per CTA
};

}  // namespace mpk

namespace mpk {

// Shuffle-wavefront plan (swf.cu): stencil-structured real sweeps, one
// phase per launch.  Records: per (group, chunk of kSwfT steps) the steps'
// factor values [step][nk/2][32 lanes][2] (+ backward: [32][divisor, RN
// reciprocal]) -- chunkb bytes, streamed by one TMA bulk copy per chunk.
constexpr int kSwfT = 16;
constexpr int kSwfMaxW = 2;

struct SPhase {
  int fwd = 1;
  int Lc = 0, lag = 0, nlanes = 0, ngroups = 0;
  int S = 0, nch = 0;     // steps per group (multiple of kSwfT), chunks
  int pat = 0, nk = 0;    // key pattern (swf.cu kPat), value slots per row
  int chunkb = 0;         // bytes per chunk record
  int wbytes = 0;         // shared memory per warp
  int rhs16 = 0;          // 16-byte right-hand-side copies possible
  int rpf = 0;            // L2 prefetch distance of the right-hand sides (chunks, 0: off)
  int pf = 0;             // L2 prefetch distance of the records (chunks, 0: off)
  int cl = 1;             // thread-block cluster size (1: ticketed CTAs)
  unsigned char *rec = nullptr;
  int *esrc = nullptr;    // value slot ((g*S+s)*nk+e)*32+j -> lu index / -1
  int *dsrc = nullptr;    // divisor slot (g*S+s)*32+j -> lu index / -1
  long long nslots = 0, ndslots = 0;
};

struct SSweep {
  int on = 0;
  SPhase f, b;
  int W = 0;           // warps (groups) per CTA
  size_t smem = 0;     // dynamic shared memory per CTA
  long long cost = 0;  // modelled critical path (steps)
};

}  // namespace mpk
