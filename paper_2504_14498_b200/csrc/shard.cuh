// shard.cuh -- row-block sharded solves (BASELINE cfg4).
//
// The ILU(0) triangular solve does not shard without changing the
// preconditioner, so every rank holds the whole matrix, factors it and runs
// both sweeps of every apply in full; the row kernels (SpMV rows, vector
// updates, reduction block partials) run on the rank's contiguous block of
// nb rows.  Two exchanges per reduction / apply, both in-place all-gathers:
//   * block partials: rank r's Gl blocks land at blocks [r*Gl, (r+1)*Gl) of
//     every rank's partial array, and the one-block finalize folds all
//     W*Gl of them in the same fixed order on every rank (identical scalar
//     recurrences, identical stop decisions -> ranks stay in lockstep);
//   * the head plane of a sweep input (8 B per row): rank r's rows
//     [r*nb, (r+1)*nb) of the plane (the sweep reads the demoted vector).
// Sweep outputs (F vectors) are then complete on every rank, so the SpMV
// rows need no halo.  x is all-gathered once at the end.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace mpk {

struct Exchange {
  int rank = 0, world = 1;
  virtual ~Exchange() {}
  // buf[q*count .. (q+1)*count) <- rank q's same range, for every q
  virtual int allgather_inplace(double *buf, size_t count, cudaStream_t st) = 0;
  virtual const char *kind() const = 0;
};

// NCCL communicator (libnccl.so.2 resolved at run time: the process usually
// has torch's copy loaded already).  id: ncclUniqueId (128 bytes).
int nccl_unique_id(void *id128, char *errbuf);
Exchange *make_nccl_exchange(int device, int rank, int world, const void *id128,
                             char *errbuf);
// W virtual ranks in one process on one device (tests): each rank's solve
// runs on its own host thread and stream; the all-gather is device copies
// ordered by events, with a host barrier between the ranks' enqueues (no
// kernel ever waits on another rank's kernel).
int make_local_exchanges(int world, Exchange **out);

// Row-kernel sharding context of the calling host thread (set by the
// sharded solver while it enqueues kernels): rows() runs over [r0, r1)
// with Gl blocks writing partial blocks [boff, boff+Gl), then all-gathers
// every reduction slot.
struct ShardCtx {
  Exchange *ex = nullptr;
  long long r0 = 0, r1 = 0;
  int gl = 0, boff = 0;
};
inline thread_local ShardCtx tl_shard;

}  // namespace mpk
