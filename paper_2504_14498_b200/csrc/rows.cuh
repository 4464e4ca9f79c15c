// rows.cuh -- SpMV row and fused row-kernel / finalize-kernel framework.
#pragma once

#include "krylov.cuh"

namespace mpk {

// ---------------------------------------------------------------------
// SpMV row (sparse.py:465-496 -> _kernels.py:243-263,281-297,326-353,
// 379-400): ascending column order, A promoted exactly per product.
// ---------------------------------------------------------------------
struct DA {
  int n;
  const int *rp, *ci;
  const double *val;
  const int *at_rp, *at_ci;
  const double *at_val;
  // MC-valued matrix (spmv_mode 'full'): A x / A^H x were formed by the
  // full-precision kernel (units.cu spmv_full_kernel) into these planar MC
  // vectors just before the row kernel; null otherwise
  const double *pre = nullptr, *pre_adj = nullptr;
  // sweep-pipelined SpMV: `pre` holds A x only for the 32-row chunks whose
  // flag is set (rows the pipeline kernel finished while the sweep ran);
  // null: every row of `pre` is valid
  const int *pflag = nullptr;
};

template <int K, bool CX>
__device__ __forceinline__ void load_pre(const double *q, long long ld, int i,
                                         double (&yr)[K], double (&yi)[K]) {
#pragma unroll
  for (int c = 0; c < K; ++c) {
    yr[c] = q[c * ld + i];
    yi[c] = CX ? q[(K + c) * ld + i] : 0.0;
  }
}

template <int K, bool CX, bool XF, bool ADJ>
__device__ __forceinline__ void spmv_row(const DA &A, int i, const double *x,
                                         long long ld, double (&yr)[K],
                                         double (&yi)[K]) {
  const int *rp = ADJ ? A.at_rp : A.rp;
  const int *ci = ADJ ? A.at_ci : A.ci;
  const double *val = ADJ ? A.at_val : A.val;
#pragma unroll
  for (int c = 0; c < K; ++c) yr[c] = yi[c] = 0.0;
  const int lo = rp[i], hi = rp[i + 1];
  for (int p = lo; p < hi; ++p) {
    const int j = ci[p];
    if constexpr (!CX) {
      const double a = val[p];
      if constexpr (XF) {
        double h, l;
        mul_ff2(a, x[j], h, l);
        add2<K>(yr, h, l, yr);
      } else {
        double xj[K], t[K];
#pragma unroll
        for (int c = 0; c < K; ++c) xj[c] = x[c * ld + j];
        mul_lf<K>(a, xj, t);
        add<K>(yr, t, yr);
      }
    } else {
      const double2 av = reinterpret_cast<const double2 *>(val)[p];
      const double ar = av.x, ai = ADJ ? -av.y : av.y;
      double pr[K], pi[K];
      if constexpr (XF) {
        const double2 xv = reinterpret_cast<const double2 *>(x)[j];
        cmul_ff<K>(ar, ai, xv.x, xv.y, pr, pi);
      } else {
        double xr[K], xi[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          xr[c] = x[c * ld + j];
          xi[c] = x[(K + c) * ld + j];
        }
        cmul_lf<K>(ar, ai, xr, xi, pr, pi);
      }
      add<K>(yr, pr, yr);
      add<K>(yi, pi, yi);
    }
  }
}

// SpMV row on an "applied" vector: the binary64 head of an ILU(0)-mixed
// output (promoted per product), or, preconditioner 'none' (mc != 0), the
// full MC vector (solvers.py:128-136: M = I returns the vector itself)
template <int K, bool CX>
__device__ __forceinline__ void spmv_fv(const DA &A, int i, const double *x,
                                        long long ld, int mc, double (&yr)[K],
                                        double (&yi)[K]) {
  if (A.pre && (!A.pflag || A.pflag[i >> 5]))
    load_pre<K, CX>(A.pre, ld, i, yr, yi);
  else if (mc)
    spmv_row<K, CX, false, false>(A, i, x, ld, yr, yi);
  else
    spmv_row<K, CX, true, false>(A, i, x, ld, yr, yi);
}

// SpMV row (plain or adjoint) on a full MC vector
template <int K, bool CX, bool ADJ>
__device__ __forceinline__ void spmv_mc(const DA &A, int i, const double *x,
                                        long long ld, double (&yr)[K],
                                        double (&yi)[K]) {
  const double *q = ADJ ? A.pre_adj : A.pre;
  if (q)
    load_pre<K, CX>(q, ld, i, yr, yi);
  else
    spmv_row<K, CX, false, ADJ>(A, i, x, ld, yr, yi);
}

// ---------------------------------------------------------------------
// row-kernel framework: NH complex-or-real hdot slots + NN norm slots
// ---------------------------------------------------------------------
template <int K, bool CX, int NH, int NN>
struct Red {
  Acc<K, CX> h[NH > 0 ? NH : 1];
  Acc<K, false> nr[NN > 0 ? NN : 1];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int s = 0; s < (NH > 0 ? NH : 1); ++s) h[s].zero();
#pragma unroll
    for (int s = 0; s < (NN > 0 ? NN : 1); ++s) nr[s].zero();
  }
  __device__ __forceinline__ void store(double *part, double *smem) {
#pragma unroll
    for (int s = 0; s < NH; ++s) {
      block_reduce<K, CX>(h[s], smem);
      store_partial<K, CX>(part, s, h[s]);
    }
#pragma unroll
    for (int s = 0; s < NN; ++s) {
      block_reduce<K, false>(nr[s], smem);
      store_partial<K, false>(part, NH + s, nr[s]);
    }
  }
};

// Blocks per SM the row kernels are compiled for (the register cap).  The
// reduction tree is fixed at kMaxGrid = 4 x 148 block partials, so a kernel
// that fits 4 blocks per SM (<= 64 registers) runs its 592 blocks in ONE
// wave; at 3 per SM (the 68-register DD SpMV / update kernels of cfg4) the
// grid took 1.33 waves with a third of the SMs' warp slots idle in the
// second (ncu r02: achieved occupancy 30 %, 44 % of cycles without an
// eligible warp).  Real DD kernels fit 64 registers without spilling; the
// complex / TD / QD kernels keep 3 blocks per SM (80 registers; concurrent
// solves of cfg2 / cfg5 compete for warp slots).
#ifndef MPK_ROWS_MIN_BLOCKS_DD
#define MPK_ROWS_MIN_BLOCKS_DD 4
#endif
#ifndef MPK_ROWS_MIN_BLOCKS
#define MPK_ROWS_MIN_BLOCKS 3
#endif
#ifndef MPK_ROWS_MIN_BLOCKS_QD
#define MPK_ROWS_MIN_BLOCKS_QD MPK_ROWS_MIN_BLOCKS
#endif
template <int K, bool CX>
constexpr int rows_min_blocks() {
  return (K == 2 && !CX) ? MPK_ROWS_MIN_BLOCKS_DD
                         : (K == 4 ? MPK_ROWS_MIN_BLOCKS_QD : MPK_ROWS_MIN_BLOCKS);
}
template <int K, bool CX, int NH, int NN, class F>
__global__ void __launch_bounds__(kBlock, rows_min_blocks<K, CX>())
    rows_kernel(long long n_total, long long n, const int *done, double *part,
                double *seq, F f, long long i0) {
  // n_total = roles * n: element i of role r is index r * n + i; only role 0
  // (i < n) contributes to the reductions
  if (done && *done) return;
  __shared__ double smem[kWarpsPerBlock * 8];
  Red<K, CX, NH, NN> red;
  red.zero();
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n_total;
       i += (long long)gridDim.x * kBlock) {
    if (seq) {  // twin mode: element i's terms -> seq[slot][i]
      const bool own = i < n;
#pragma unroll
      for (int s = 0; s < NH; ++s)
        red.h[s].seq = own ? seq + ((size_t)s * n + i) * 2 * K : nullptr;
#pragma unroll
      for (int s = 0; s < NN; ++s)
        red.nr[s].seq = own ? seq + ((size_t)(NH + s) * n + i) * 2 * K : nullptr;
    }
    f(i0 + i, red);
  }
  if constexpr (NH + NN > 0)
    if (!seq) red.store(part, smem);
}

// Twin mode: one lane per chain folds the element terms in ascending order
// exactly like dot_real / hdot_cx / sumsq_* (_kernels.py:487-552), and
// stores the sum as block partial 0 of its slot (the finalize then runs
// with G = 1; adding the zero lanes of its tree is exact for a renormalised
// value).  Chains: hdot slots 1 (real) or 2 (re, im); norm slots 1, with
// two terms per element for the complex field.
template <int K, bool CX, int NH, int NN>
__global__ void seq_chain_kernel(long long n, const int *done,
                                 const double *seq, double *part) {
  if (done && *done) return;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;
  constexpr int NHC = NH * (CX ? 2 : 1);
  int slot, off, per;
  if (w < NHC) {
    slot = CX ? w / 2 : w;
    off = CX ? (w % 2) * K : 0;
    per = 1;
  } else if (w < NHC + NN) {
    slot = NH + (w - NHC);
    off = 0;
    per = CX ? 2 : 1;
  } else {
    return;
  }
  const double *b = seq + (size_t)slot * n * 2 * K;
  double acc[K], t[K], nx[K];
#pragma unroll
  for (int c = 0; c < K; ++c) acc[c] = 0.0;
  const long long m = n * per;
  auto term = [&](long long j, double(&o)[K]) {
    const long long i = per == 2 ? j >> 1 : j;
    const int o2 = per == 2 ? (int)(j & 1) * K : off;
#pragma unroll
    for (int c = 0; c < K; ++c) o[c] = b[(size_t)i * 2 * K + o2 + c];
  };
  if (m > 0) term(0, nx);
  for (long long j = 0; j < m; ++j) {
#pragma unroll
    for (int c = 0; c < K; ++c) t[c] = nx[c];
    if (j + 1 < m) term(j + 1, nx);  // prefetch overlaps the add
    add<K>(acc, t, acc);
  }
  double *q = part + ((size_t)slot * kMaxGrid) * 8;
  const int base = (CX && w < NHC && (w % 2)) ? 4 : 0;
#pragma unroll
  for (int c = 0; c < K; ++c) q[base + c] = acc[c];
  if (!CX || w >= NHC) {
#pragma unroll
    for (int c = 0; c < K; ++c) q[4 + c] = 0.0;
  }
}

// Every kernel of the solver asks for the max-shared-memory carveout, so
// SMs never have to be reconfigured between the SMEM-resident sweep and the
// other kernels (which would serialise concurrent solves on other streams).
template <class KFn>
inline void prefer_max_smem(KFn kfn) {
  static bool done_once = false;
  static const bool off = getenv("MPK_NO_MAX_SMEM") != nullptr;  // A/B knob
  if (!done_once && !off) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    done_once = true;
  }
}

// roles > 1: the kernel runs roles * n threads; f(i) with i >= n does the
// independent part of element i % n assigned to role i / n (see callers)
//
// Row-block sharded solve (shard.cuh, tl_shard set): the kernel covers the
// rank's rows [r0, r1) with Gl blocks whose partials land at blocks
// [boff, boff+Gl) of every slot, then each reduction slot is all-gathered
// in place so that every rank folds the same W*Gl partials.
template <int K, bool CX, int NH, int NN, class F>
void rows(long long n, const int *done, double *part, cudaStream_t st, F f,
          int roles = 1) {
  ++tl_launches;
  prefer_max_smem(rows_kernel<K, CX, NH, NN, F>);
  double *seq = (NH + NN > 0) ? tl_seq : nullptr;
  const ShardCtx &sh = tl_shard;
  if (sh.ex && roles == 1 && !seq) {
    const long long nl = sh.r1 - sh.r0;
    rows_kernel<K, CX, NH, NN, F><<<sh.gl, kBlock, 0, st>>>(
        nl, nl, done, part + (size_t)sh.boff * 8, nullptr, f, sh.r0);
    for (int s = 0; s < NH + NN; ++s)
      sh.ex->allgather_inplace(part + (size_t)s * kMaxGrid * 8, (size_t)sh.gl * 8, st);
    return;
  }
  const long long nt = n * roles;
  rows_kernel<K, CX, NH, NN, F><<<grid_for(nt), kBlock, 0, st>>>(nt, n, done, part,
                                                                  seq, f, 0);
  if (seq) {
    ++tl_launches;
    constexpr int chains = NH * (CX ? 2 : 1) + NN;
    seq_chain_kernel<K, CX, NH, NN><<<1, 32 * chains, 0, st>>>(n, done, seq, part);
  }
}

template <class F>
__global__ void __launch_bounds__(kBlock)
    fin_kernel(State *S, const int *err, const double *part, int G, F f) {
  if (S->done) return;
  if (err && *err) {
    if (threadIdx.x == 0) {
      S->iterations = 0;
      S->converged = 0;
      S->breakdown = kBdNumericSweep;
      S->sweep_err = 1;
      S->done = 1;
    }
    return;
  }
  __shared__ double smem[kWarpsPerBlock * 16];  // finalize_slots scratch
  f(S, part, G, smem);
}

template <class F>
void fin(State *S, const int *err, const double *part, int G, cudaStream_t st,
         F f) {
  ++tl_launches;
  prefer_max_smem(fin_kernel<F>);
  fin_kernel<F><<<1, kBlock, 0, st>>>(S, err, part, G, f);
}

}  // namespace mpk
