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
};

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

template <int K, bool CX, int NH, int NN, class F>
__global__ void __launch_bounds__(kBlock)
    rows_kernel(long long n, const int *done, double *part, F f) {
  if (done && *done) return;
  __shared__ double smem[kWarpsPerBlock * 8];
  Red<K, CX, NH, NN> red;
  red.zero();
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n;
       i += (long long)gridDim.x * kBlock)
    f(i, red);
  if constexpr (NH + NN > 0) red.store(part, smem);
}

// Every kernel of the solver asks for the max-shared-memory carveout, so
// SMs never have to be reconfigured between the SMEM-resident sweep and the
// other kernels (which would serialise concurrent solves on other streams).
template <class KFn>
inline void prefer_max_smem(KFn kfn) {
  static bool done_once = false;
  if (!done_once) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    done_once = true;
  }
}

template <int K, bool CX, int NH, int NN, class F>
void rows(long long n, const int *done, double *part, cudaStream_t st, F f) {
  ++tl_launches;
  prefer_max_smem(rows_kernel<K, CX, NH, NN, F>);
  rows_kernel<K, CX, NH, NN, F><<<grid_for(n), kBlock, 0, st>>>(n, done, part, f);
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
  __shared__ double smem[kWarpsPerBlock * 8];
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
