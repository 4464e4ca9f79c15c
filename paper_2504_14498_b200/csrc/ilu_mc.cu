// ilu_mc.cu -- working-precision ILU(0) (precond 'ilu0'):
// factorization in K-component arithmetic and its forward / backward
// sweeps on K-component vectors, real field.
//
// Reference: ilu.py:178-276 (_factorize_tuples with k > 1: lik = mc_div,
// a_ij = _mcfast.rmulsubK(a_ij, lik, u_kj)), ilu.py:322-343 (sweeps:
// acc = rmulsubK(acc, l_ij, y_j) ascending j; backward acc / U_ii through
// _mcfast.RealDiag = rmulK(acc, mc_div(1, U_ii))), ilu.py:374-420.
// Scheduling is the sync-free ticket scheme of ilu.cu (one row per thread,
// rows claimed in dependency-compatible order, a row waits only on rows
// with smaller tickets).  A K-component value is published by writing
// components 1..K-1, a fence, then component 0 over its signalling-NaN
// sentinel; a reader polls component 0, fences, then reads the rest.
#include <climits>

#include "ilu_mc.cuh"

namespace mpk {

namespace {

constexpr unsigned kFullM = 0xffffffffu;

__device__ __forceinline__ int mc_grab(int *tick) {
  int base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(tick, 32);
  return __shfl_sync(kFullM, base, 0);
}
__device__ __forceinline__ void mc_exit(int *tick) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    const int total = gridDim.x * (blockDim.x >> 5);
    __threadfence();
    if (atomicAdd(&tick[1], 1) == total - 1) {
      atomicExch(&tick[0], 0);
      atomicExch(&tick[1], 0);
    }
  }
}
__device__ __forceinline__ double ldr(const double *p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void str(double *p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ int ldri(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// K-component value j of a planar vector (stride ld), published by another row
template <int K>
__device__ __forceinline__ void poll_mc(const double *v, long long ld, int j,
                                        double (&o)[K]) {
  double h = ldr(v + j);
  while (is_sent(h)) {
    __nanosleep(32);
    h = ldr(v + j);
  }
  __threadfence();
  o[0] = h;
#pragma unroll
  for (int c = 1; c < K; ++c) o[c] = ldr(v + c * ld + j);
}
template <int K>
__device__ __forceinline__ void pub_mc(double *v, long long ld, int j,
                                       const double (&x)[K]) {
#pragma unroll
  for (int c = 1; c < K; ++c) str(v + c * ld + j, x[c]);
  __threadfence();
  str(v + j, unsent(x[0]));
}

template <int K>
__device__ void factor_mc_row(const FactorMcArgs &a, int i) {
  const int lo = a.rp[i], hi = a.rp[i + 1], d = a.dp[i];
  double *lu = a.lu;
  for (int t = lo; t < d; ++t) {
    const int kc = a.ci[t];
    while (ldri(&a.rowflag[kc]) == 0) __nanosleep(32);
    __threadfence();
    const int uk = a.dp[kc], kend = a.rp[kc + 1];
    double at[K], ukk[K], l[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      at[c] = __ldcg(&lu[(size_t)t * K + c]);
      ukk[c] = __ldcg(&lu[(size_t)uk * K + c]);
    }
    div<K>(at, ukk, l);  // mc_div (_mccore.py:222-237)
#pragma unroll
    for (int c = 0; c < K; ++c) __stcg(&lu[(size_t)t * K + c], l[c]);
    int q = t + 1;
    for (int s = uk + 1; s < kend; ++s) {
      const int col = a.ci[s];
      while (q < hi && a.ci[q] < col) ++q;
      if (q < hi && a.ci[q] == col) {
        double v[K], u[K], r[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          v[c] = __ldcg(&lu[(size_t)q * K + c]);
          u[c] = __ldcg(&lu[(size_t)s * K + c]);
        }
        fmulsub<K>(v, l, u, r);  // _mcfast.rmulsubK(a_ij, lik, u_kj)
#pragma unroll
        for (int c = 0; c < K; ++c) __stcg(&lu[(size_t)q * K + c], r[c]);
      }
    }
  }
  bool zero = true, fin = true;
#pragma unroll
  for (int c = 0; c < K; ++c) zero = zero && __ldcg(&lu[(size_t)d * K + c]) == 0.0;
  for (int p = lo; p < hi; ++p)
    for (int c = 0; c < K; ++c) fin = fin && isfin(__ldcg(&lu[(size_t)p * K + c]));
  if (zero) atomicMin(a.bad_row, i);
  if (!fin) atomicOr(a.nonfinite, 1);
  __threadfence();
  atomicExch(&a.rowflag[i], 1);
}

template <int K>
__global__ void __launch_bounds__(256) factor_mc_kernel(FactorMcArgs a) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const int base = mc_grab(a.tick);
    if (base >= a.n) break;
    const int t = base + lane;
    if (t < a.n) factor_mc_row<K>(a, t);
  }
  mc_exit(a.tick);
}

// RealDiag.recip = mc_div((1, 0..), U_ii) per row (_mcfast.py:390-402)
template <int K>
__global__ void recip_mc_kernel(int n, const int *dp, const double *lu, double *rcp) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double one[K], u[K], r[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      one[c] = c == 0 ? 1.0 : 0.0;
      u[c] = lu[(size_t)dp[i] * K + c];
    }
    div<K>(one, u, r);
#pragma unroll
    for (int c = 0; c < K; ++c) rcp[(size_t)i * K + c] = r[c];
  }
}

template <int K>
__global__ void __launch_bounds__(256) sweep_mc_kernel(SweepMcArgs a) {
  if (a.done && *a.done) return;
  const int lane = threadIdx.x & 31;
  const int n = a.n;
  const long long ld = a.ld;
  for (;;) {
    const int base = mc_grab(a.tick);
    if (base >= 2 * n) break;
    const int t = base + lane;
    if (t < n) {  // _sweep_forward ilu.py:322-331
      const int i = t;
      double acc[K];
#pragma unroll
      for (int c = 0; c < K; ++c) acc[c] = a.in[c * ld + i];
      for (int p = a.rp[i]; p < a.dp[i]; ++p) {
        double y[K], l[K], r[K];
        poll_mc<K>(a.y, ld, a.ci[p], y);
#pragma unroll
        for (int c = 0; c < K; ++c) l[c] = a.lu[(size_t)p * K + c];
        fmulsub<K>(acc, l, y, r);
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = r[c];
      }
      pub_mc<K>(a.y, ld, i, acc);
    } else if (t < 2 * n) {  // _sweep_backward ilu.py:334-343
      const int i = 2 * n - 1 - t;
      double acc[K];
      poll_mc<K>(a.y, ld, i, acc);
      for (int p = a.dp[i] + 1; p < a.rp[i + 1]; ++p) {
        double z[K], u[K], r[K];
        poll_mc<K>(a.z, ld, a.ci[p], z);
#pragma unroll
        for (int c = 0; c < K; ++c) u[c] = a.lu[(size_t)p * K + c];
        fmulsub<K>(acc, u, z, r);
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = r[c];
      }
      double rc[K], q[K];
#pragma unroll
      for (int c = 0; c < K; ++c) rc[c] = a.rcp[(size_t)i * K + c];
      fmul<K>(acc, rc, q);  // RealDiag.solve
      bool fin = true;
#pragma unroll
      for (int c = 0; c < K; ++c) fin = fin && isfin(q[c]);
      if (!fin) atomicOr(a.err, 1);
      pub_mc<K>(a.z, ld, i, q);
    }
  }
  mc_exit(a.tick);
}

// (LU)^-T at working precision, real (ilu.py:346-371, ilu0_apply_adjoint
// :423-433): U^T forward in gather form -- row c folds the scatter
// contributions of rows j < c in ascending j, then RealDiag.solve; L^T
// backward -- row c folds rows j > c in descending j, no division.
template <int K>
__global__ void __launch_bounds__(256) sweep_mc_adj_kernel(SweepMcArgs a) {
  if (a.done && *a.done) return;
  const int lane = threadIdx.x & 31;
  const int n = a.n;
  const long long ld = a.ld;
  for (;;) {
    const int base = mc_grab(a.tick);
    if (base >= 2 * n) break;
    const int t = base + lane;
    if (t < n) {
      const int c = t;
      double acc[K];
#pragma unroll
      for (int q = 0; q < K; ++q) acc[q] = a.in[q * ld + c];
      for (int p = a.ut_rp[c]; p < a.ut_rp[c + 1]; ++p) {
        double y[K], u[K], r[K];
        poll_mc<K>(a.y, ld, a.ut_ci[p], y);
        const long long e = a.ut_perm[p];
#pragma unroll
        for (int q = 0; q < K; ++q) u[q] = a.lu[e * K + q];
        fmulsub<K>(acc, u, y, r);
#pragma unroll
        for (int q = 0; q < K; ++q) acc[q] = r[q];
      }
      double rc[K], o[K];
#pragma unroll
      for (int q = 0; q < K; ++q) rc[q] = a.rcp[(size_t)c * K + q];
      fmul<K>(acc, rc, o);
      pub_mc<K>(a.y, ld, c, o);
    } else if (t < 2 * n) {
      const int c = 2 * n - 1 - t;
      double acc[K];
      poll_mc<K>(a.y, ld, c, acc);
      for (int p = a.lt_rp[c]; p < a.lt_rp[c + 1]; ++p) {
        double z[K], l[K], r[K];
        poll_mc<K>(a.z, ld, a.lt_ci[p], z);
        const long long e = a.lt_perm[p];
#pragma unroll
        for (int q = 0; q < K; ++q) l[q] = a.lu[e * K + q];
        fmulsub<K>(acc, l, z, r);
#pragma unroll
        for (int q = 0; q < K; ++q) acc[q] = r[q];
      }
      bool fin = true;
#pragma unroll
      for (int q = 0; q < K; ++q) fin = fin && isfin(acc[q]);
      if (!fin) atomicOr(a.err, 1);
      pub_mc<K>(a.z, ld, c, acc);
    }
  }
  mc_exit(a.tick);
}

template <int K>
__global__ void reset_mc_kernel(double *y, double *z, int n, const int *done) {
  if (done && *done) return;
  const double s = sent_val();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    y[i] = s;
    z[i] = s;
  }
}

}  // namespace

void launch_factor_mc(const FactorMcArgs &a, int k, cudaStream_t st) {
  ++tl_launches;
  long long warps = (a.n + 31) / 32;
  long long blocks = (warps + 7) / 8;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 6) blocks = 148 * 6;
  if (k == 2) factor_mc_kernel<2><<<(int)blocks, 256, 0, st>>>(a);
  if (k == 3) factor_mc_kernel<3><<<(int)blocks, 256, 0, st>>>(a);
  if (k == 4) factor_mc_kernel<4><<<(int)blocks, 256, 0, st>>>(a);
}

void launch_recip_mc(int n, const int *dp, const double *lu, double *rcp, int k,
                     cudaStream_t st) {
  if (n <= 0) return;
  ++tl_launches;
  const int g = (n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8;
  if (k == 2) recip_mc_kernel<2><<<g, 256, 0, st>>>(n, dp, lu, rcp);
  if (k == 3) recip_mc_kernel<3><<<g, 256, 0, st>>>(n, dp, lu, rcp);
  if (k == 4) recip_mc_kernel<4><<<g, 256, 0, st>>>(n, dp, lu, rcp);
}

void launch_sweep_mc(const SweepMcArgs &a, int k, cudaStream_t st) {
  const int g = (a.n + 255) / 256 < 148 * 8 ? ((a.n + 255) / 256 > 0 ? (a.n + 255) / 256 : 1)
                                              : 148 * 8;
  tl_launches += 2;
  if (k == 2) reset_mc_kernel<2><<<g, 256, 0, st>>>(a.y, a.z, a.n, a.done);
  if (k == 3) reset_mc_kernel<3><<<g, 256, 0, st>>>(a.y, a.z, a.n, a.done);
  if (k == 4) reset_mc_kernel<4><<<g, 256, 0, st>>>(a.y, a.z, a.n, a.done);
  long long warps = (2LL * a.n + 31) / 32;
  long long blocks = (warps + 7) / 8;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 6) blocks = 148 * 6;
  if (a.adjoint) {
    if (k == 2) sweep_mc_adj_kernel<2><<<(int)blocks, 256, 0, st>>>(a);
    if (k == 3) sweep_mc_adj_kernel<3><<<(int)blocks, 256, 0, st>>>(a);
    if (k == 4) sweep_mc_adj_kernel<4><<<(int)blocks, 256, 0, st>>>(a);
    return;
  }
  if (k == 2) sweep_mc_kernel<2><<<(int)blocks, 256, 0, st>>>(a);
  if (k == 3) sweep_mc_kernel<3><<<(int)blocks, 256, 0, st>>>(a);
  if (k == 4) sweep_mc_kernel<4><<<(int)blocks, 256, 0, st>>>(a);
}

}  // namespace mpk
