// ilu_mc.cu -- working-precision ILU(0) (precond 'ilu0'):
// factorization in K-component arithmetic and its forward / backward
// sweeps on K-component vectors, real and complex fields.
//
// Reference: ilu.py:178-276 (_factorize_tuples with k > 1: lik = mc_div,
// a_ij = _mcfast.rmulsubK(a_ij, lik, u_kj)), ilu.py:322-343 (sweeps:
// acc = rmulsubK(acc, l_ij, y_j) ascending j; backward acc / U_ii through
// _mcfast.RealDiag = rmulK(acc, mc_div(1, U_ii))), ilu.py:374-420.
// Scheduling is the sync-free ticket scheme of ilu.cu (one row per thread,
// rows claimed in dependency-compatible order, a row waits only on rows
// with smaller tickets).  Every component plane of the outputs starts as
// signalling-NaN sentinels; a value is complete when none of its
// components is a sentinel (each changes exactly once per sweep).
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

// K-component value j of a planar vector (stride ld), published by another
// row: EVERY component plane is sentinel-reset before the sweep and each
// component changes once (sentinel -> final value), so a value is complete
// when no component still carries the sentinel -- no fence on either side.
template <int W>
__device__ __forceinline__ bool any_sent(const double (&o)[W]) {
  bool b = false;
#pragma unroll
  for (int c = 0; c < W; ++c) b |= is_sent(o[c]);
  return b;
}
template <int W>
__device__ __forceinline__ void load_mc(const double *v, long long ld, int j, double (&o)[W]) {
#pragma unroll
  for (int c = 0; c < W; ++c) o[c] = ldr(v + c * ld + j);
}
template <int K>
__device__ __forceinline__ void poll_mc(const double *v, long long ld, int j,
                                        double (&o)[K]) {
  load_mc<K>(v, ld, j, o);
  while (any_sent<K>(o)) {
    __nanosleep(32);
    load_mc<K>(v, ld, j, o);
  }
}
template <int K>
__device__ __forceinline__ void pub_mc(double *v, long long ld, int j,
                                       const double (&x)[K]) {
#pragma unroll
  for (int c = 0; c < K; ++c) str(v + c * ld + j, unsent(x[c]));
}

// Up to kMcBatch published values at cols[0..m) requested together (all
// components); the caller consumes them in order through wait_mc, so the
// later requests are in flight while the earlier products are computed.
constexpr int kMcBatch = 4;
template <int W>
__device__ __forceinline__ void gather_mc(const double *v, long long ld, const int *cols,
                                          int m, double (&o)[kMcBatch][W]) {
#pragma unroll
  for (int b = 0; b < kMcBatch; ++b)
    if (b < m) load_mc<W>(v, ld, cols[b], o[b]);
}
template <int W>
__device__ __forceinline__ void wait_mc(const double *v, long long ld, int col,
                                        double (&o)[W]) {
  while (any_sent<W>(o)) {
    __nanosleep(32);
    load_mc<W>(v, ld, col, o);
  }
}

// value helpers on flat (re..., im...) arrays of W = K or 2K components
template <int K, bool CX>
__device__ __forceinline__ void mc_mulsub(const double *a, const double *b,
                                          const double *c, double *o) {
  if constexpr (CX) {
    double ar[K], ai[K], br[K], bi[K], cr[K], ci[K], orr[K], oi[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      ar[q] = a[q]; ai[q] = a[K + q]; br[q] = b[q]; bi[q] = b[K + q];
      cr[q] = c[q]; ci[q] = c[K + q];
    }
    fcmulsub<K>(ar, ai, br, bi, cr, ci, orr, oi);  // _mcfast.cmulsubK
#pragma unroll
    for (int q = 0; q < K; ++q) {
      o[q] = orr[q];
      o[K + q] = oi[q];
    }
  } else {
    double x[K], y[K], z[K], r[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      x[q] = a[q]; y[q] = b[q]; z[q] = c[q];
    }
    fmulsub<K>(x, y, z, r);  // _mcfast.rmulsubK
#pragma unroll
    for (int q = 0; q < K; ++q) o[q] = r[q];
  }
}

template <int K, bool CX>
__device__ void factor_mc_row(const FactorMcArgs &a, int i) {
  constexpr int W = CX ? 2 * K : K;
  const int lo = a.rp[i], hi = a.rp[i + 1], d = a.dp[i];
  double *lu = a.lu;
  for (int t = lo; t < d; ++t) {
    const int kc = a.ci[t];
    while (ldri(&a.rowflag[kc]) == 0) __nanosleep(32);
    __threadfence();
    const int uk = a.dp[kc], kend = a.rp[kc + 1];
    double at[W], ukk[W], l[W];
#pragma unroll
    for (int c = 0; c < W; ++c) {
      at[c] = __ldcg(&lu[(size_t)t * W + c]);
      ukk[c] = __ldcg(&lu[(size_t)uk * W + c]);
    }
    if constexpr (CX) {  // cx_div (_mccore.py:328-347), flat pair
      double xr[K], xi[K], yr[K], yi[K], qr[K], qi[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        xr[q] = at[q]; xi[q] = at[K + q]; yr[q] = ukk[q]; yi[q] = ukk[K + q];
      }
      cdiv<K>(xr, xi, yr, yi, qr, qi);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        l[q] = qr[q];
        l[K + q] = qi[q];
      }
    } else {
      double x[K], y[K], q2[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        x[q] = at[q];
        y[q] = ukk[q];
      }
      div<K>(x, y, q2);  // mc_div (_mccore.py:222-237)
#pragma unroll
      for (int q = 0; q < K; ++q) l[q] = q2[q];
    }
#pragma unroll
    for (int c = 0; c < W; ++c) __stcg(&lu[(size_t)t * W + c], l[c]);
    int q = t + 1;
    for (int s = uk + 1; s < kend; ++s) {
      const int col = a.ci[s];
      while (q < hi && a.ci[q] < col) ++q;
      if (q < hi && a.ci[q] == col) {
        double v[W], u[W], r[W];
#pragma unroll
        for (int c = 0; c < W; ++c) {
          v[c] = __ldcg(&lu[(size_t)q * W + c]);
          u[c] = __ldcg(&lu[(size_t)s * W + c]);
        }
        mc_mulsub<K, CX>(v, l, u, r);  // mulsub(a_ij, lik, u_kj)
#pragma unroll
        for (int c = 0; c < W; ++c) __stcg(&lu[(size_t)q * W + c], r[c]);
      }
    }
  }
  bool zero = true, fin = true;
#pragma unroll
  for (int c = 0; c < W; ++c) zero = zero && __ldcg(&lu[(size_t)d * W + c]) == 0.0;
  for (int p = lo; p < hi; ++p)
    for (int c = 0; c < W; ++c) fin = fin && isfin(__ldcg(&lu[(size_t)p * W + c]));
  if (zero) atomicMin(a.bad_row, i);
  if (!fin) atomicOr(a.nonfinite, 1);
  __threadfence();
  atomicExch(&a.rowflag[i], 1);
}

template <int K, bool CX>
__global__ void __launch_bounds__(256) factor_mc_kernel(FactorMcArgs a) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const int base = mc_grab(a.tick);
    if (base >= a.n) break;
    const int t = base + lane;
    if (t < a.n) factor_mc_row<K, CX>(a, a.ord ? a.ord[t] : t);
  }
  mc_exit(a.tick);
}

// Diagonal solvers of the backward sweeps, per row (_mcfast.py:386-439):
// real RealDiag.recip = mc_div(1, U_ii) [K]; complex ComplexDiag (Smith):
// {t [K], recip [K], swapped} = 2K+1 values, for the plain sweep and, at
// offset n*(2K+1), for the adjoint sweep (built from conj(U_ii)).
template <int K>
__device__ void complex_diag(const double (&dr)[K], const double (&di)[K], double *o) {
  double one[K], t[K], den[K], tmp[K], rc[K];
#pragma unroll
  for (int q = 0; q < K; ++q) one[q] = q == 0 ? 1.0 : 0.0;
  const bool swapped = !(fabs(dr[0]) >= fabs(di[0]));
  if (!swapped) {
    div<K>(di, dr, t);
    mul<K>(di, t, tmp);
    add<K>(dr, tmp, den);
  } else {
    div<K>(dr, di, t);
    mul<K>(dr, t, tmp);
    add<K>(tmp, di, den);
  }
  div<K>(one, den, rc);
#pragma unroll
  for (int q = 0; q < K; ++q) {
    o[q] = t[q];
    o[K + q] = rc[q];
  }
  o[2 * K] = swapped ? 1.0 : 0.0;
}

template <int K, bool CX>
__global__ void recip_mc_kernel(int n, const int *dp, const double *lu, double *rcp) {
  constexpr int W = CX ? 2 * K : K;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if constexpr (CX) {
      double dr[K], di[K], nd[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        dr[q] = lu[(size_t)dp[i] * W + q];
        di[q] = lu[(size_t)dp[i] * W + K + q];
        nd[q] = -di[q];
      }
      complex_diag<K>(dr, di, rcp + (size_t)i * (2 * K + 1));
      complex_diag<K>(dr, nd, rcp + ((size_t)n + i) * (2 * K + 1));
    } else {
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
}

// acc / U_ii through the precomputed diagonal solver (flat W components)
template <int K, bool CX>
__device__ __forceinline__ void diag_solve(const double *acc, const double *dg, double *o) {
  if constexpr (CX) {  // ComplexDiag.solve
    double xr[K], xi[K], nxr[K], nxi[K], t[K], rc[K], nr[K], ni[K], qr[K], qi[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      xr[q] = acc[q]; xi[q] = acc[K + q]; nxr[q] = -xr[q]; nxi[q] = -xi[q];
      t[q] = dg[q]; rc[q] = dg[K + q];
    }
    if (dg[2 * K] == 0.0) {
      fmulsub<K>(xr, nxi, t, nr);   // xr + xi*t
      fmulsub<K>(xi, xr, t, ni);    // xi - xr*t
    } else {
      fmulsub<K>(xi, nxr, t, nr);   // xi + xr*t
      fmulsub<K>(nxr, nxi, t, ni);  // xi*t - xr
    }
    fmul<K>(nr, rc, qr);
    fmul<K>(ni, rc, qi);
#pragma unroll
    for (int q = 0; q < K; ++q) {
      o[q] = qr[q];
      o[K + q] = qi[q];
    }
  } else {  // RealDiag.solve
    double x[K], rc[K], q2[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      x[q] = acc[q];
      rc[q] = dg[q];
    }
    fmul<K>(x, rc, q2);
#pragma unroll
    for (int q = 0; q < K; ++q) o[q] = q2[q];
  }
}

template <int K, bool CX>
__global__ void __launch_bounds__(256) sweep_mc_kernel(SweepMcArgs a) {
  // _sweep_forward / _sweep_backward ilu.py:322-343 (flat W components;
  // planar vectors: component q at q*ld, complex = K real then K imag)
  constexpr int W = CX ? 2 * K : K;
  constexpr int DW = CX ? 2 * K + 1 : K;
  {  // stopped solve: skip, but count this warp out (ticket reset)
    int d = 0;
    if ((threadIdx.x & 31) == 0 && a.done) d = ldri(a.done);
    if (__shfl_sync(kFullM, d, 0)) {
      mc_exit(a.tick);
      return;
    }
  }
  const int lane = threadIdx.x & 31;
  const int n = a.n;
  const long long ld = a.ld;
  for (;;) {
    const int base = mc_grab(a.tick);
    if (base >= 2 * n) break;
    const int t = base + lane;
    if (t < n) {
      const int i = a.ord_f ? a.ord_f[t] : t;
      double acc[W];
#pragma unroll
      for (int c = 0; c < W; ++c) acc[c] = a.in[c * ld + i];
      for (int p0 = a.rp[i]; p0 < a.dp[i]; p0 += kMcBatch) {
        const int m = min(kMcBatch, a.dp[i] - p0);
        int cols[kMcBatch];
        double yv[kMcBatch][W];
#pragma unroll
        for (int b = 0; b < kMcBatch; ++b) cols[b] = b < m ? a.ci[p0 + b] : 0;
        gather_mc<W>(a.y, ld, cols, m, yv);
#pragma unroll
        for (int b = 0; b < kMcBatch; ++b)
          if (b < m) {
            double l[W], r[W];
#pragma unroll
            for (int c = 0; c < W; ++c) l[c] = a.lu[(size_t)(p0 + b) * W + c];
            wait_mc<W>(a.y, ld, cols[b], yv[b]);
            mc_mulsub<K, CX>(acc, l, yv[b], r);
#pragma unroll
            for (int c = 0; c < W; ++c) acc[c] = r[c];
          }
      }
      pub_mc<W>(a.y, ld, i, acc);
    } else if (t < 2 * n) {
      const int i = a.ord_b ? a.ord_b[t - n] : 2 * n - 1 - t;
      double acc[W];
      poll_mc<W>(a.y, ld, i, acc);
      for (int p0 = a.dp[i] + 1; p0 < a.rp[i + 1]; p0 += kMcBatch) {
        const int m = min(kMcBatch, a.rp[i + 1] - p0);
        int cols[kMcBatch];
        double zv[kMcBatch][W];
#pragma unroll
        for (int b = 0; b < kMcBatch; ++b) cols[b] = b < m ? a.ci[p0 + b] : 0;
        gather_mc<W>(a.z, ld, cols, m, zv);
#pragma unroll
        for (int b = 0; b < kMcBatch; ++b)
          if (b < m) {
            double u[W], r[W];
#pragma unroll
            for (int c = 0; c < W; ++c) u[c] = a.lu[(size_t)(p0 + b) * W + c];
            wait_mc<W>(a.z, ld, cols[b], zv[b]);
            mc_mulsub<K, CX>(acc, u, zv[b], r);
#pragma unroll
            for (int c = 0; c < W; ++c) acc[c] = r[c];
          }
      }
      double q[W];
      diag_solve<K, CX>(acc, a.rcp + (size_t)i * DW, q);
      bool fin = true;
#pragma unroll
      for (int c = 0; c < W; ++c) fin = fin && isfin(q[c]);
      if (!fin) atomicOr(a.err, 1);
      pub_mc<W>(a.z, ld, i, q);
    }
  }
  mc_exit(a.tick);
}

// (LU)^-H at working precision (ilu.py:346-371, ilu0_apply_adjoint
// :423-433): U^H forward in gather form -- row c folds the scatter
// contributions of rows j < c in ascending j with conjugated values, then
// the diagonal solver of conj(U_cc); L^H backward -- row c folds rows j > c
// in descending j, no division.
template <int K, bool CX>
__global__ void __launch_bounds__(256) sweep_mc_adj_kernel(SweepMcArgs a) {
  constexpr int W = CX ? 2 * K : K;
  constexpr int DW = CX ? 2 * K + 1 : K;
  {  // stopped solve: skip, but count this warp out (ticket reset)
    int d = 0;
    if ((threadIdx.x & 31) == 0 && a.done) d = ldri(a.done);
    if (__shfl_sync(kFullM, d, 0)) {
      mc_exit(a.tick);
      return;
    }
  }
  const int lane = threadIdx.x & 31;
  const int n = a.n;
  const long long ld = a.ld;
  const double *dg0 = a.rcp + (CX ? (size_t)n * DW : 0);
  for (;;) {
    const int base = mc_grab(a.tick);
    if (base >= 2 * n) break;
    const int t = base + lane;
    if (t < n) {
      const int c = a.ord_f ? a.ord_f[t] : t;
      double acc[W];
#pragma unroll
      for (int q = 0; q < W; ++q) acc[q] = a.in[q * ld + c];
      for (int p0 = a.ut_rp[c]; p0 < a.ut_rp[c + 1]; p0 += kMcBatch) {
        const int m = min(kMcBatch, a.ut_rp[c + 1] - p0);
        int cols[kMcBatch];
        double yv[kMcBatch][W];
#pragma unroll
        for (int b = 0; b < kMcBatch; ++b) cols[b] = b < m ? a.ut_ci[p0 + b] : 0;
        gather_mc<W>(a.y, ld, cols, m, yv);
#pragma unroll
        for (int b = 0; b < kMcBatch; ++b)
          if (b < m) {
            double u[W], r[W];
            const long long e = a.ut_perm[p0 + b];
#pragma unroll
            for (int q = 0; q < W; ++q) u[q] = (CX && q >= K) ? -a.lu[e * W + q] : a.lu[e * W + q];
            wait_mc<W>(a.y, ld, cols[b], yv[b]);
            mc_mulsub<K, CX>(acc, u, yv[b], r);
#pragma unroll
            for (int q = 0; q < W; ++q) acc[q] = r[q];
          }
      }
      double o[W];
      diag_solve<K, CX>(acc, dg0 + (size_t)c * DW, o);
      pub_mc<W>(a.y, ld, c, o);
    } else if (t < 2 * n) {
      const int c = a.ord_b ? a.ord_b[t - n] : 2 * n - 1 - t;
      double acc[W];
      poll_mc<W>(a.y, ld, c, acc);
      for (int p0 = a.lt_rp[c]; p0 < a.lt_rp[c + 1]; p0 += kMcBatch) {
        const int m = min(kMcBatch, a.lt_rp[c + 1] - p0);
        int cols[kMcBatch];
        double zv[kMcBatch][W];
#pragma unroll
        for (int b = 0; b < kMcBatch; ++b) cols[b] = b < m ? a.lt_ci[p0 + b] : 0;
        gather_mc<W>(a.z, ld, cols, m, zv);
#pragma unroll
        for (int b = 0; b < kMcBatch; ++b)
          if (b < m) {
            double l[W], r[W];
            const long long e = a.lt_perm[p0 + b];
#pragma unroll
            for (int q = 0; q < W; ++q) l[q] = (CX && q >= K) ? -a.lu[e * W + q] : a.lu[e * W + q];
            wait_mc<W>(a.z, ld, cols[b], zv[b]);
            mc_mulsub<K, CX>(acc, l, zv[b], r);
#pragma unroll
            for (int q = 0; q < W; ++q) acc[q] = r[q];
          }
      }
      bool fin = true;
#pragma unroll
      for (int q = 0; q < W; ++q) fin = fin && isfin(acc[q]);
      if (!fin) atomicOr(a.err, 1);
      pub_mc<W>(a.z, ld, c, acc);
    }
  }
  mc_exit(a.tick);
}

__global__ void reset_mc_kernel(double *y, double *z, int n, long long ld, int w,
                                const int *done) {
  if (done && *done) return;
  const double s = sent_val();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int c = 0; c < w; ++c) {
      y[c * ld + i] = s;
      z[c * ld + i] = s;
    }
}

}  // namespace

// Ticket grids of the K-component factor / sweeps: one 8-warp CTA per SM
// (≈ 38 k rows in flight) is enough to keep every level of a stencil busy;
// more resident warps only add sentinel polls to L2 (cfg4 apply 1.6x slower
// at 6 CTAs per SM).  MPK_MC_BLOCKS overrides.
static int mc_grid_cap() {
  static const int cap = [] {
    const char *e = getenv("MPK_MC_BLOCKS");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : sm_count();
  }();
  return cap;
}

void launch_factor_mc(const FactorMcArgs &a, int k, cudaStream_t st) {
  ++tl_launches;
  long long warps = (a.n + 31) / 32;
  long long blocks = (warps + 7) / 8;
  if (blocks < 1) blocks = 1;
  if (blocks > mc_grid_cap()) blocks = mc_grid_cap();
  const int g = (int)blocks;
  const bool cx = a.cx != 0;
  if (k == 2 && !cx) factor_mc_kernel<2, false><<<g, 256, 0, st>>>(a);
  if (k == 3 && !cx) factor_mc_kernel<3, false><<<g, 256, 0, st>>>(a);
  if (k == 4 && !cx) factor_mc_kernel<4, false><<<g, 256, 0, st>>>(a);
  if (k == 2 && cx) factor_mc_kernel<2, true><<<g, 256, 0, st>>>(a);
  if (k == 3 && cx) factor_mc_kernel<3, true><<<g, 256, 0, st>>>(a);
  if (k == 4 && cx) factor_mc_kernel<4, true><<<g, 256, 0, st>>>(a);
}

void launch_recip_mc(int n, const int *dp, const double *lu, double *rcp, int k, bool cx,
                     cudaStream_t st) {
  if (n <= 0) return;
  ++tl_launches;
  const int g = (n + 255) / 256 < sm_count() * 8 ? (n + 255) / 256 : sm_count() * 8;
  if (k == 2 && !cx) recip_mc_kernel<2, false><<<g, 256, 0, st>>>(n, dp, lu, rcp);
  if (k == 3 && !cx) recip_mc_kernel<3, false><<<g, 256, 0, st>>>(n, dp, lu, rcp);
  if (k == 4 && !cx) recip_mc_kernel<4, false><<<g, 256, 0, st>>>(n, dp, lu, rcp);
  if (k == 2 && cx) recip_mc_kernel<2, true><<<g, 256, 0, st>>>(n, dp, lu, rcp);
  if (k == 3 && cx) recip_mc_kernel<3, true><<<g, 256, 0, st>>>(n, dp, lu, rcp);
  if (k == 4 && cx) recip_mc_kernel<4, true><<<g, 256, 0, st>>>(n, dp, lu, rcp);
}

void launch_sweep_mc(const SweepMcArgs &a, int k, cudaStream_t st) {
  const int nb = (a.n + 255) / 256 > 0 ? (a.n + 255) / 256 : 1;
  const int g = nb < sm_count() * 8 ? nb : sm_count() * 8;
  tl_launches += 2;
  reset_mc_kernel<<<g, 256, 0, st>>>(a.y, a.z, a.n, a.ld, (a.cx ? 2 : 1) * k, a.done);
  long long warps = (2LL * a.n + 31) / 32;
  long long blocks = (warps + 7) / 8;
  if (blocks < 1) blocks = 1;
  if (blocks > mc_grid_cap()) blocks = mc_grid_cap();
  const int gb = (int)blocks;
  const bool cx = a.cx != 0;
  if (a.adjoint) {
    if (k == 2 && !cx) sweep_mc_adj_kernel<2, false><<<gb, 256, 0, st>>>(a);
    if (k == 3 && !cx) sweep_mc_adj_kernel<3, false><<<gb, 256, 0, st>>>(a);
    if (k == 4 && !cx) sweep_mc_adj_kernel<4, false><<<gb, 256, 0, st>>>(a);
    if (k == 2 && cx) sweep_mc_adj_kernel<2, true><<<gb, 256, 0, st>>>(a);
    if (k == 3 && cx) sweep_mc_adj_kernel<3, true><<<gb, 256, 0, st>>>(a);
    if (k == 4 && cx) sweep_mc_adj_kernel<4, true><<<gb, 256, 0, st>>>(a);
    return;
  }
  if (k == 2 && !cx) sweep_mc_kernel<2, false><<<gb, 256, 0, st>>>(a);
  if (k == 3 && !cx) sweep_mc_kernel<3, false><<<gb, 256, 0, st>>>(a);
  if (k == 4 && !cx) sweep_mc_kernel<4, false><<<gb, 256, 0, st>>>(a);
  if (k == 2 && cx) sweep_mc_kernel<2, true><<<gb, 256, 0, st>>>(a);
  if (k == 3 && cx) sweep_mc_kernel<3, true><<<gb, 256, 0, st>>>(a);
  if (k == 4 && cx) sweep_mc_kernel<4, true><<<gb, 256, 0, st>>>(a);
}

}  // namespace mpk
