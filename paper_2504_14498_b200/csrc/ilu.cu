// ilu.cu -- sync-free binary64 ILU(0) factorization and sweeps (see ilu.cuh)
#include <climits>

#include "ilu.cuh"

namespace mpk {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int ld_volatile_i(const int *p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ int grab_ticket(int *tick) {
  int base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(tick, 32);
  return __shfl_sync(kFull, base, 0);
}

// Last warp out resets the ticket so the next launch (or graph replay)
// starts from zero.
__device__ __forceinline__ void exit_protocol(int *tick) {
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

// ---------------------------------------------------------------------
// factorization: _factorize_tuples ilu.py:234-252 (k = 1), one row per
// thread, ascending L columns, merge-walk of row kc's upper part.
// ---------------------------------------------------------------------
template <bool CX>
__device__ void factor_row(const FactorArgs &a, int i) {
  const int lo = a.rp[i], hi = a.rp[i + 1], d = a.dp[i];
  double2 *lu2 = reinterpret_cast<double2 *>(a.lu);
  for (int t = lo; t < d; ++t) {
    const int kc = a.ci[t];
    while (ld_volatile_i(&a.rowflag[kc]) == 0) __nanosleep(32);
    __threadfence();
    const int uk = a.dp[kc];
    const int kend = a.rp[kc + 1];
    if constexpr (!CX) {
      const double l = ddiv(__ldcg(&a.lu[t]), __ldcg(&a.lu[uk]));
      __stcg(&a.lu[t], l);
      int q = t + 1;
      for (int s = uk + 1; s < kend; ++s) {
        const int col = a.ci[s];
        while (q < hi && a.ci[q] < col) ++q;
        if (q < hi && a.ci[q] == col) {
          __stcg(&a.lu[q], dsub(__ldcg(&a.lu[q]), dmul(l, __ldcg(&a.lu[s]))));
        }
      }
    } else {
      const double2 at = __ldcg(&lu2[t]);
      const double2 ukk = __ldcg(&lu2[uk]);
      double lr, li;
      py_cdiv(at.x, at.y, ukk.x, ukk.y, lr, li);
      __stcg(&lu2[t], make_double2(lr, li));
      int q = t + 1;
      for (int s = uk + 1; s < kend; ++s) {
        const int col = a.ci[s];
        while (q < hi && a.ci[q] < col) ++q;
        if (q < hi && a.ci[q] == col) {
          const double2 u = __ldcg(&lu2[s]);
          double pr, pi;
          py_cmul(lr, li, u.x, u.y, pr, pi);
          const double2 v = __ldcg(&lu2[q]);
          __stcg(&lu2[q], make_double2(dsub(v.x, pr), dsub(v.y, pi)));
        }
      }
    }
  }
  bool zero, fin = true;
  if constexpr (!CX) {
    zero = __ldcg(&a.lu[d]) == 0.0;
    for (int p = lo; p < hi; ++p) fin = fin && isfin(__ldcg(&a.lu[p]));
  } else {
    const double2 v = __ldcg(&lu2[d]);
    zero = (v.x == 0.0) && (v.y == 0.0);
    for (int p = lo; p < hi; ++p) {
      const double2 w = __ldcg(&lu2[p]);
      fin = fin && isfin(w.x) && isfin(w.y);
    }
  }
  if (zero) atomicMin(a.bad_row, i);
  if (!fin) atomicOr(a.nonfinite, 1);
  __threadfence();
  atomicExch(&a.rowflag[i], 1);
}

template <bool CX>
__global__ void __launch_bounds__(kBlock) factor_kernel(FactorArgs a) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const int base = grab_ticket(a.tick);
    if (base >= a.n) break;
    const int i = base + lane;
    if (i < a.n) factor_row<CX>(a, i);
  }
  exit_protocol(a.tick);
}

// ---------------------------------------------------------------------
// sweeps
// ---------------------------------------------------------------------
template <bool CX>
__device__ __forceinline__ void load_in(const SweepArgs &a, int i, double &r,
                                        double &m) {
  if constexpr (CX) {
    // numpy demotion re + 1j*im (sparse.py:392)
    const double re0 = a.in_re[i], im0 = a.in_im[i];
    r = dadd(re0, dsub(dmul(0.0, im0), 0.0));
    m = dadd(0.0, im0);
  } else {
    r = a.in_re[i];
    m = 0.0;
  }
}

// acc -= l * v   (real: a - l*u; complex: CPython a - l*u, conj optional)
template <bool CX, bool CONJ>
__device__ __forceinline__ void mulsub(double &ar, double &ai, double lr,
                                       double li, double vr, double vi) {
  if constexpr (CX) {
    double pr, pi;
    py_cmul(lr, CONJ ? -li : li, vr, vi, pr, pi);
    ar = dsub(ar, pr);
    ai = dsub(ai, pi);
  } else {
    ar = dsub(ar, dmul(lr, vr));
  }
}

template <bool CX>
__device__ __forceinline__ void ldval(const double *v, int p, double &r,
                                      double &m) {
  if constexpr (CX) {
    const double2 w = reinterpret_cast<const double2 *>(v)[p];
    r = w.x;
    m = w.y;
  } else {
    r = v[p];
    m = 0.0;
  }
}

template <bool CX>
__device__ __forceinline__ void pollv(const double *buf, int j, double &r,
                                      double &m) {
  if constexpr (CX) {
    const double2 w = poll2(reinterpret_cast<const double2 *>(buf) + j);
    r = w.x;
    m = w.y;
  } else {
    r = poll1(buf + j);
    m = 0.0;
  }
}

template <bool CX>
__device__ __forceinline__ void publish(double *buf, int j, double r,
                                        double m) {
  if constexpr (CX) {
    st_volatile2(reinterpret_cast<double2 *>(buf) + j,
                 make_double2(unsent(r), unsent(m)));
  } else {
    st_volatile(buf + j, unsent(r));
  }
}

// _sweep_forward ilu.py:322-331
template <bool CX>
__device__ void fwd_row(const SweepArgs &a, int i) {
  double ar, ai;
  load_in<CX>(a, i, ar, ai);
  const int lo = a.rp[i], d = a.dp[i];
  for (int p = lo; p < d; ++p) {
    const int j = a.ci[p];
    double lr, li, yr, yi;
    ldval<CX>(a.lu, p, lr, li);
    pollv<CX>(a.y, j, yr, yi);
    mulsub<CX, false>(ar, ai, lr, li, yr, yi);
  }
  publish<CX>(a.y, i, ar, ai);
}

// _sweep_backward ilu.py:334-343
template <bool CX>
__device__ void bwd_row(const SweepArgs &a, int i) {
  double ar, ai;
  pollv<CX>(a.y, i, ar, ai);
  const int d = a.dp[i], hi = a.rp[i + 1];
  for (int p = d + 1; p < hi; ++p) {
    const int j = a.ci[p];
    double ur, ui, zr, zi;
    ldval<CX>(a.lu, p, ur, ui);
    pollv<CX>(a.z, j, zr, zi);
    mulsub<CX, false>(ar, ai, ur, ui, zr, zi);
  }
  double dr, di, qr, qi;
  ldval<CX>(a.lu, d, dr, di);
  if constexpr (CX) {
    py_cdiv(ar, ai, dr, di, qr, qi);
  } else {
    qr = ddiv(ar, dr);
    qi = 0.0;
  }
  if (!isfin(qr) || !isfin(qi)) atomicOr(a.err, 1);
  publish<CX>(a.z, i, qr, qi);
}

// _sweep_forward_adjoint ilu.py:346-357 in gather form: U^H is lower
// triangular; the scatter of row j into acc[c] runs in ascending j, so the
// gather over column c of U visits rows in ascending order.
template <bool CX>
__device__ void fwd_row_adj(const SweepArgs &a, int c) {
  double ar, ai;
  load_in<CX>(a, c, ar, ai);
  const int lo = a.ut_rp[c], hi = a.ut_rp[c + 1];
  for (int q = lo; q < hi; ++q) {
    const int j = a.ut_ci[q];
    double ur, ui, yr, yi;
    ldval<CX>(a.ut_val, q, ur, ui);
    pollv<CX>(a.y, j, yr, yi);
    mulsub<CX, true>(ar, ai, ur, ui, yr, yi);
  }
  double dr, di, qr, qi;
  ldval<CX>(a.lu, a.dp[c], dr, di);
  if constexpr (CX) {
    py_cdiv(ar, ai, dr, -di, qr, qi);
  } else {
    qr = ddiv(ar, dr);
    qi = 0.0;
  }
  publish<CX>(a.y, c, qr, qi);
}

// _sweep_backward_adjoint ilu.py:360-371: L^H unit upper; rows j scatter in
// DESCENDING order, so the gather over column c of L visits rows j > c in
// descending order (lt_ci is stored that way).
template <bool CX>
__device__ void bwd_row_adj(const SweepArgs &a, int c) {
  double ar, ai;
  pollv<CX>(a.y, c, ar, ai);
  const int lo = a.lt_rp[c], hi = a.lt_rp[c + 1];
  for (int q = lo; q < hi; ++q) {
    const int j = a.lt_ci[q];
    double lr, li, zr, zi;
    ldval<CX>(a.lt_val, q, lr, li);
    pollv<CX>(a.z, j, zr, zi);
    mulsub<CX, true>(ar, ai, lr, li, zr, zi);
  }
  if (!isfin(ar) || !isfin(ai)) atomicOr(a.err, 1);
  publish<CX>(a.z, c, ar, ai);
}

template <bool CX, bool ADJ>
__global__ void __launch_bounds__(kBlock) sweep_kernel(SweepArgs a) {
  if (a.done && *a.done) return;
  const int lane = threadIdx.x & 31;
  const int n = a.n;
  for (;;) {
    const int base = grab_ticket(a.tick);
    if (base >= 2 * n) break;
    const int t = base + lane;
    if (t < n) {
      if constexpr (ADJ)
        fwd_row_adj<CX>(a, t);
      else
        fwd_row<CX>(a, t);
    } else if (t < 2 * n) {
      if constexpr (ADJ)
        bwd_row_adj<CX>(a, 2 * n - 1 - t);
      else
        bwd_row<CX>(a, 2 * n - 1 - t);
    }
  }
  exit_protocol(a.tick);
}

template <bool CX>
__global__ void sweep_reset_kernel(double *y, double *z, int n,
                                   const int *done) {
  if (done && *done) return;
  const double s = sent_val();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    if constexpr (CX) {
      reinterpret_cast<double2 *>(y)[i] = make_double2(s, s);
      reinterpret_cast<double2 *>(z)[i] = make_double2(s, s);
    } else {
      y[i] = s;
      z[i] = s;
    }
  }
}

int sweep_grid(int n) {
  // enough resident warps to expose the DAG's width; extra warps idle out
  long long warps = (2LL * n + 31) / 32;
  long long blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 6) blocks = 148 * 6;
  return (int)blocks;
}

}  // namespace

void launch_sweep(const SweepArgs &a, bool cx, bool adjoint,
                  cudaStream_t st) {
  const int g = sweep_grid(a.n);
  if (!cx && !adjoint) sweep_kernel<false, false><<<g, kBlock, 0, st>>>(a);
  if (!cx && adjoint) sweep_kernel<false, true><<<g, kBlock, 0, st>>>(a);
  if (cx && !adjoint) sweep_kernel<true, false><<<g, kBlock, 0, st>>>(a);
  if (cx && adjoint) sweep_kernel<true, true><<<g, kBlock, 0, st>>>(a);
}

void launch_sweep_reset(double *y, double *z, int n, bool cx,
                        const int *done, cudaStream_t st) {
  const int g = grid_for(n);
  if (cx)
    sweep_reset_kernel<true><<<g, kBlock, 0, st>>>(y, z, n, done);
  else
    sweep_reset_kernel<false><<<g, kBlock, 0, st>>>(y, z, n, done);
}

void launch_factor(const FactorArgs &a, bool cx, cudaStream_t st) {
  long long warps = (a.n + 31) / 32;
  long long blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 6) blocks = 148 * 6;
  if (cx)
    factor_kernel<true><<<(int)blocks, kBlock, 0, st>>>(a);
  else
    factor_kernel<false><<<(int)blocks, kBlock, 0, st>>>(a);
}

}  // namespace mpk
