// units.cu -- single-operation device kernels behind the C-ABI unit entry
// points (spmv, hdot, norm2, axpy, element-wise MC ops, layout transposes).
// They reuse the solver's row framework so the parity tests exercise the
// exact code the solver runs.
#include <cstdio>

#include "rows.cuh"

namespace mpk {

template <int K, bool CX>
static void spmv_typed(DMat &A, bool adjoint, bool xf, const double *d_x,
                       double *d_y, cudaStream_t st) {
  const DA a{A.n, A.rp, A.ci, A.val, A.at_rp, A.at_ci, A.at_val};
  const long long L = plane_ld(A.n);
  const MV<K, CX> Y{d_y, L};
  if (xf && !adjoint)
    rows<K, CX, 0, 0>(A.n, nullptr, nullptr, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double yr[K], yi[K];
                        spmv_row<K, CX, true, false>(a, (int)i, d_x, L, yr, yi);
                        Y.store(i, yr, yi);
                      });
  else if (xf && adjoint)
    rows<K, CX, 0, 0>(A.n, nullptr, nullptr, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double yr[K], yi[K];
                        spmv_row<K, CX, true, true>(a, (int)i, d_x, L, yr, yi);
                        Y.store(i, yr, yi);
                      });
  else if (!adjoint)
    rows<K, CX, 0, 0>(A.n, nullptr, nullptr, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double yr[K], yi[K];
                        spmv_row<K, CX, false, false>(a, (int)i, d_x, L, yr, yi);
                        Y.store(i, yr, yi);
                      });
  else
    rows<K, CX, 0, 0>(A.n, nullptr, nullptr, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double yr[K], yi[K];
                        spmv_row<K, CX, false, true>(a, (int)i, d_x, L, yr, yi);
                        Y.store(i, yr, yi);
                      });
}

int unit_spmv(DMat &A, int k, bool adjoint, bool x_is_f, const double *d_x,
              double *d_y, cudaStream_t st) {
  if (adjoint) ensure_adjoint(A, st);
#define DISPATCH(KK)                                              \
  if (k == KK) {                                                  \
    if (A.cx)                                                     \
      spmv_typed<KK, true>(A, adjoint, x_is_f, d_x, d_y, st);     \
    else                                                          \
      spmv_typed<KK, false>(A, adjoint, x_is_f, d_x, d_y, st);    \
    return 0;                                                     \
  }
  DISPATCH(2)
  DISPATCH(3)
  DISPATCH(4)
#undef DISPATCH
  return 3;
}

// ---------------------------------------------------------------------
// Full-precision SpMV on an MC-valued matrix (sparse.py:414-451 ->
// _kernels.py:224-240 spmv_real, :266-278 spmv_adjoint_real, :300-323
// spmv_cx, :356-376 spmv_adjoint_cx): every product is the generic
// K x K `mul` / `cmul`, rows accumulate in ascending column order; the
// adjoint is a gather over the transposed pattern in ascending source-row
// order (the reference's scatter order per output row) with the matrix
// entry conjugated.  Values are planar: component c of entry p at
// mcv[c * vld + p], imaginary planes after the K real ones.  xf != 0: x is
// an F vector (binary64 head of an ILU(0)-mixed apply; zero tails).
// ---------------------------------------------------------------------
template <int K, bool CX, bool ADJ>
__global__ void __launch_bounds__(kBlock)
    spmv_full_kernel(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                     const int *__restrict__ perm, const double *__restrict__ mcv,
                     long long vld, const double *__restrict__ x, long long ld, int xf,
                     double *__restrict__ y, const int *done) {
  if (done && *done) return;
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n;
       i += (long long)gridDim.x * kBlock) {
    double yr[K], yi[K];
#pragma unroll
    for (int c = 0; c < K; ++c) yr[c] = yi[c] = 0.0;
    const int lo = rp[i], hi = rp[i + 1];
    for (int q = lo; q < hi; ++q) {
      const int j = ci[q];
      const long long p = ADJ ? perm[q] : q;
      double ar[K], xr[K];
#pragma unroll
      for (int c = 0; c < K; ++c) ar[c] = mcv[c * vld + p];
      if constexpr (!CX) {
        if (xf) {
#pragma unroll
          for (int c = 0; c < K; ++c) xr[c] = 0.0;
          xr[0] = x[j];
        } else {
#pragma unroll
          for (int c = 0; c < K; ++c) xr[c] = x[c * ld + j];
        }
        double t[K];
        mul<K>(ar, xr, t);
        add<K>(yr, t, yr);
      } else {
        double ai[K], xi[K], pr[K], pi[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double v = mcv[(K + c) * vld + p];
          ai[c] = ADJ ? -v : v;
        }
        if (xf) {
          const double2 xv = reinterpret_cast<const double2 *>(x)[j];
#pragma unroll
          for (int c = 0; c < K; ++c) xr[c] = xi[c] = 0.0;
          xr[0] = xv.x;
          xi[0] = xv.y;
        } else {
#pragma unroll
          for (int c = 0; c < K; ++c) {
            xr[c] = x[c * ld + j];
            xi[c] = x[(K + c) * ld + j];
          }
        }
        cmul<K>(ar, ai, xr, xi, pr, pi);
        add<K>(yr, pr, yr);
        add<K>(yi, pi, yi);
      }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
      y[c * ld + i] = yr[c];
      if constexpr (CX) y[(K + c) * ld + i] = yi[c];
    }
  }
}

int unit_spmv_full(DMat &A, int k, bool adjoint, bool x_is_f, const double *d_x,
                   double *d_y, const int *done, cudaStream_t st) {
  if (!A.mcv || A.mcv_k != k) return 3;
  if (adjoint) ensure_adjoint(A, st);
  const long long L = plane_ld(A.n);
  const int *rp = adjoint ? A.at_rp : A.rp, *ci = adjoint ? A.at_ci : A.ci;
  const int grid = grid_for(A.n);
  ++tl_launches;
#define LAUNCH(KK, CXX, ADJJ)                                                        \
  spmv_full_kernel<KK, CXX, ADJJ><<<grid, kBlock, 0, st>>>(                          \
      A.n, rp, ci, A.at_perm, A.mcv, A.mcv_ld, d_x, L, x_is_f ? 1 : 0, d_y, done)
#define DISPATCH(KK)                                   \
  if (k == KK) {                                       \
    if (A.cx) {                                        \
      if (adjoint) LAUNCH(KK, true, true);             \
      else LAUNCH(KK, true, false);                    \
    } else {                                           \
      if (adjoint) LAUNCH(KK, false, true);            \
      else LAUNCH(KK, false, false);                   \
    }                                                  \
    return 0;                                          \
  }
  DISPATCH(2)
  DISPATCH(3)
  DISPATCH(4)
#undef DISPATCH
#undef LAUNCH
  return 3;
}

// ---------------------------------------------------------------------
// Sweep-pipelined SpMV.  In BiCGSTAB / CGS / GPBiCG every SpMV multiplies
// the output z of an ILU(0)-mixed apply (solvers.py:303-304, 311-312).  On
// a large stencil pattern the apply is the shuffle-wavefront sweep
// (swf.cu), a latency-bound kernel on 64 of the 148 SMs; this kernel runs
// beside its backward phase on the other SMs and forms y_i = sum_j a_ij z_j
// for each 32-row chunk as soon as the sweep has published the chunk's
// inputs (z is sentinel-filled before the sweep, so "published" is visible
// in the value itself).  Per row the operations and their order are those
// of spmv_row (ascending columns, exact product + MC add), so y is the SpMV
// bit for bit; the fused row kernel that follows loads y for the chunks
// flagged here and computes the rest itself.
//  * Chunks are claimed in the order their inputs become complete (host:
//    max backward-DAG level over the rows' columns), through one counter;
//    a warp waits on ONE value (the chunk's last-produced column) with one
//    lane, so the ~2700 waiting warps cost L2 one load each per poll.
//  * No deadlock: a block first waits -- for a bounded time -- until every
//    CTA of the backward phase is running (they count themselves in), and
//    exits without claiming anything otherwise; once the sweep is resident
//    it completes on its own, so every wait on z ends.  The 88 KB of
//    dynamic shared memory only keep these blocks off the SMs of the sweep
//    CTAs (which own 142 KB each), whose single compute warp must not
//    share issue slots.
// ---------------------------------------------------------------------
struct PipeArgs {
  int n, nchunks, need_started;
  const int *rp, *ci;
  const double *val;
  const double *z;
  double *y;
  long long ld;
  const int *order, *last;
  int *state, *flag;
  const int *done;
};
constexpr int kPipeThreads = 512;

__global__ void pipe_delay_kernel() { __nanosleep(4000); }

template <int K>
__global__ void __launch_bounds__(kPipeThreads, 2) pspmv_kernel(PipeArgs a) {
  if (a.done && *(volatile const int *)a.done) return;
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    int go = 0;
    for (int t = 0; t < 1500 && !go; ++t) {  // <= ~0.3 ms
      go = *(volatile int *)(a.state + 1) >= a.need_started;
      if (!go) __nanosleep(200);
    }
    s_go = go;
  }
  __syncthreads();
  if (!s_go) return;
  const int lane = threadIdx.x & 31;
  const int sent_hi = (int)(kSentBits >> 32);
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(a.state, 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= a.nchunks) break;
    const int chunk = a.order[c];
    // gate: one lane polls the value that the sweep produces last for this
    // chunk (host: highest backward level among its columns); the lanes'
    // own loads below re-check every value
    if (lane == 0) {
      const double *g = a.z + a.last[chunk];
      while (__double2hiint(ld_relaxed(g)) == sent_hi) __nanosleep(300);
    }
    __syncwarp();
    const int i = chunk * 32 + lane;
    if (i < a.n) {
      const int lo = a.rp[i], len = a.rp[i + 1] - lo;
      int cj[kPipeRow];
      double xv[kPipeRow];
#pragma unroll
      for (int q = 0; q < kPipeRow; ++q) cj[q] = q < len ? a.ci[lo + q] : 0;
      for (;;) {
        bool ready = true;
#pragma unroll
        for (int q = 0; q < kPipeRow; ++q) {
          if (q < len) {
            xv[q] = ld_relaxed(a.z + cj[q]);
            ready = ready && (__double2hiint(xv[q]) != sent_hi);
          }
        }
        if (ready) break;
        __nanosleep(100);
      }
      double yr[K];
#pragma unroll
      for (int cc = 0; cc < K; ++cc) yr[cc] = 0.0;
#pragma unroll
      for (int q = 0; q < kPipeRow; ++q) {
        if (q < len) {  // spmv_row<K, false, true, false>: ascending columns
          double h, l;
          mul_ff2(a.val[lo + q], xv[q], h, l);
          add2<K>(yr, h, l, yr);
        }
      }
#pragma unroll
      for (int cc = 0; cc < K; ++cc) a.y[cc * a.ld + i] = yr[cc];
    }
    __syncwarp();
    if (lane == 0) a.flag[chunk] = 1;
  }
}

__global__ void pipe_reset_kernel(int *state, int *flag, int nchunks) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 4) state[t] = 0;
  for (int c = t; c < nchunks; c += gridDim.x * blockDim.x) flag[c] = 0;
}

// (measured: giving these side kernels the row kernels' max-shared-memory
// carveout preference costs 1 % on cfg4 -- they run on SMs without sweep CTAs
// and profit from the larger L1)
void launch_pipe_delay(cudaStream_t st) {
  ++tl_launches;
  pipe_delay_kernel<<<1, 1, 0, st>>>();
}

void launch_pipe_reset(DMat &A, cudaStream_t st) {
  ++tl_launches;
  pipe_reset_kernel<<<sm_count(), 256, 0, st>>>(A.pipe_state, A.pipe_flag, A.pipe_nchunks);
}

template <int K>
static void launch_pspmv_k(const PipeArgs &a, int grid, cudaStream_t st) {
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(pspmv_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kPipeSmem);
    once = true;
  }
  pspmv_kernel<K><<<grid, kPipeThreads, kPipeSmem, st>>>(a);
}

bool launch_pspmv(DMat &A, int k, const double *z, double *y, const int *done,
                  cudaStream_t st) {
  const int need = ssweep_bwd_ctas(A.smat.ss);
  if (!A.pipe_order || A.cx || need <= 0 || need >= sm_count()) return false;
  PipeArgs a{};
  a.n = A.n;
  // the chunks that become ready last are left to the consumer kernel, which
  // runs on all SMs right after the sweep (MPK_PIPE_FRAC: percent piped)
  static const int frac = getenv("MPK_PIPE_FRAC") ? atoi(getenv("MPK_PIPE_FRAC")) : 100;
  a.nchunks = (int)((long long)A.pipe_nchunks * (frac < 1 ? 1 : frac > 100 ? 100 : frac) / 100);
  a.need_started = need;
  a.rp = A.rp;
  a.ci = A.ci;
  a.val = A.val;
  a.z = z;
  a.y = y;
  a.ld = plane_ld(A.n);
  a.order = A.pipe_order;
  a.last = A.pipe_last;
  a.state = A.pipe_state;
  a.flag = A.pipe_flag;
  a.done = done;
  static const int bps = getenv("MPK_PIPE_BPS") ? atoi(getenv("MPK_PIPE_BPS")) : 2;  // A/B knob
  const int grid = (sm_count() - need) * (bps > 0 ? bps : 2);
  ++tl_launches;
  launch_pipe_delay(st);
  switch (k) {
    case 2: launch_pspmv_k<2>(a, grid, st); break;
    case 3: launch_pspmv_k<3>(a, grid, st); break;
    default: launch_pspmv_k<4>(a, grid, st); break;
  }
  return true;
}

template <int K, bool CX>
__global__ void unit_fin_kernel(const double *part, int G, int op,
                                double *out) {
  __shared__ double sm[kWarpsPerBlock * 8];
  if (op == 0) {
    const Sc s = finalize_slot<K, CX>(part, 0, G, sm);
    if (threadIdx.x == 0)
      for (int c = 0; c < K; ++c) {
        out[c] = s.re[c];
        out[4 + c] = s.im[c];
      }
  } else {
    const Sc s = finalize_slot<K, false>(part, 0, G, sm);
    if (threadIdx.x == 0) {
      double o[K];
      sqrt_mc<K>(R<K>(s), o);
      for (int c = 0; c < K; ++c) out[c] = o[c];
    }
  }
}

template <int K, bool CX>
static int reduce_typed(int op, long long n, const double *d_x,
                        const double *d_y, double *h_out, cudaStream_t st,
                        int seq_mode) {
  const long long L = plane_ld(n);
  const MV<K, CX> X{const_cast<double *>(d_x), L},
      Y{const_cast<double *>(d_y), L};
  double *part = nullptr, *out = nullptr, *seq = nullptr;
  cudaMalloc(&part, sizeof(double) * kMaxGrid * 8);
  cudaMalloc(&out, sizeof(double) * 8);
  if (seq_mode) cudaMalloc(&seq, sizeof(double) * 2 * K * (size_t)(n > 0 ? n : 1));
  tl_seq = seq;  // twin mode: ascending chain instead of the tree
  if (op == 0)
    rows<K, CX, 1, 0>(n, nullptr, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 0> &red) {
                        double xr[K], xi[K], yr[K], yi[K];
                        X.load(i, xr, xi);
                        Y.load(i, yr, yi);
                        acc_hdot<K, CX>(red.h[0], xr, xi, yr, yi);
                      });
  else
    rows<K, CX, 0, 1>(n, nullptr, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 1> &red) {
                        double xr[K], xi[K];
                        X.load(i, xr, xi);
                        acc_sumsq<K, CX>(red.nr[0], xr, xi);
                      });
  tl_seq = nullptr;
  unit_fin_kernel<K, CX><<<1, kBlock, 0, st>>>(part, seq ? 1 : grid_for(n), op, out);
  cudaMemcpyAsync(h_out, out, sizeof(double) * 8, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(part);
  cudaFree(out);
  if (seq) cudaFree(seq);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int unit_reduce(int k, bool cx, int op, long long n, const double *d_x,
                const double *d_y, double *h_out, cudaStream_t st, int seq) {
#define DISPATCH(KK)                                                      \
  if (k == KK)                                                            \
    return cx ? reduce_typed<KK, true>(op, n, d_x, d_y, h_out, st, seq)   \
              : reduce_typed<KK, false>(op, n, d_x, d_y, h_out, st, seq);
  DISPATCH(2)
  DISPATCH(3)
  DISPATCH(4)
#undef DISPATCH
  return 3;
}

template <int K, bool CX>
static int axpy_typed(long long n, const double *are, const double *aim,
                      const double *d_x, const double *d_y, double *d_out,
                      cudaStream_t st) {
  const long long L = plane_ld(n);
  const MV<K, CX> X{const_cast<double *>(d_x), L},
      Y{const_cast<double *>(d_y), L}, O{d_out, L};
  Sc al = sc_zero();
  for (int c = 0; c < K; ++c) {
    al.re[c] = are[c];
    al.im[c] = aim ? aim[c] : 0.0;
  }
  rows<K, CX, 0, 0>(n, nullptr, nullptr, st,
                    [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                      double xr[K], xi[K], yr[K], yi[K], orr[K], oi[K];
                      X.load(i, xr, xi);
                      Y.load(i, yr, yi);
                      e_axpy<K, CX>(al, xr, xi, yr, yi, orr, oi);
                      O.store(i, orr, oi);
                    });
  return 0;
}

int unit_axpy(int k, bool cx, long long n, const double *alpha_re,
              const double *alpha_im, const double *d_x, const double *d_y,
              double *d_out, cudaStream_t st) {
#define DISPATCH(KK)                                                        \
  if (k == KK)                                                              \
    return cx ? axpy_typed<KK, true>(n, alpha_re, alpha_im, d_x, d_y, d_out, \
                                     st)                                    \
              : axpy_typed<KK, false>(n, alpha_re, alpha_im, d_x, d_y,      \
                                      d_out, st);
  DISPATCH(2)
  DISPATCH(3)
  DISPATCH(4)
#undef DISPATCH
  return 3;
}

// element-wise MC ops on (n,k) AoS arrays (twin tests)
template <int K>
__host__ __device__ void mc_op_one(int op, const double *ar, const double *ai,
                                   const double *br, const double *bi,
                                   double *orr, double *oi) {
  double a[K], b[K], c[K], d[K], o[K], o2[K];
  for (int q = 0; q < K; ++q) {
    a[q] = ar[q];
    b[q] = br ? br[q] : 0.0;
    c[q] = ai ? ai[q] : 0.0;
    d[q] = bi ? bi[q] : 0.0;
    o[q] = o2[q] = 0.0;
  }
  switch (op) {
    case 0: add<K>(a, b, o); break;
    case 1: sub<K>(a, b, o); break;
    case 2: mul<K>(a, b, o); break;
    case 3: div<K>(a, b, o); break;
    case 4: sqrt_mc<K>(a, o); break;
    case 5: cmul<K>(a, c, b, d, o, o2); break;
    case 6: cdiv<K>(a, c, b, d, o, o2); break;
    case 7: {
      double t[7];
      for (int q = 0; q < 7; ++q) t[q] = ar[q];
      renorm<7, K>(t, o);
      break;
    }
    case 8: mul_lf<K>(a[0], b, o); break;
    case 9: mul_rf<K>(a, b[0], o); break;
    case 10: {
      double h, l;
      mul_ff2(a[0], b[0], h, l);
      o[0] = h;
      o[1] = l;
      break;
    }
    case 11: fmulsub<K>(a, b, c, o); break;  // a - b*c, c passed as a_im
    case 12: fmul<K>(a, b, o); break;
    default: break;
  }
  for (int q = 0; q < K; ++q) {
    orr[q] = o[q];
    if (oi) oi[q] = o2[q];
  }
}

template <int K>
__global__ void mc_kernel(int op, long long n, const double *ar,
                          const double *ai, const double *br,
                          const double *bi, double *orr, double *oi) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int sa = (op == 7) ? 7 : K;
  mc_op_one<K>(op, ar + i * sa, ai ? ai + i * K : nullptr,
               br ? br + i * K : nullptr, bi ? bi + i * K : nullptr,
               orr + i * K, oi ? oi + i * K : nullptr);
}

int unit_mc(int op, int k, const double *a_re, const double *a_im,
            const double *b_re, const double *b_im, double *o_re,
            double *o_im, int n, cudaStream_t st) {
  const int g = (n + 127) / 128;
  if (n <= 0) return 0;
  switch (k) {
    case 2: mc_kernel<2><<<g, 128, 0, st>>>(op, n, a_re, a_im, b_re, b_im, o_re, o_im); break;
    case 3: mc_kernel<3><<<g, 128, 0, st>>>(op, n, a_re, a_im, b_re, b_im, o_re, o_im); break;
    case 4: mc_kernel<4><<<g, 128, 0, st>>>(op, n, a_re, a_im, b_re, b_im, o_re, o_im); break;
    default: return 3;
  }
  return 0;
}

int host_mc(int op, int k, const double *a_re, const double *a_im,
            const double *b_re, const double *b_im, double *o_re,
            double *o_im) {
  // host-only error-free transformations (two_sum / two_prod exports,
  // _mccore.py:19-51): o = (s, e)
  if (op == 13 || op == 14) {
    double s, e;
    if (op == 13)
      two_sum(a_re[0], b_re[0], s, e);
    else
      two_prod(a_re[0], b_re[0], s, e);
    o_re[0] = s;
    o_re[1] = e;
    return 0;
  }
  switch (k) {
    case 1: {
      // k = 1 degenerates to native binary64 (multicomponent.py:31-66)
      double o = 0.0;
      switch (op) {
        case 0: o = dadd(a_re[0], b_re[0]); break;
        case 1: o = dsub(a_re[0], b_re[0]); break;
        case 2: o = dmul(a_re[0], b_re[0]); break;
        case 3: {
          const double x[1] = {a_re[0]}, y[1] = {b_re[0]};
          double q[1];
          div<1>(x, y, q);
          o = q[0];
          break;
        }
        case 4: {
          const double x[1] = {a_re[0]};
          double q[1];
          sqrt_mc<1>(x, q);
          o = q[0];
          break;
        }
        case 5:
        case 6: {  // complex mul / Smith division in plain binary64
          const double ar[1] = {a_re[0]}, ai[1] = {a_im ? a_im[0] : 0.0};
          const double br[1] = {b_re[0]}, bi[1] = {b_im ? b_im[0] : 0.0};
          double orr[1], oi[1];
          if (op == 5)
            cmul<1>(ar, ai, br, bi, orr, oi);
          else
            cdiv<1>(ar, ai, br, bi, orr, oi);
          o_re[0] = orr[0];
          if (o_im) o_im[0] = oi[0];
          return 0;
        }
        default: return 3;
      }
      o_re[0] = o;
      return 0;
    }
    case 2: mc_op_one<2>(op, a_re, a_im, b_re, b_im, o_re, o_im); return 0;
    case 3: mc_op_one<3>(op, a_re, a_im, b_re, b_im, o_re, o_im); return 0;
    case 4: mc_op_one<4>(op, a_re, a_im, b_re, b_im, o_re, o_im); return 0;
    default: return 3;
  }
}

// (n,k) AoS <-> planar
__global__ void to_planar_kernel(long long n, int k, const double *re,
                                 const double *im, double *dev, long long L) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int c = 0; c < k; ++c) {
    dev[c * L + i] = re[i * k + c];
    if (im) dev[(k + c) * L + i] = im[i * k + c];
  }
}
__global__ void from_planar_kernel(long long n, int k, const double *dev,
                                   long long L, double *re, double *im) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int c = 0; c < k; ++c) {
    re[i * k + c] = dev[c * L + i];
    if (im) im[i * k + c] = dev[(k + c) * L + i];
  }
}
void launch_to_planar(long long n, int k, const double *re, const double *im,
                      double *dev, cudaStream_t st) {
  if (n <= 0) return;
  ++tl_launches;
  to_planar_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      n, k, re, im, dev, plane_ld(n));
}
void launch_from_planar(long long n, int k, const double *dev, double *re,
                        double *im, cudaStream_t st) {
  if (n <= 0) return;
  ++tl_launches;
  from_planar_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      n, k, dev, plane_ld(n), re, im);
}

}  // namespace mpk
