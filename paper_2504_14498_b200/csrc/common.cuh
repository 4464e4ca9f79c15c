// common.cuh -- shared device infrastructure for the mpkrylov B200 hot path.
//
// HBM layout:
//   * MC vector (reference DenseVector, sparse.py:341-404) is PLANAR on the
//     device: component c of element i at p[c*ld + i]; complex vectors keep
//     the K real planes first, then the K imaginary planes.  Each plane is a
//     coalesced binary64 stream; the head plane is the binary64 demotion.
//   * F vector = an exactly promoted binary64 vector (ILU(0)-mixed outputs,
//     ilu.py:436-445): only the head is stored.  Real: double[n]; complex:
//     double2[n] (re, im interleaved, one 16-byte load per element).
#pragma once

#include <chrono>

#include <cuda_runtime.h>
#include <stdint.h>

#include "mc.cuh"

namespace mpk {

constexpr int kBlock = 256;       // threads per block for streaming kernels
constexpr int kMaxGrid = 592;     // 4 x 148 SMs: fixed => deterministic trees
constexpr int kWarpsPerBlock = kBlock / 32;

// Host-side count of kernels launched (or captured) by this thread; the
// C ABI reports per-call deltas (mpk_report.launches).
inline thread_local long long tl_launches = 0;
// Sequential-reduction twin mode (set by the solver while it builds its
// graphs): row kernels write every element's reduction term here instead of
// accumulating, and a chain kernel folds them in the reference's ascending
// order.  nullptr: fixed-shape tree reductions.
inline thread_local double *tl_seq = nullptr;
// host-side phase marks of the current solve (MPK_PHASE_TIMES diagnostics)
inline thread_local double tl_phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
// SM count of the current device (B200: 148), queried once
inline int sm_count() {
  static const int n = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    return v;
  }();
  return n;
}
inline double host_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Sentinel for sync-free triangular sweeps: a signalling NaN payload that no
// binary64 operation produces (hardware NaNs are quiet).
constexpr unsigned long long kSentBits = 0x7FF40000DEADBEEFull;
constexpr unsigned long long kQNaNBits = 0x7FF8000000000000ull;

__device__ __forceinline__ double sent_val() {
  return __longlong_as_double((long long)kSentBits);
}
__device__ __forceinline__ bool is_sent(double v) {
  return (unsigned long long)__double_as_longlong(v) == kSentBits;
}
__device__ __forceinline__ double unsent(double v) {
  return is_sent(v) ? __longlong_as_double((long long)kQNaNBits) : v;
}
__device__ __forceinline__ double ld_volatile(const double *p) {
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_volatile2(const double2 *p) {
  double2 v;
  asm volatile("ld.volatile.global.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_relaxed(const double *p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_relaxed2(const double2 *p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile(double *p, double v) {
  asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_volatile2(double2 *p, double2 v) {
  asm volatile("st.volatile.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x),
               "d"(v.y)
               : "memory");
}

// Spin until a sentinel-initialised slot has been published.
__device__ __forceinline__ double poll1(const double *p) {
  double v = ld_volatile(p);
  while (is_sent(v)) {
    __nanosleep(20);
    v = ld_volatile(p);
  }
  return v;
}
__device__ __forceinline__ double2 poll2(const double2 *p) {
  double2 v = ld_volatile2(p);
  while (is_sent(v.x) || is_sent(v.y)) {
    __nanosleep(20);
    v = ld_volatile2(p);
  }
  return v;
}

// ---------------------------------------------------------------------
// vector views
// ---------------------------------------------------------------------
template <int K, bool CX>
struct MV {
  double *p;
  int64_t ld;
  __device__ __forceinline__ void load(int64_t i, double (&re)[K],
                                       double (&im)[K]) const {
#pragma unroll
    for (int c = 0; c < K; ++c) re[c] = p[c * ld + i];
    if constexpr (CX) {
#pragma unroll
      for (int c = 0; c < K; ++c) im[c] = p[(K + c) * ld + i];
    }
  }
  __device__ __forceinline__ void store(int64_t i, const double (&re)[K],
                                        const double (&im)[K]) const {
#pragma unroll
    for (int c = 0; c < K; ++c) p[c * ld + i] = re[c];
    if constexpr (CX) {
#pragma unroll
      for (int c = 0; c < K; ++c) p[(K + c) * ld + i] = im[c];
    }
  }
  // binary64 demotion of element i (sparse.py:388-392): real head, or the
  // numpy `re + 1j*im` rounding for complex (re + (0*im - 0), 0 + im).
  __device__ __forceinline__ void head(int64_t i, double &hr,
                                       double &hi) const {
    if constexpr (CX) {
      const double re0 = p[i], im0 = p[K * ld + i];
      hr = dadd(re0, dsub(dmul(0.0, im0), 0.0));
      hi = dadd(0.0, im0);
    } else {
      hr = p[i];
      hi = 0.0;
    }
  }
};

// F vector view: the output of an ILU(0)-mixed apply, stored as its
// binary64 head only.  mc != 0 (preconditioner 'none', M = I): the "applied"
// vector is a full planar MC copy (ld stride), read back unchanged.
template <bool CX>
struct FV {
  double *p;
  long long ld = 0;
  int mc = 0;
  __device__ __forceinline__ void load(int64_t i, double &re,
                                       double &im) const {
    if constexpr (CX) {
      const double2 v = reinterpret_cast<const double2 *>(p)[i];
      re = v.x;
      im = v.y;
    } else {
      re = p[i];
      im = 0.0;
    }
  }
  // promoted MC element (zero tails)
  template <int K>
  __device__ __forceinline__ void load_mc(int64_t i, double (&re)[K],
                                          double (&im)[K]) const {
    if (mc) {
#pragma unroll
      for (int c = 0; c < K; ++c) {
        re[c] = p[c * ld + i];
        im[c] = CX ? p[(K + c) * ld + i] : 0.0;
      }
      return;
    }
    double r, m;
    load(i, r, m);
#pragma unroll
    for (int c = 0; c < K; ++c) re[c] = im[c] = 0.0;
    re[0] = r;
    im[0] = m;
  }
  __device__ __forceinline__ void set_sent(int64_t i) const {
    if constexpr (CX) {
      reinterpret_cast<double2 *>(p)[i] = make_double2(sent_val(), sent_val());
    } else {
      p[i] = sent_val();
    }
  }
};

// ---------------------------------------------------------------------
// scalars (MCFloat / MCComplex, multicomponent.py:79-401) on the device
// ---------------------------------------------------------------------
struct Sc {
  double re[4];
  double im[4];
};

template <int K>
__host__ __device__ __forceinline__ double (&R(Sc &s))[K] {
  return *reinterpret_cast<double(*)[K]>(s.re);
}
template <int K>
__host__ __device__ __forceinline__ double (&I(Sc &s))[K] {
  return *reinterpret_cast<double(*)[K]>(s.im);
}
template <int K>
__host__ __device__ __forceinline__ const double (&R(const Sc &s))[K] {
  return *reinterpret_cast<const double(*)[K]>(s.re);
}
template <int K>
__host__ __device__ __forceinline__ const double (&I(const Sc &s))[K] {
  return *reinterpret_cast<const double(*)[K]>(s.im);
}

__host__ __device__ __forceinline__ Sc sc_zero() {
  Sc s;
  for (int i = 0; i < 4; ++i) s.re[i] = s.im[i] = 0.0;
  return s;
}

template <int K, bool CX>
__device__ __noinline__ Sc s_add(Sc a, Sc b) {
  Sc o = sc_zero();
  add<K>(R<K>(a), R<K>(b), R<K>(o));
  if constexpr (CX) add<K>(I<K>(a), I<K>(b), I<K>(o));
  return o;
}
template <int K, bool CX>
__device__ __noinline__ Sc s_sub(Sc a, Sc b) {
  Sc o = sc_zero();
  sub<K>(R<K>(a), R<K>(b), R<K>(o));
  if constexpr (CX) sub<K>(I<K>(a), I<K>(b), I<K>(o));
  return o;
}
template <int K, bool CX>
__device__ __noinline__ Sc s_mul(Sc a, Sc b) {
  Sc o = sc_zero();
  if constexpr (CX)
    cmul<K>(R<K>(a), I<K>(a), R<K>(b), I<K>(b), R<K>(o), I<K>(o));
  else
    mul<K>(R<K>(a), R<K>(b), R<K>(o));
  return o;
}
template <int K, bool CX>
__device__ __noinline__ Sc s_div(Sc a, Sc b) {
  Sc o = sc_zero();
  if constexpr (CX)
    cdiv<K>(R<K>(a), I<K>(a), R<K>(b), I<K>(b), R<K>(o), I<K>(o));
  else
    div<K>(R<K>(a), R<K>(b), R<K>(o));
  return o;
}
template <int K>
__device__ __forceinline__ Sc s_neg(const Sc &a) {
  Sc o = sc_zero();
#pragma unroll
  for (int i = 0; i < K; ++i) {
    o.re[i] = -a.re[i];
    o.im[i] = -a.im[i];
  }
  return o;
}
template <int K, bool CX>
__device__ __forceinline__ Sc s_conj(const Sc &a) {
  Sc o = a;
  if constexpr (CX) {
#pragma unroll
    for (int i = 0; i < K; ++i) o.im[i] = -a.im[i];
  }
  return o;
}
template <int K, bool CX>
__device__ __forceinline__ bool s_is_zero(const Sc &a) {
  bool z = is_zero<K>(R<K>(a));
  if constexpr (CX) z = z && is_zero<K>(I<K>(a));
  return z;
}

// ---------------------------------------------------------------------
// element-level vector ops (mirrors of _kernels.py:408-552)
// ---------------------------------------------------------------------
// out = y + alpha*x  (axpy_real :408-418 / axpy_cx :421-434)
template <int K, bool CX>
__device__ __forceinline__ void e_axpy(const Sc &al, const double (&xr)[K],
                                       const double (&xi)[K],
                                       const double (&yr)[K],
                                       const double (&yi)[K], double (&or_)[K],
                                       double (&oi)[K]) {
  if constexpr (CX) {
    double pr[K], pi[K];
    cmul<K>(R<K>(al), I<K>(al), xr, xi, pr, pi);
    add<K>(yr, pr, or_);
    add<K>(yi, pi, oi);
  } else {
    double t[K];
    mul<K>(R<K>(al), xr, t);
    add<K>(yr, t, or_);
  }
}
// out = alpha*x  (scale_real :437-447 / scale_cx :450-464)
template <int K, bool CX>
__device__ __forceinline__ void e_scale(const Sc &al, const double (&xr)[K],
                                        const double (&xi)[K],
                                        double (&or_)[K], double (&oi)[K]) {
  if constexpr (CX) {
    cmul<K>(R<K>(al), I<K>(al), xr, xi, or_, oi);
  } else {
    mul<K>(R<K>(al), xr, or_);
  }
}
// out = x - y (sub_real :467-474 per plane)
template <int K, bool CX>
__device__ __forceinline__ void e_sub(const double (&xr)[K],
                                      const double (&xi)[K],
                                      const double (&yr)[K],
                                      const double (&yi)[K], double (&or_)[K],
                                      double (&oi)[K]) {
  sub<K>(xr, yr, or_);
  if constexpr (CX) sub<K>(xi, yi, oi);
}
template <int K, bool CX>
__device__ __forceinline__ void e_add(const double (&xr)[K],
                                      const double (&xi)[K],
                                      const double (&yr)[K],
                                      const double (&yi)[K], double (&or_)[K],
                                      double (&oi)[K]) {
  add<K>(xr, yr, or_);
  if constexpr (CX) add<K>(xi, yi, oi);
}

// ---------------------------------------------------------------------
// reductions: per-thread ascending accumulation, then a fixed-shape
// shuffle / shared-memory tree (deterministic for a fixed grid).
// ---------------------------------------------------------------------
template <int K, bool CX>
struct Acc {
  double re[K];
  double im[K];
  double *seq;  // twin mode: this element's term slot (2K doubles), else null
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < K; ++c) re[c] = im[c] = 0.0;
    seq = nullptr;
  }
};

// acc += conj(x)*y  (dot_real :487-499, hdot_cx :502-522)
template <int K, bool CX>
__device__ __forceinline__ void acc_hdot(Acc<K, CX> &a, const double (&xr)[K],
                                         const double (&xi)[K],
                                         const double (&yr)[K],
                                         const double (&yi)[K]) {
  if constexpr (CX) {
    double cj[K], pr[K], pi[K];
#pragma unroll
    for (int c = 0; c < K; ++c) cj[c] = -xi[c];
    cmul<K>(xr, cj, yr, yi, pr, pi);
    if (a.seq) {
#pragma unroll
      for (int c = 0; c < K; ++c) {
        a.seq[c] = pr[c];
        a.seq[K + c] = pi[c];
      }
      return;
    }
    add<K>(a.re, pr, a.re);
    add<K>(a.im, pi, a.im);
  } else {
    double t[K];
    mul<K>(xr, yr, t);
    if (a.seq) {
#pragma unroll
      for (int c = 0; c < K; ++c) a.seq[c] = t[c];
      return;
    }
    add<K>(a.re, t, a.re);
  }
}
// acc += |x|^2 (sumsq_real :525-536, sumsq_cx :539-552)
template <int K, bool CX>
__device__ __forceinline__ void acc_sumsq(Acc<K, false> &a,
                                          const double (&xr)[K],
                                          const double (&xi)[K]) {
  double t[K];
  mul<K>(xr, xr, t);
  if (a.seq) {  // complex: two terms (re^2, im^2) in the reference order
#pragma unroll
    for (int c = 0; c < K; ++c) a.seq[c] = t[c];
    if constexpr (CX) {
      mul<K>(xi, xi, t);
#pragma unroll
      for (int c = 0; c < K; ++c) a.seq[K + c] = t[c];
    }
    return;
  }
  add<K>(a.re, t, a.re);
  if constexpr (CX) {
    mul<K>(xi, xi, t);
    add<K>(a.re, t, a.re);
  }
}

template <int K, bool CX>
__device__ __forceinline__ void acc_combine(Acc<K, CX> &a,
                                            const Acc<K, CX> &b) {
  add<K>(a.re, b.re, a.re);
  if constexpr (CX) add<K>(a.im, b.im, a.im);
}

// The one-block finalize kernels run a few thousand instructions ONCE, on a
// cold instruction cache: their time follows their code size (ncu: 4.4 k
// instructions 17 us, 9.9 k instructions 41 us).  Their reduction trees
// therefore call ONE copy of the MC addition instead of inlining it at each
// of the ~9 tree levels (x2 for the complex variant).
template <int K>
__device__ __noinline__ void add_call(double *x, const double *y) {
  double a[K], b[K], r[K];
#pragma unroll
  for (int c = 0; c < K; ++c) {
    a[c] = x[c];
    b[c] = y[c];
  }
  add<K>(a, b, r);
#pragma unroll
  for (int c = 0; c < K; ++c) x[c] = r[c];
}
template <int K, bool CX>
__device__ __forceinline__ void acc_combine_call(Acc<K, CX> &a, const Acc<K, CX> &b) {
  add_call<K>(a.re, b.re);
  if constexpr (CX) add_call<K>(a.im, b.im);
}

template <int K, bool CX>
__device__ __forceinline__ void acc_shfl_down(Acc<K, CX> &o,
                                              const Acc<K, CX> &a, int off) {
#pragma unroll
  for (int c = 0; c < K; ++c) o.re[c] = __shfl_down_sync(0xffffffffu, a.re[c], off);
  if constexpr (CX) {
#pragma unroll
    for (int c = 0; c < K; ++c)
      o.im[c] = __shfl_down_sync(0xffffffffu, a.im[c], off);
  } else {
#pragma unroll
    for (int c = 0; c < K; ++c) o.im[c] = 0.0;
  }
}

// Block tree: lane tree (16,8,4,2,1) then warp leaders in smem, then warp 0
// tree over kWarpsPerBlock entries.  Result valid in threadIdx.x == 0.
// smem must hold kWarpsPerBlock * 2K doubles.  All threads must call.
template <int K, bool CX, bool CALL = false>
__device__ __forceinline__ void block_reduce(Acc<K, CX> &a, double *smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    Acc<K, CX> o;
    acc_shfl_down<K, CX>(o, a, off);
    if (lane < off) {
      if constexpr (CALL)
        acc_combine_call<K, CX>(a, o);
      else
        acc_combine<K, CX>(a, o);
    }
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      smem[warp * 2 * K + c] = a.re[c];
      smem[warp * 2 * K + K + c] = CX ? a.im[c] : 0.0;
    }
  }
  __syncthreads();
  if (warp == 0) {
    Acc<K, CX> b;
    if (lane < kWarpsPerBlock) {
#pragma unroll
      for (int c = 0; c < K; ++c) {
        b.re[c] = smem[lane * 2 * K + c];
        b.im[c] = smem[lane * 2 * K + K + c];
      }
    } else {
      b.zero();
    }
#pragma unroll
    for (int off = kWarpsPerBlock / 2; off >= 1; off >>= 1) {
      Acc<K, CX> o;
      acc_shfl_down<K, CX>(o, b, off);
      if (lane < off) {
        if constexpr (CALL)
          acc_combine_call<K, CX>(b, o);
        else
          acc_combine<K, CX>(b, o);
      }
    }
    a = b;
  }
  __syncthreads();
}

// write the block partial of slot s: part[(s*G + block)*8 + c]
template <int K, bool CX>
__device__ __forceinline__ void store_partial(double *part, int slot,
                                              const Acc<K, CX> &a) {
  if (threadIdx.x == 0) {
    double *q = part + ((size_t)slot * kMaxGrid + blockIdx.x) * 8;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      q[c] = a.re[c];
      q[4 + c] = CX ? a.im[c] : 0.0;
    }
  }
}

// Reduce G block partials of one slot in a fixed tree (one block).
template <int K, bool CX>
__device__ __forceinline__ Sc finalize_slot(const double *part, int slot,
                                            int G, double *smem) {
  Acc<K, CX> a;
  a.zero();
  for (int b = threadIdx.x; b < G; b += blockDim.x) {
    Acc<K, CX> v;
    const double *q = part + ((size_t)slot * kMaxGrid + b) * 8;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      v.re[c] = q[c];
      v.im[c] = q[4 + c];
    }
    acc_combine_call<K, CX>(a, v);
  }
  block_reduce<K, CX, true>(a, smem);
  Sc s = sc_zero();
#pragma unroll
  for (int c = 0; c < K; ++c) {
    s.re[c] = a.re[c];
    s.im[c] = CX ? a.im[c] : 0.0;
  }
  return s;  // valid in thread 0
}

// Reduce the G block partials of NS slots AT ONCE (slot s complex iff the
// s-th template flag): slot s gets W = kWarpsPerBlock / NS warps, each lane
// folds a strided subset of the partials, then a lane tree and a tree over
// the W warps -- the slots' trees run side by side instead of one after the
// other.  Fixed shape for a given (G, NS): deterministic.  Results are
// returned in out[] for every thread.  Uses smem[0, 8 * kWarpsPerBlock +
// 8 * NS) doubles.  All threads must call.
template <int K, bool C>
__device__ __forceinline__ void fin_slot_warp(const double *part, int slot, int G,
                                              int wi, int W, int lane,
                                              double *wsm) {
  Acc<K, C> a;
  a.zero();
  for (int b = wi * 32 + lane; b < G; b += 32 * W) {
    Acc<K, C> v;
    const double *q = part + ((size_t)slot * kMaxGrid + b) * 8;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      v.re[c] = q[c];
      v.im[c] = q[4 + c];
    }
    acc_combine_call<K, C>(a, v);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    Acc<K, C> o;
    acc_shfl_down<K, C>(o, a, off);
    if (lane < off) acc_combine_call<K, C>(a, o);
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      wsm[c] = a.re[c];
      wsm[4 + c] = C ? a.im[c] : 0.0;
    }
  }
}

template <int K, bool C>
__device__ __forceinline__ void fin_slot_cross(const double *wsm0, int W,
                                               int lane, Sc *dst) {
  Acc<K, C> b;
  b.zero();
  if (lane < W) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      b.re[c] = wsm0[lane * 8 + c];
      b.im[c] = wsm0[lane * 8 + 4 + c];
    }
  }
  for (int off = kWarpsPerBlock / 2; off >= 1; off >>= 1) {
    if (off >= W) continue;  // uniform
    Acc<K, C> o;
    acc_shfl_down<K, C>(o, b, off);
    if (lane < off) acc_combine_call<K, C>(b, o);
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      dst->re[c] = c < K ? b.re[c] : 0.0;
      dst->im[c] = (C && c < K) ? b.im[c] : 0.0;
    }
  }
}

template <int K, bool... CXS>
__device__ __forceinline__ void finalize_slots(const double *part, int G,
                                               double *smem, Sc *out) {
  constexpr int NS = sizeof...(CXS);
  static_assert(NS >= 1 && NS <= kWarpsPerBlock, "slots per finalize");
  constexpr bool cxs[NS] = {CXS...};
  constexpr int W = kWarpsPerBlock / NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = warp / W, wi = warp % W;
  Sc *res = reinterpret_cast<Sc *>(smem + 8 * kWarpsPerBlock);
  // only the variants the slot list needs are compiled (a real solve has no
  // complex slot: half the code of this cold single-block kernel)
  constexpr bool anyc = (CXS || ...), allc = (CXS && ...);
  if (s < NS) {
    if constexpr (!anyc) {
      fin_slot_warp<K, false>(part, s, G, wi, W, lane, smem + 8 * warp);
    } else if constexpr (allc) {
      fin_slot_warp<K, true>(part, s, G, wi, W, lane, smem + 8 * warp);
    } else {
      if (cxs[s])
        fin_slot_warp<K, true>(part, s, G, wi, W, lane, smem + 8 * warp);
      else
        fin_slot_warp<K, false>(part, s, G, wi, W, lane, smem + 8 * warp);
    }
  }
  __syncthreads();
  if (s < NS && wi == 0) {
    if constexpr (!anyc) {
      fin_slot_cross<K, false>(smem + 8 * warp, W, lane, res + s);
    } else if constexpr (allc) {
      fin_slot_cross<K, true>(smem + 8 * warp, W, lane, res + s);
    } else {
      if (cxs[s])
        fin_slot_cross<K, true>(smem + 8 * warp, W, lane, res + s);
      else
        fin_slot_cross<K, false>(smem + 8 * warp, W, lane, res + s);
    }
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < NS; ++t) out[t] = res[t];
}

inline int grid_for(int64_t n) {
  int64_t g = (n + kBlock - 1) / kBlock;
  if (g < 1) g = 1;
  if (g > kMaxGrid) g = kMaxGrid;
  return (int)g;
}

}  // namespace mpk
