// mc.cuh -- multi-component (DD/TD/QD) binary64 arithmetic, host+device.
//
// Bit-identical twin of the reference's scalar MC arithmetic
// (/root/reference/pkg/src/mpkrylov/_mccore.py:19-186,222-266,322-347 and
// its numba twin _kernels.py:24-214), re-designed for registers:
//
//  * renorm<M,K> runs the reference's distillation passes (VecSum +
//    zero-eliminating extraction + strictness check, <= 8 passes,
//    _mccore.py:54-116) on a FIXED M-slot register array.  Instead of
//    compacting the list (dynamic indexing -> local memory), eliminated
//    slots are left as +0.0 "holes".  A zero term is transparent to every
//    step of a pass: two_sum(x, 0) = (x, 0) exactly, extraction skips it, and
//    the strictness check / final truncation skip it as well, so the emitted
//    component sequence is identical to the compacted reference (only the
//    sign of zero results can differ, and the reference normalises those to
//    +0.0 at the end, _mccore.py:112-115).  This also means terms that are
//    known to be zero (zero tails of promoted binary64 values) can be dropped
//    at compile time: mul_lf / mul_rf / mul_ff below are the reference's
//    mc_mul with a promoted binary64 operand, minus its zero terms.
//  * TwoProd uses FMA when both operands lie in [2^-480, 2^480] (then it is
//    bit-identical to the reference's Dekker split, SURVEY.md finding 8) and
//    the reference's Dekker split itself otherwise (underflowing errors
//    differ between the two).  All other binary64 operations use explicit
//    _rn intrinsics, so no FMA contraction can occur regardless of flags.
//
// Non-finite operands follow the reference's non-finite path (plain sum of
// the terms in the head) except that products of a dropped zero term with
// an infinite operand are not formed; the result is non-finite either way.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define MPK_HD __host__ __device__ __forceinline__
// scalar-only operations (run once per iteration by one thread): keep them
// out of line so the kernels that call them stay small.
#define MPK_SCALAR __host__ __device__ __noinline__
#else
#define MPK_HD inline
#define MPK_SCALAR inline
#endif

namespace mpk {

MPK_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
MPK_HD double dsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  volatile double r = a - b;
  return r;
#endif
}
MPK_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
MPK_HD double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  volatile double r = a / b;
  return r;
#endif
}
MPK_HD double dfma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
MPK_HD double dsqrt(double a) {
#ifdef __CUDA_ARCH__
  return __dsqrt_rn(a);
#else
  return std::sqrt(a);
#endif
}
MPK_HD bool isfin(double a) {
#ifdef __CUDA_ARCH__
  return isfinite(a);
#else
  return std::isfinite(a);
#endif
}
MPK_HD double dabs(double a) { return fabs(a); }
MPK_HD int __builtin_ctz_dev(unsigned m) {
#ifdef __CUDA_ARCH__
  return __ffs((int)m) - 1;
#else
  return __builtin_ctz(m);
#endif
}

// two_sum _mccore.py:19-24
MPK_HD void two_sum(double a, double b, double &s, double &e) {
  double q = dadd(a, b);
  double bb = dsub(q, a);
  e = dadd(dsub(a, dsub(q, bb)), dsub(b, bb));
  s = q;
}

// Dekker split / two_prod exactly as the reference (_mccore.py:34-51)
MPK_HD double dekker_err(double a, double b, double p) {
  double t = dmul(134217729.0, a);
  const double ah = dsub(t, dsub(t, a));
  const double al = dsub(a, ah);
  t = dmul(134217729.0, b);
  const double bh = dsub(t, dsub(t, b));
  const double bl = dsub(b, bh);
  return dadd(dadd(dadd(dsub(dmul(ah, bh), p), dmul(ah, bl)), dmul(al, bh)),
              dmul(al, bl));
}

// |x| in [2^-480, 2^480] or x == 0: every partial product of Dekker's
// algorithm and the exact error of a*b are multiples of >= 2^-1064 below
// 2^1000, hence representable, so fma(a,b,-p) == Dekker bit for bit.
MPK_HD bool fma_safe(double x) {
#ifdef __CUDA_ARCH__
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
#else
  unsigned long long u;
  std::memcpy(&u, &x, sizeof u);
#endif
  const unsigned ex = (unsigned)((u >> 52) & 0x7ffu);
  return ((u << 1) == 0ull) || (ex - (1023u - 480u) <= 960u);
}

// two_prod _mccore.py:40-51: FMA form where provably identical (header)
MPK_HD void two_prod(double a, double b, double &p, double &e) {
  p = dmul(a, b);
  if (fma_safe(a) && fma_safe(b))
    e = dfma(a, b, -p);
  else
    e = dekker_err(a, b, p);
}

// finite test on the exponent bits (2 integer ops, no branch)
MPK_HD bool fin_bits(double x) {
#ifdef __CUDA_ARCH__
  return (__double2hiint(x) & 0x7ff00000) != 0x7ff00000;
#else
  return std::isfinite(x);
#endif
}

// Bit-level helpers (integer pipe): for finite values, |a| >= |b| iff the
// sign-cleared bit patterns compare so as unsigned integers, and x != 0.0
// iff its sign-cleared pattern is nonzero (NaN also counts as nonzero).
MPK_HD unsigned long long dbits(double x) {
#ifdef __CUDA_ARCH__
  return (unsigned long long)__double_as_longlong(x);
#else
  unsigned long long u;
  std::memcpy(&u, &x, sizeof u);
  return u;
#endif
}
MPK_HD unsigned long long mag(double x) { return dbits(x) & 0x7FFFFFFFFFFFFFFFull; }
MPK_HD bool nzb(double x) { return mag(x) != 0ull; }

// |x| < 2^1000 (and finite): no partial sum of <= 16 such terms can overflow
MPK_HD bool no_ovf(double x) {
  return mag(x) < ((unsigned long long)(1023 + 1000) << 52);
}

// implementation knobs (A/B-measured, see tools/ubench/mclat.cu)
#ifndef MPK_RN_COMPACT
#define MPK_RN_COMPACT 0  // 0: select chain, 1: local-array gather
#endif
#ifndef MPK_RN_INTCMP
#define MPK_RN_INTCMP 0   // magnitude / zero tests: 0 FP64 pipe, 1 integer pipe
#endif
#ifndef MPK_RN_S1FAST
#define MPK_RN_S1FAST 0   // sweep 1 errors by Fast2Sum (1) or TwoSum (0)
#endif
#ifdef MPK_COUNT_PASSES
__device__ unsigned long long g_pass_hist[20][8];
#endif
#ifdef MPK_RENORM_TIMING
__device__ long long g_rt[16];
#endif
#if defined(MPK_RENORM_TIMING) && defined(__CUDA_ARCH__)
#define MPK_RT(k) (g_rt[k] = clock64())
#else
#define MPK_RT(k) ((void)0)
#endif

// The pass loop of renorm_terms (_mccore.py:90-116).
//
// fast (all terms finite and below 2^1000, so no partial sum overflows):
// every TwoSum error is computed by Fast2Sum on the larger-magnitude
// operand, chosen by an integer compare beside the sum.  The error of an
// addition is unique, so the value equals TwoSum's; a zero error is forced
// to +0.0, which is what TwoSum yields for an exact sum (x - x = +0 in
// round-to-nearest), so even the signs of zeros agree.  In sweep 2 the sign
// of a zero error is never observed (only en != 0 is tested).
template <int M, bool fast>
MPK_HD void renorm_passes(double (&t)[M]) {
#pragma unroll 1
  for (int pass = 0; pass < 8; ++pass) {
    double e[M];
    double s = t[M - 1];
#pragma unroll
    for (int i = M - 2; i >= 0; --i) {
      double q, err;
      if constexpr (fast && MPK_RN_S1FAST) {
        const double a = t[i];
        q = dadd(a, s);
        const bool ge = MPK_RN_INTCMP ? (mag(a) >= mag(s)) : (dabs(a) >= dabs(s));
        const double big = ge ? a : s, sml = ge ? s : a;
        err = dsub(sml, dsub(q, big));
        err = (MPK_RN_INTCMP ? nzb(err) : (err != 0.0)) ? err : 0.0;
      } else {
        two_sum(t[i], s, q, err);
      }
      e[i + 1] = err;
      s = q;
    }
    e[0] = s;
    MPK_RT(2);
    double eps = e[0];
#pragma unroll
    for (int i = 1; i < M; ++i) {
      double q, en;
      if constexpr (fast) {
        const double ei = e[i];
        q = dadd(eps, ei);
        const bool ge = MPK_RN_INTCMP ? (mag(eps) >= mag(ei)) : (dabs(eps) >= dabs(ei));
        const double big = ge ? eps : ei, sml = ge ? ei : eps;
        en = dsub(sml, dsub(q, big));
      } else {
        two_sum(eps, e[i], q, en);
      }
      const bool em = MPK_RN_INTCMP ? nzb(en) : (en != 0.0);
      t[i - 1] = em ? q : 0.0;
      eps = em ? en : q;
    }
    t[M - 1] = eps;
    MPK_RT(3);
    // strictness over consecutive non-hole components (branch-free); for a
    // nonzero finite prev, fl(prev + c) != prev iff the bit patterns differ
    bool ok = true;
    double prev = 0.0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const double c = t[i];
#if MPK_RN_INTCMP
      const bool nz = nzb(c);
      const bool viol = nz & nzb(prev) & (dbits(dadd(prev, c)) != dbits(prev));
#else
      const bool nz = (c != 0.0);
      const bool viol = nz & (prev != 0.0) & (dadd(prev, c) != prev);
#endif
      ok = ok & !viol;
      prev = nz ? c : prev;
    }
#if defined(MPK_COUNT_PASSES) && defined(__CUDA_ARCH__)
    atomicAdd(&g_pass_hist[M][pass], 1ull);
#endif
    MPK_RT(4);
    if (ok) break;
  }
}

template <int M, int K>
MPK_HD void renorm_body(double (&t)[M], double (&out)[K]);

// TD / QD on the device: ONE copy of each renormalisation per kernel, called.
// The TD / QD row kernels of the BASELINE configs run on small systems (one
// element per thread: the body executes once per warp), where ncu attributes
// a third of the stall cycles to instruction fetch (r02 cfg5 captures: 34 %
// "no instruction") -- the inlined renormalisations are most of the code.
// DD keeps the inlined form (cfg4: the loop body is reused 28 times).
#if defined(__CUDACC__)
template <int M, int K>
__device__ __noinline__ void renorm_call(double *t, double *out) {
  double a[M], o[K];
#pragma unroll
  for (int i = 0; i < M; ++i) a[i] = t[i];
  renorm_body<M, K>(a, o);
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = o[i];
}
#endif

template <int M, int K>
MPK_HD void renorm(double (&t)[M], double (&out)[K]) {
#ifndef MPK_RENORM_CALL_MIN_K
#define MPK_RENORM_CALL_MIN_K 3  // DD measured slower when called (cfg1 --precond ilu0 455 -> 406 it/s)
#endif
#if defined(__CUDA_ARCH__) && !defined(MPK_INLINE_RENORM)
  if constexpr (K >= MPK_RENORM_CALL_MIN_K) {
    renorm_call<M, K>(t, out);
    return;
  }
#endif
  renorm_body<M, K>(t, out);
}

template <int M, int K>
MPK_HD void renorm_body(double (&t)[M], double (&out)[K]) {
  MPK_RT(0);
  bool small = true;
#pragma unroll
  for (int i = 0; i < M; ++i) small = small & no_ovf(t[i]);
  if (!small) {
    bool fin = true;
#pragma unroll
    for (int i = 0; i < M; ++i) fin = fin & fin_bits(t[i]);
    if (!fin) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < M; ++i) s = dadd(s, t[i]);
      out[0] = s;
#pragma unroll
      for (int i = 1; i < K; ++i) out[i] = 0.0;
      return;
    }
    renorm_passes<M, false>(t);
  } else {
    MPK_RT(1);
    renorm_passes<M, true>(t);
    MPK_RT(5);
  }
#if MPK_RN_COMPACT == 0
  // first K non-hole components (branch-free predicated selects)
#pragma unroll
  for (int j = 0; j < K; ++j) out[j] = 0.0;
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const double c = t[i];
    const bool nz = (c != 0.0);
#pragma unroll
    for (int j = 0; j < K; ++j) out[j] = (nz & (cnt == j)) ? c : out[j];
    cnt += nz ? 1 : 0;
  }
#else
  // first K non-hole components: positions by clearing the lowest set bit
  // of the nonzero mask, values gathered from a local copy (independent
  // loads instead of a select chain through a running count)
  unsigned mask = 0u;
#pragma unroll
  for (int i = 0; i < M; ++i) mask |= nzb(t[i]) ? (1u << i) : 0u;
  double tl[M];
#pragma unroll
  for (int i = 0; i < M; ++i) tl[i] = t[i];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int p = mask ? (__builtin_ctz_dev(mask)) : 0;
    out[j] = mask ? tl[p] : 0.0;
    mask &= mask - 1u;
  }
#endif
  MPK_RT(6);
}

// Reference merge of two component lists by magnitude, ties prefer x
// (_mccore.py:134-154), for arbitrary (not necessarily sorted) inputs.
// The two inputs are consumed as shift registers (heads xq[0] / yq[0]) so
// every index is static: a dynamically indexed x[i] is lowered to local
// memory, which put an L1 round trip on each merge step.
template <int KX, int KY, bool INTCMP>
MPK_HD void merge_q(const double (&x)[KX], const double (&y)[KY],
                    double (&buf)[KX + KY]) {
  double xq[KX], yq[KY];
#pragma unroll
  for (int a = 0; a < KX; ++a) xq[a] = x[a];
#pragma unroll
  for (int a = 0; a < KY; ++a) yq[a] = y[a];
  int nx = KX, ny = KY;  // remaining
#pragma unroll
  for (int t = 0; t < KX + KY; ++t) {
    const bool xv = nx > 0, yv = ny > 0;
    const bool ge = (INTCMP && MPK_RN_INTCMP) ? (mag(xq[0]) >= mag(yq[0]))
                                              : (dabs(xq[0]) >= dabs(yq[0]));
    const bool tx = xv && (!yv || ge);
    buf[t] = tx ? xq[0] : yq[0];
#pragma unroll
    for (int a = 0; a + 1 < KX; ++a) xq[a] = tx ? xq[a + 1] : xq[a];
#pragma unroll
    for (int a = 0; a + 1 < KY; ++a) yq[a] = tx ? yq[a] : yq[a + 1];
    nx -= tx ? 1 : 0;
    ny -= tx ? 0 : 1;
  }
}

// magnitude compares on the integer pipe when every input is finite (for
// NaN the IEEE compare is false, which the integer one would not reproduce)
template <int KX, int KY>
MPK_HD void merge(const double (&x)[KX], const double (&y)[KY],
                  double (&buf)[KX + KY]) {
  bool fin = true;
#pragma unroll
  for (int a = 0; a < KX; ++a) fin = fin & fin_bits(x[a]);
#pragma unroll
  for (int a = 0; a < KY; ++a) fin = fin & fin_bits(y[a]);
  if (fin)
    merge_q<KX, KY, true>(x, y, buf);
  else
    merge_q<KX, KY, false>(x, y, buf);
}

// mc_add _mccore.py:129-155
template <int K>
MPK_HD void add(const double (&x)[K], const double (&y)[K], double (&out)[K]) {
  if (K == 1) {
    out[0] = dadd(x[0], y[0]);
    return;
  }
  double buf[2 * K];
  merge<K, K>(x, y, buf);
  renorm<2 * K, K>(buf, out);
}

// mc_add(x, (y0, y1, 0, ..., 0)): the trailing zeros of y are merged after
// every element of x (|x_i| >= 0), so they are transparent.
template <int K>
MPK_HD void add2(const double (&x)[K], double y0, double y1,
                 double (&out)[K]) {
  if (K == 1) {
    out[0] = dadd(x[0], y0);
    return;
  }
  const double y[2] = {y0, y1};
  double buf[K + 2];
  merge<K, 2>(x, y, buf);
  renorm<K + 2, K>(buf, out);
}

// mc_sub _mccore.py:158-159 (add of the componentwise negation)
template <int K>
MPK_HD void sub(const double (&x)[K], const double (&y)[K], double (&out)[K]) {
  double ny[K];
#pragma unroll
  for (int i = 0; i < K; ++i) ny[i] = -y[i];
  add<K>(x, ny, out);
}

template <int K>
MPK_HD void neg(const double (&x)[K], double (&out)[K]) {
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = -x[i];
}

// mc_mul _mccore.py:162-186: level l < K-1 two-prods (errors carried to
// level l+1), level K-1 plain products, renorm of the K*K terms.
template <int K>
MPK_HD void mul(const double (&x)[K], const double (&y)[K], double (&out)[K]) {
  if (K == 1) {
    out[0] = dmul(x[0], y[0]);
    return;
  }
  double t[K * K];
  double carry[K > 1 ? K - 1 : 1];
  double nxt[K > 1 ? K - 1 : 1];
  int nt = 0;
#pragma unroll
  for (int lvl = 0; lvl < K; ++lvl) {
    if (lvl < K - 1) {
#pragma unroll
      for (int i = 0; i <= lvl; ++i) {
        double p, e;
        two_prod(x[i], y[lvl - i], p, e);
        t[nt++] = p;
        nxt[i] = e;
      }
    } else {
#pragma unroll
      for (int i = 0; i <= lvl; ++i) t[nt++] = dmul(x[i], y[lvl - i]);
    }
#pragma unroll
    for (int c = 0; c < lvl; ++c) t[nt++] = carry[c];
    if (lvl < K - 1) {
#pragma unroll
      for (int c = 0; c <= lvl; ++c) carry[c] = nxt[c];
    }
  }
  renorm<K * K, K>(t, out);
}

// mc_mul((a,0,..,0), y): non-zero terms in reference order are
// p(a,y0) | p(a,y1) e(a,y0) | ... | a*y_{K-1} e(a,y_{K-2})  (2K-1 slots)
template <int K>
MPK_HD void mul_lf(double a, const double (&y)[K], double (&out)[K]) {
  if (K == 1) {
    out[0] = dmul(a, y[0]);
    return;
  }
  double t[2 * K - 1];
  double pe = 0.0;
  int nt = 0;
#pragma unroll
  for (int l = 0; l < K; ++l) {
    if (l < K - 1) {
      double p, e;
      two_prod(a, y[l], p, e);
      t[nt++] = p;
      if (l > 0) t[nt++] = pe;
      pe = e;
    } else {
      t[nt++] = dmul(a, y[l]);
      t[nt++] = pe;
    }
  }
  renorm<2 * K - 1, K>(t, out);
}

// mc_mul(x, (f,0,..,0)): same slot pattern with p(x_l, f).
template <int K>
MPK_HD void mul_rf(const double (&x)[K], double f, double (&out)[K]) {
  if (K == 1) {
    out[0] = dmul(x[0], f);
    return;
  }
  double t[2 * K - 1];
  double pe = 0.0;
  int nt = 0;
#pragma unroll
  for (int l = 0; l < K; ++l) {
    if (l < K - 1) {
      double p, e;
      two_prod(x[l], f, p, e);
      t[nt++] = p;
      if (l > 0) t[nt++] = pe;
      pe = e;
    } else {
      t[nt++] = dmul(x[l], f);
      t[nt++] = pe;
    }
  }
  renorm<2 * K - 1, K>(t, out);
}

// mc_mul((a,0..), (f,0..)) = renorm([p, e]) = (p+0, e+0, 0, ..) when p is
// finite (|e| <= ulp(p)/2 and fl(p+e) = p by round-to-nearest-even).
MPK_HD void mul_ff2(double a, double f, double &h, double &l) {
  double p, e;
  if (fma_safe(a) && fma_safe(f)) {
    p = dmul(a, f);
    e = dfma(a, f, -p);
    h = dadd(p, 0.0);
    l = dadd(e, 0.0);
  } else {
    p = dmul(a, f);
    e = dekker_err(a, f, p);
    double t[2] = {p, e}, o[2];
    renorm<2, 2>(t, o);
    h = o[0];
    l = o[1];
  }
}

// complex product (twin _cmul1 _kernels.py:206-214 / cx_mul _mccore.py:322)
template <int K>
MPK_HD void cmul(const double (&ar)[K], const double (&ai)[K],
                 const double (&br)[K], const double (&bi)[K],
                 double (&outr)[K], double (&outi)[K]) {
  double t1[K], t2[K], r[K];
  mul<K>(ar, br, t1);
  mul<K>(ai, bi, t2);
  sub<K>(t1, t2, r);
  mul<K>(ar, bi, t1);
  mul<K>(ai, br, t2);
  add<K>(t1, t2, outi);
#pragma unroll
  for (int i = 0; i < K; ++i) outr[i] = r[i];
}

// complex product with a promoted binary64 left operand (ar,0..)+i(ai,0..)
template <int K>
MPK_HD void cmul_lf(double ar, double ai, const double (&br)[K],
                    const double (&bi)[K], double (&outr)[K],
                    double (&outi)[K]) {
  double t1[K], t2[K], r[K];
  mul_lf<K>(ar, br, t1);
  mul_lf<K>(ai, bi, t2);
  sub<K>(t1, t2, r);
  mul_lf<K>(ar, bi, t1);
  mul_lf<K>(ai, br, t2);
  add<K>(t1, t2, outi);
#pragma unroll
  for (int i = 0; i < K; ++i) outr[i] = r[i];
}

// complex product of two promoted binary64 values: each real product is a
// 2-term value (p, e); sub/add merge two 2-term lists (zeros transparent).
template <int K>
MPK_HD void cmul_ff(double ar, double ai, double br, double bi,
                    double (&outr)[K], double (&outi)[K]) {
  double h1, l1, h2, l2;
  mul_ff2(ar, br, h1, l1);
  mul_ff2(ai, bi, h2, l2);
  {
    const double x[2] = {h1, l1};
    const double y[2] = {-h2, -l2};
    double buf[4];
    merge<2, 2>(x, y, buf);
    renorm<4, K>(buf, outr);
  }
  mul_ff2(ar, bi, h1, l1);
  mul_ff2(ai, br, h2, l2);
  {
    const double x[2] = {h1, l1};
    const double y[2] = {h2, l2};
    double buf[4];
    merge<2, 2>(x, y, buf);
    renorm<4, K>(buf, outi);
  }
}

template <int K>
MPK_HD bool is_zero(const double (&x)[K]) {
  bool z = true;
#pragma unroll
  for (int i = 0; i < K; ++i) z = z && (x[i] == 0.0);
  return z;
}

template <int K>
MPK_HD bool is_finite(const double (&x)[K]) {
  bool f = true;
#pragma unroll
  for (int i = 0; i < K; ++i) f = f && isfin(x[i]);
  return f;
}

// Out-of-line MC operations for the scalar recurrences.  They take and
// return small structs BY VALUE (register ABI): passing references to a
// caller's register arrays into a __noinline__ function is exactly what
// faulted on sm_100a, so no pointer to a caller-local array ever crosses
// these call boundaries.  Division / sqrt call them instead of inlining 13
// full operations: the inlined bodies overflowed the instruction cache
// (a single-thread division streamed ~100 KB of code per call).
template <int K>
struct V {
  double c[K];
};
template <int K>
struct V2 {
  double r[K];
  double i[K];
};
template <int K>
MPK_SCALAR V<K> mul_v(V<K> x, V<K> y) {
  V<K> o;
  mul<K>(x.c, y.c, o.c);
  return o;
}
template <int K>
MPK_SCALAR V<K> add_v(V<K> x, V<K> y) {
  V<K> o;
  add<K>(x.c, y.c, o.c);
  return o;
}
template <int K>
MPK_HD void mul_o(const double (&x)[K], const double (&y)[K], double (&out)[K]) {
  V<K> a, b;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    a.c[i] = x[i];
    b.c[i] = y[i];
  }
  const V<K> o = mul_v<K>(a, b);
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = o.c[i];
}
template <int K>
MPK_HD void add_o(const double (&x)[K], const double (&y)[K], double (&out)[K]) {
  V<K> a, b;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    a.c[i] = x[i];
    b.c[i] = y[i];
  }
  const V<K> o = add_v<K>(a, b);
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = o.c[i];
}
template <int K>
MPK_HD void sub_o(const double (&x)[K], const double (&y)[K], double (&out)[K]) {
  double ny[K];
#pragma unroll
  for (int i = 0; i < K; ++i) ny[i] = -y[i];
  add_o<K>(x, ny, out);
}

// _div_by_zero _mccore.py:216-219
MPK_HD double div_by_zero(double x0, double y0) {
  if (x0 == 0.0) return NAN;
  return dmul(copysign(INFINITY, x0), copysign(1.0, y0));
}

// mc_div _mccore.py:222-237 (Newton reciprocal seeded by binary64 1/y0)
template <int K>
MPK_HD void div_a(const double (&x)[K], const double (&y)[K], double (&out)[K]) {
  if (K == 1) {
    out[0] = (y[0] == 0.0) ? div_by_zero(x[0], y[0]) : ddiv(x[0], y[0]);
    return;
  }
  if (y[0] == 0.0 && is_zero<K>(y)) {
    out[0] = div_by_zero(x[0], y[0]);
#pragma unroll
    for (int i = 1; i < K; ++i) out[i] = 0.0;
    return;
  }
  double one[K], w[K], t1[K], t2[K];
#pragma unroll
  for (int i = 0; i < K; ++i) one[i] = w[i] = 0.0;
  one[0] = 1.0;
  w[0] = ddiv(1.0, y[0]);
  const int iters = (K == 2) ? 1 : 2;
  for (int it = 0; it < iters; ++it) {
    mul_o<K>(y, w, t1);
    sub_o<K>(one, t1, t2);
    mul_o<K>(w, t2, t1);
    add_o<K>(w, t1, t2);
#pragma unroll
    for (int i = 0; i < K; ++i) w[i] = t2[i];
  }
  double q[K], r[K];
  mul_o<K>(x, w, q);
  mul_o<K>(q, y, t1);
  sub_o<K>(x, t1, r);
  mul_o<K>(r, w, t2);
  add_o<K>(q, t2, out);
}

// mc_sqrt _mccore.py:245-266 (Newton on rsqrt). Returns false if x0 < 0.
template <int K>
MPK_HD bool sqrt_a(const double (&x)[K], double (&out)[K]) {
  if (x[0] < 0.0) {
#pragma unroll
    for (int i = 0; i < K; ++i) out[i] = NAN;
    return false;
  }
  if (x[0] == 0.0 && is_zero<K>(x)) {
#pragma unroll
    for (int i = 0; i < K; ++i) out[i] = 0.0;
    return true;
  }
  if (K == 1) {
    out[0] = dsqrt(x[0]);
    return true;
  }
  double one[K], z[K], t[K], a[K], b[K];
#pragma unroll
  for (int i = 0; i < K; ++i) one[i] = z[i] = 0.0;
  one[0] = 1.0;
  z[0] = ddiv(1.0, dsqrt(x[0]));
  const int iters = (K == 2) ? 1 : 2;
  for (int it = 0; it < iters; ++it) {
    mul_o<K>(z, z, a);
    mul_o<K>(x, a, b);
    sub_o<K>(one, b, t);
    mul_o<K>(z, t, a);
#pragma unroll
    for (int i = 0; i < K; ++i) a[i] = dmul(a[i], 0.5);
    add_o<K>(z, a, b);
#pragma unroll
    for (int i = 0; i < K; ++i) z[i] = b[i];
  }
  double r[K];
  mul_o<K>(x, z, r);
  mul_o<K>(r, r, a);
  sub_o<K>(x, a, t);
#pragma unroll
  for (int i = 0; i < K; ++i) b[i] = dmul(z[i], 0.5);
  mul_o<K>(t, b, a);
  add_o<K>(r, a, out);
  return true;
}

// mc_cmp _mccore.py:283-290
template <int K>
MPK_HD int cmp_a(const double (&x)[K], const double (&y)[K]) {
  double d[K];
  sub_o<K>(x, y, d);
  if (d[0] > 0.0) return 1;
  if (d[0] < 0.0) return -1;
  return 0;
}

// Out-of-line scalar entry points (by-value structs, see V above).

template <int K>
MPK_SCALAR V<K> div_v(V<K> x, V<K> y) {
  V<K> o;
  div_a<K>(x.c, y.c, o.c);
  return o;
}
template <int K>
MPK_SCALAR V<K> sqrt_v(V<K> x) {
  V<K> o;
  sqrt_a<K>(x.c, o.c);
  return o;
}
template <int K>
MPK_SCALAR int cmp_v(V<K> x, V<K> y) {
  return cmp_a<K>(x.c, y.c);
}

template <int K>
MPK_HD void div(const double (&x)[K], const double (&y)[K], double (&out)[K]) {
  V<K> a, b;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    a.c[i] = x[i];
    b.c[i] = y[i];
  }
  const V<K> o = div_v<K>(a, b);
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = o.c[i];
}
template <int K>
MPK_HD bool sqrt_mc(const double (&x)[K], double (&out)[K]) {
  V<K> a;
#pragma unroll
  for (int i = 0; i < K; ++i) a.c[i] = x[i];
  const V<K> o = sqrt_v<K>(a);
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = o.c[i];
  return !(x[0] < 0.0);
}
template <int K>
MPK_HD int cmp(const double (&x)[K], const double (&y)[K]) {
  V<K> a, b;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    a.c[i] = x[i];
    b.c[i] = y[i];
  }
  return cmp_v<K>(a, b);
}

// cx_div _mccore.py:328-347 (Smith)
template <int K>
MPK_HD void cdiv_a(const double (&ar)[K], const double (&ai)[K],
                 const double (&br)[K], const double (&bi)[K],
                 double (&outr)[K], double (&outi)[K]) {
  double t[K], d[K], u[K], v[K], re[K], im[K];
  if (dabs(br[0]) >= dabs(bi[0])) {
    if (is_zero<K>(br) && is_zero<K>(bi)) {
      outr[0] = div_by_zero(ar[0], 0.0);
      outi[0] = div_by_zero(ai[0], 0.0);
#pragma unroll
      for (int i = 1; i < K; ++i) outr[i] = outi[i] = 0.0;
      return;
    }
    div<K>(bi, br, t);
    mul_o<K>(bi, t, u);
    add_o<K>(br, u, d);
    mul_o<K>(ai, t, u);
    add_o<K>(ar, u, v);
    div<K>(v, d, re);
    mul_o<K>(ar, t, u);
    sub_o<K>(ai, u, v);
    div<K>(v, d, im);
  } else {
    div<K>(br, bi, t);
    mul_o<K>(br, t, u);
    add_o<K>(u, bi, d);
    mul_o<K>(ar, t, u);
    add_o<K>(u, ai, v);
    div<K>(v, d, re);
    mul_o<K>(ai, t, u);
    sub_o<K>(u, ar, v);
    div<K>(v, d, im);
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    outr[i] = re[i];
    outi[i] = im[i];
  }
}

template <int K>
MPK_SCALAR V2<K> cdiv_v(V2<K> a, V2<K> b) {
  V2<K> o;
  cdiv_a<K>(a.r, a.i, b.r, b.i, o.r, o.i);
  return o;
}

template <int K>
MPK_HD void cdiv(const double (&ar)[K], const double (&ai)[K],
                 const double (&br)[K], const double (&bi)[K],
                 double (&outr)[K], double (&outi)[K]) {
  V2<K> a, b;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    a.r[i] = ar[i];
    a.i[i] = ai[i];
    b.r[i] = br[i];
    b.i[i] = bi[i];
  }
  const V2<K> o = cdiv_v<K>(a, b);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    outr[i] = o.r[i];
    outi[i] = o.i[i];
  }
}

// ---------------------------------------------------------------------
// CPython binary64 complex arithmetic (k=1 complex ILU(0), ilu.py:195-220,
// :377-381): product without FMA, Smith division as in _Py_c_quot.
// ---------------------------------------------------------------------
MPK_HD void py_cmul(double ar, double ai, double br, double bi, double &pr,
                    double &pi) {
  pr = dsub(dmul(ar, br), dmul(ai, bi));
  pi = dadd(dmul(ar, bi), dmul(ai, br));
}

MPK_HD void py_cdiv(double ar, double ai, double br, double bi, double &qr,
                    double &qi) {
  const double abr = br < 0 ? -br : br;
  const double abi = bi < 0 ? -bi : bi;
  if (abr >= abi) {
    if (abr == 0.0) {
      qr = qi = 0.0;  // CPython raises ZeroDivisionError; unreachable
    } else {
      const double ratio = ddiv(bi, br);
      const double denom = dadd(br, dmul(bi, ratio));
      qr = ddiv(dadd(ar, dmul(ai, ratio)), denom);
      qi = ddiv(dsub(ai, dmul(ar, ratio)), denom);
    }
  } else if (abi >= abr) {
    const double ratio = ddiv(br, bi);
    const double denom = dadd(dmul(br, ratio), bi);
    qr = ddiv(dadd(dmul(ar, ratio), ai), denom);
    qi = ddiv(dsub(dmul(ai, ratio), ar), denom);
  } else {
    qr = qi = NAN;
  }
}

// ---------------------------------------------------------------------
// Fused sweep primitives of the working-precision ILU(0) (_mcfast.py:80-183):
// r = a - b*c and p = a*b build the full partial-product term list (Dekker
// errors of the leading products, plain binary64 sums of the highest kept
// level) and renormalise ONCE.  The reference's _fr is one distillation
// pass with the fixpoint renorm_terms as fallback when the pass is not
// strict, i.e. renorm_terms itself for finite terms (same VecSum, same
// zero-eliminating extraction, same strictness test, same -0 -> +0
// normalisation); renorm<M,K> is the device twin of renorm_terms.
// ---------------------------------------------------------------------
template <int K>
MPK_HD void fmulsub(const double (&a)[K], const double (&b)[K],
                    const double (&c)[K], double (&out)[K]) {
  static_assert(K >= 2 && K <= 4, "fused ops: k = 2..4");
  if constexpr (K == 2) {
    double p, e;
    two_prod(b[0], c[0], p, e);
    double t[5] = {a[0], -p, a[1], -dadd(dmul(b[0], c[1]), dmul(b[1], c[0])), -e};
    renorm<5, 2>(t, out);
  } else if constexpr (K == 3) {
    double p00, e00, p01, e01, p10, e10;
    two_prod(b[0], c[0], p00, e00);
    two_prod(b[0], c[1], p01, e01);
    two_prod(b[1], c[0], p10, e10);
    const double top = dadd(dadd(dmul(b[0], c[2]), dmul(b[1], c[1])), dmul(b[2], c[0]));
    double t[10] = {a[0], -p00, a[1], -p01, -p10, -e00, a[2], -top, -e01, -e10};
    renorm<10, 3>(t, out);
  } else {
    double p00, e00, p01, e01, p10, e10, p02, e02, p11, e11, p20, e20;
    two_prod(b[0], c[0], p00, e00);
    two_prod(b[0], c[1], p01, e01);
    two_prod(b[1], c[0], p10, e10);
    two_prod(b[0], c[2], p02, e02);
    two_prod(b[1], c[1], p11, e11);
    two_prod(b[2], c[0], p20, e20);
    const double top = dadd(dadd(dadd(dmul(b[0], c[3]), dmul(b[1], c[2])), dmul(b[2], c[1])),
                            dmul(b[3], c[0]));
    double t[17] = {a[0], -p00, a[1], -p01, -p10, -e00, a[2], -p02, -p11,
                    -p20, -e01, -e10, a[3], -top, -e02, -e11, -e20};
    renorm<17, 4>(t, out);
  }
}

template <int K>
MPK_HD void fmul(const double (&a)[K], const double (&b)[K], double (&out)[K]) {
  static_assert(K >= 2 && K <= 4, "fused ops: k = 2..4");
  if constexpr (K == 2) {
    double p, e;
    two_prod(a[0], b[0], p, e);
    double t[3] = {p, dadd(dmul(a[0], b[1]), dmul(a[1], b[0])), e};
    renorm<3, 2>(t, out);
  } else if constexpr (K == 3) {
    double p00, e00, p01, e01, p10, e10;
    two_prod(a[0], b[0], p00, e00);
    two_prod(a[0], b[1], p01, e01);
    two_prod(a[1], b[0], p10, e10);
    const double top = dadd(dadd(dmul(a[0], b[2]), dmul(a[1], b[1])), dmul(a[2], b[0]));
    double t[7] = {p00, p01, p10, e00, top, e01, e10};
    renorm<7, 3>(t, out);
  } else {
    double p00, e00, p01, e01, p10, e10, p02, e02, p11, e11, p20, e20;
    two_prod(a[0], b[0], p00, e00);
    two_prod(a[0], b[1], p01, e01);
    two_prod(a[1], b[0], p10, e10);
    two_prod(a[0], b[2], p02, e02);
    two_prod(a[1], b[1], p11, e11);
    two_prod(a[2], b[0], p20, e20);
    const double top = dadd(dadd(dadd(dmul(a[0], b[3]), dmul(a[1], b[2])), dmul(a[2], b[1])),
                            dmul(a[3], b[0]));
    double t[13] = {p00, p01, p10, e00, p02, p11, p20, e01, e10, top, e02, e11, e20};
    renorm<13, 4>(t, out);
  }
}

// complex fused a - b*c on (re, im) component arrays (_mcfast.py:195-377):
// the real and imaginary parts are each ONE renormalisation of their
// partial-product term list (cmulsub2/3; k = 4 via _rmulsub4_pair / _pair2)
template <int K>
MPK_HD void fcmulsub(const double (&ar)[K], const double (&ai)[K],
                     const double (&br)[K], const double (&bi)[K],
                     const double (&cr)[K], const double (&ci)[K],
                     double (&orr)[K], double (&oi)[K]) {
  static_assert(K >= 2 && K <= 4, "fused ops: k = 2..4");
  if constexpr (K == 2) {
    double p1, e1, p2, e2, p3, e3, p4, e4;
    two_prod(br[0], cr[0], p1, e1);
    two_prod(bi[0], ci[0], p2, e2);
    const double tr = dadd(-dadd(dmul(br[0], cr[1]), dmul(br[1], cr[0])),
                           dadd(dmul(bi[0], ci[1]), dmul(bi[1], ci[0])));
    double t1[7] = {ar[0], -p1, p2, ar[1], tr, -e1, e2};
    renorm<7, 2>(t1, orr);
    two_prod(br[0], ci[0], p3, e3);
    two_prod(bi[0], cr[0], p4, e4);
    const double ti = -dadd(dadd(dadd(dmul(br[0], ci[1]), dmul(br[1], ci[0])), dmul(bi[0], cr[1])),
                            dmul(bi[1], cr[0]));
    double t2[7] = {ai[0], -p3, -p4, ai[1], ti, -e3, -e4};
    renorm<7, 2>(t2, oi);
  } else if constexpr (K == 3) {
    double q00, f00, q01, f01, q10, f10, s00, g00, s01, g01, s10, g10;
    two_prod(br[0], cr[0], q00, f00);
    two_prod(br[0], cr[1], q01, f01);
    two_prod(br[1], cr[0], q10, f10);
    two_prod(bi[0], ci[0], s00, g00);
    two_prod(bi[0], ci[1], s01, g01);
    two_prod(bi[1], ci[0], s10, g10);
    const double tr = dadd(-dadd(dadd(dmul(br[0], cr[2]), dmul(br[1], cr[1])), dmul(br[2], cr[0])),
                           dadd(dadd(dmul(bi[0], ci[2]), dmul(bi[1], ci[1])), dmul(bi[2], ci[0])));
    double t1[16] = {ar[0], -q00, s00, ar[1], -q01, -q10, s01, s10,
                     -f00, g00, ar[2], tr, -f01, -f10, g01, g10};
    renorm<16, 3>(t1, orr);
    two_prod(br[0], ci[0], q00, f00);
    two_prod(br[0], ci[1], q01, f01);
    two_prod(br[1], ci[0], q10, f10);
    two_prod(bi[0], cr[0], s00, g00);
    two_prod(bi[0], cr[1], s01, g01);
    two_prod(bi[1], cr[0], s10, g10);
    const double ti =
        -dadd(dadd(dadd(dadd(dadd(dmul(br[0], ci[2]), dmul(br[1], ci[1])), dmul(br[2], ci[0])),
                        dmul(bi[0], cr[2])),
                   dmul(bi[1], cr[1])),
              dmul(bi[2], cr[0]));
    double t2[16] = {ai[0], -q00, -s00, ai[1], -q01, -q10, -s01, -s10,
                     -f00, -g00, ai[2], ti, -f01, -f10, -g01, -g10};
    renorm<16, 3>(t2, oi);
  } else {
    // re = a_r - br*cr + bi*ci (pair), im = a_i - br*ci - bi*cr (pair2)
    auto pair = [](const double (&a)[4], const double (&b)[4], const double (&c)[4],
                   const double (&d)[4], const double (&e)[4], double sgn,
                   double (&o)[4]) {
      double p00, f00, p01, f01, p10, f10, p02, f02, p11, f11, p20, f20;
      double q00, g00, q01, g01, q10, g10, q02, g02, q11, g11, q20, g20;
      two_prod(b[0], c[0], p00, f00);
      two_prod(b[0], c[1], p01, f01);
      two_prod(b[1], c[0], p10, f10);
      two_prod(b[0], c[2], p02, f02);
      two_prod(b[1], c[1], p11, f11);
      two_prod(b[2], c[0], p20, f20);
      two_prod(d[0], e[0], q00, g00);
      two_prod(d[0], e[1], q01, g01);
      two_prod(d[1], e[0], q10, g10);
      two_prod(d[0], e[2], q02, g02);
      two_prod(d[1], e[1], q11, g11);
      two_prod(d[2], e[0], q20, g20);
      const double sb = dadd(dadd(dadd(dmul(b[0], c[3]), dmul(b[1], c[2])), dmul(b[2], c[1])),
                             dmul(b[3], c[0]));
      const double sd = dadd(dadd(dadd(dmul(d[0], e[3]), dmul(d[1], e[2])), dmul(d[2], e[1])),
                             dmul(d[3], e[0]));
      // sgn = +1: -(sb) + (sd); sgn = -1: -(sb) - (sd)
      const double top = sgn > 0 ? dadd(-sb, sd) : dsub(-sb, sd);
      const double s = sgn;  // q / g terms enter with this sign
      double t[29] = {a[0], -p00, s * q00, a[1], -p01, -p10, s * q01, s * q10, -f00, s * g00,
                      a[2], -p02, -p11, -p20, s * q02, s * q11, s * q20, -f01, -f10,
                      s * g01, s * g10, a[3], top, -f02, -f11, -f20, s * g02, s * g11,
                      s * g20};
      renorm<29, 4>(t, o);
    };
    double a4r[4], a4i[4], b4r[4], b4i[4], c4r[4], c4i[4], o4r[4], o4i[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a4r[q] = ar[q]; a4i[q] = ai[q]; b4r[q] = br[q]; b4i[q] = bi[q];
      c4r[q] = cr[q]; c4i[q] = ci[q];
    }
    pair(a4r, b4r, c4r, b4i, c4i, 1.0, o4r);
    pair(a4i, b4r, c4i, b4i, c4r, -1.0, o4i);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      orr[q] = o4r[q];
      oi[q] = o4i[q];
    }
  }
}

}  // namespace mpk
