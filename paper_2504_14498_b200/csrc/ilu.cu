// ilu.cu -- sync-free binary64 ILU(0) factorization and sweeps (see ilu.cuh)
#include <climits>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

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
  // each elimination step waits only for its own pivot row, so the work on
  // early L entries overlaps the wait for later ones
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

// Real rows of at most kFactRow entries: the row lives in registers / local
// memory for the whole elimination and each pivot row's upper part is
// fetched in independent batches (the merge-walk of factor_row issues one
// dependent L2 load per entry).  Same operations in the same order.
constexpr int kFactRow = 32;
constexpr int kFactBatch = 8;

// The wait for pivot row kc is an acquire load of its completion flag (its
// factors were written before the producer's release store), and everything
// that does not depend on the pivot row's VALUES -- its extent and the column
// indices of its upper part, which belong to the static pattern -- is loaded
// before the wait, so that one L2 round trip (the diagonal and the first
// batch of upper values, independent loads) separates "row kc is done" from
// the division: the per-level latency of a deep DAG (cfg4: 6142 levels).
__device__ __forceinline__ int ld_acquire_i(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ void factor_row_local(const FactorArgs &a, int i) {
  const int lo = a.rp[i], hi = a.rp[i + 1], d = a.dp[i];
  const int len = hi - lo;
  int cols[kFactRow];
  double vals[kFactRow];
  for (int q = 0; q < len; ++q) {
    cols[q] = a.ci[lo + q];
    vals[q] = __ldcg(&a.lu[lo + q]);
  }
  const int nl = d - lo;  // L entries
  int uks[kFactRow], kends[kFactRow];
  for (int t = 0; t < nl; ++t) {
    uks[t] = a.dp[cols[t]];
    kends[t] = a.rp[cols[t] + 1];
  }
  const bool byval = a.pub != nullptr;
  const int sent_hi = (int)(kSentBits >> 32);
  for (int t = 0; t < nl; ++t) {
    const int kc = cols[t];
    const int uk = uks[t], kend = kends[t];
    int cb[kFactBatch];
#pragma unroll
    for (int b = 0; b < kFactBatch; ++b) {
      const int s = uk + 1 + b;
      cb[b] = s < kend ? a.ci[s] : INT_MAX;
    }
    double ukk, ub[kFactBatch];
    if (byval) {
      // the pivot row's diagonal and first batch arrive with the poll itself
      for (;;) {
        ukk = ld_relaxed(a.pub + uk);
        bool ready = __double2hiint(ukk) != sent_hi;
#pragma unroll
        for (int b = 0; b < kFactBatch; ++b) {
          const int s = uk + 1 + b;
          ub[b] = s < kend ? ld_relaxed(a.pub + s) : 0.0;
          ready = ready && (__double2hiint(ub[b]) != sent_hi);
        }
        if (ready) break;
        __nanosleep(20);
      }
    } else {
      while (ld_acquire_i(&a.rowflag[kc]) == 0) __nanosleep(20);
      ukk = __ldcg(&a.lu[uk]);
#pragma unroll
      for (int b = 0; b < kFactBatch; ++b) {
        const int s = uk + 1 + b;
        ub[b] = s < kend ? __ldcg(&a.lu[s]) : 0.0;
      }
    }
    const double l = ddiv(vals[t], ukk);
    vals[t] = l;
    int q = t + 1;
    for (int s0 = uk + 1;;) {
#pragma unroll
      for (int b = 0; b < kFactBatch; ++b) {
        const int col = cb[b];
        if (col == INT_MAX) break;
        while (q < len && cols[q] < col) ++q;
        if (q < len && cols[q] == col) vals[q] = dsub(vals[q], dmul(l, ub[b]));
      }
      s0 += kFactBatch;
      if (s0 >= kend) break;
#pragma unroll
      for (int b = 0; b < kFactBatch; ++b) {
        const int s = s0 + b;
        cb[b] = s < kend ? a.ci[s] : INT_MAX;
        ub[b] = 0.0;
        if (s < kend) {
          if (byval) {  // the diagonal was seen; the rest of the row follows at once
            double v = ld_relaxed(a.pub + s);
            while (__double2hiint(v) == sent_hi) v = ld_relaxed(a.pub + s);
            ub[b] = v;
          } else {
            ub[b] = __ldcg(&a.lu[s]);
          }
        }
      }
    }
  }
  bool fin = true;
  if (byval) {  // publish the diagonal and the upper part first (consumers wait on them)
    for (int q = d - lo; q < len; ++q) {
      const double v = vals[q];
      const double w = __double2hiint(v) == sent_hi
                           ? __longlong_as_double((long long)kQNaNBits) : v;
      asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(a.pub + lo + q), "d"(w)
                   : "memory");
    }
  }
  for (int q = 0; q < len; ++q) {
    __stcg(&a.lu[lo + q], vals[q]);
    fin = fin && isfin(vals[q]);
  }
  if (vals[d - lo] == 0.0) atomicMin(a.bad_row, i);
  if (!fin) atomicOr(a.nonfinite, 1);
  if (!byval) st_release_i(&a.rowflag[i], 1);
}

template <bool CX>
__global__ void __launch_bounds__(kBlock) factor_kernel(FactorArgs a) {
  const int lane = threadIdx.x & 31;
  const int nt = a.ord ? a.nt : a.n;
  for (;;) {
    const int base = grab_ticket(a.tick);
    if (base >= nt) break;
    const int t = base + lane;
    const int row = t < nt ? (a.ord ? a.ord[t] : t) : -1;
    if (row >= 0) {
      if (!CX && a.rp[row + 1] - a.rp[row] <= kFactRow)
        factor_row_local(a, row);
      else
        factor_row<CX>(a, row);
    }
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

// Loads of values published by other threads of the same kernel: volatile
// (L1-bypassing, system scope) or relaxed at gpu scope.
template <bool CX, bool REL>
__device__ __forceinline__ void ldpub(const double *buf, int j, double &r,
                                      double &m) {
  if constexpr (CX) {
    const double2 *p = reinterpret_cast<const double2 *>(buf) + j;
    const double2 w = REL ? ld_relaxed2(p) : ld_volatile2(p);
    r = w.x;
    m = w.y;
  } else {
    r = REL ? ld_relaxed(buf + j) : ld_volatile(buf + j);
    m = 0.0;
  }
}

template <bool CX, bool REL>
__device__ __forceinline__ void pollv(const double *buf, int j, double &r,
                                      double &m) {
  ldpub<CX, REL>(buf, j, r, m);
  while (is_sent(r) || (CX && is_sent(m))) {
    __nanosleep(20);
    ldpub<CX, REL>(buf, j, r, m);
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

// acc -= val[q] * buf[col[q]] for q = lo..hi-1 IN ORDER (the reference's
// per-row accumulation order).  PREF > 1 fetches the dependency values in
// batches of PREF independent loads before the ordered chain consumes them
// (a value still carrying the sentinel is re-polled individually).
template <bool CX, bool CONJ, int PREF, bool REL>
__device__ __forceinline__ void chain(double &ar, double &ai, const int *col,
                                      const double *val, const double *buf,
                                      int lo, int hi) {
  if constexpr (PREF == 1) {
    for (int p = lo; p < hi; ++p) {
      double vr, vi, lr, li;
      pollv<CX, REL>(buf, col[p], vr, vi);
      ldval<CX>(val, p, lr, li);
      mulsub<CX, CONJ>(ar, ai, lr, li, vr, vi);
    }
  } else {
    for (int p0 = lo; p0 < hi; p0 += PREF) {
      double vr[PREF], vi[PREF];
#pragma unroll
      for (int q = 0; q < PREF; ++q) {
        vr[q] = vi[q] = 0.0;
        if (p0 + q < hi) ldpub<CX, REL>(buf, col[p0 + q], vr[q], vi[q]);
      }
#pragma unroll
      for (int q = 0; q < PREF; ++q) {
        if (p0 + q < hi) {
          if (is_sent(vr[q]) || (CX && is_sent(vi[q])))
            pollv<CX, REL>(buf, col[p0 + q], vr[q], vi[q]);
          double lr, li;
          ldval<CX>(val, p0 + q, lr, li);
          mulsub<CX, CONJ>(ar, ai, lr, li, vr[q], vi[q]);
        }
      }
    }
  }
}

// _sweep_forward ilu.py:322-331
template <bool CX, int PREF, bool REL>
__device__ void fwd_row(const SweepArgs &a, int i) {
  double ar, ai;
  load_in<CX>(a, i, ar, ai);
  chain<CX, false, PREF, REL>(ar, ai, a.ci, a.lu, a.y, a.rp[i], a.dp[i]);
  publish<CX>(a.y, i, ar, ai);
}

// _sweep_backward ilu.py:334-343
template <bool CX, int PREF, bool REL>
__device__ void bwd_row(const SweepArgs &a, int i) {
  double ar, ai;
  pollv<CX, REL>(a.y, i, ar, ai);
  const int d = a.dp[i], hi = a.rp[i + 1];
  chain<CX, false, PREF, REL>(ar, ai, a.ci, a.lu, a.z, d + 1, hi);
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
template <bool CX, int PREF, bool REL>
__device__ void fwd_row_adj(const SweepArgs &a, int c) {
  double ar, ai;
  load_in<CX>(a, c, ar, ai);
  chain<CX, true, PREF, REL>(ar, ai, a.ut_ci, a.ut_val, a.y, a.ut_rp[c],
                             a.ut_rp[c + 1]);
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
template <bool CX, int PREF, bool REL>
__device__ void bwd_row_adj(const SweepArgs &a, int c) {
  double ar, ai;
  pollv<CX, REL>(a.y, c, ar, ai);
  chain<CX, true, PREF, REL>(ar, ai, a.lt_ci, a.lt_val, a.z, a.lt_rp[c],
                             a.lt_rp[c + 1]);
  if (!isfin(ar) || !isfin(ai)) atomicOr(a.err, 1);
  publish<CX>(a.z, c, ar, ai);
}

template <bool CX, bool ADJ, int PREF, bool REL>
__global__ void __launch_bounds__(kBlock) sweep_kernel(SweepArgs a) {
  const int lane = threadIdx.x & 31;
  // solve already stopped (the flag may flip while the grid launches, e.g.
  // from a finalize on a side stream): skip the work but still take part in
  // the exit count, so the ticket is reset for the next launch
  {
    int d = 0;
    if (lane == 0 && a.done) d = ld_volatile_i(a.done);
    if (__shfl_sync(kFull, d, 0)) {
      exit_protocol(a.tick);
      return;
    }
  }
  const int n = a.n;
  for (;;) {
    const int base = grab_ticket(a.tick);
    if (base >= 2 * n) break;
    const int t = base + lane;
    if (t < n) {
      const int row = a.ord_f ? a.ord_f[t] : t;
      if constexpr (ADJ)
        fwd_row_adj<CX, PREF, REL>(a, row);
      else
        fwd_row<CX, PREF, REL>(a, row);
    } else if (t < 2 * n) {
      const int row = a.ord_b ? a.ord_b[t - n] : 2 * n - 1 - t;
      if constexpr (ADJ)
        bwd_row_adj<CX, PREF, REL>(a, row);
      else
        bwd_row<CX, PREF, REL>(a, row);
    }
  }
  exit_protocol(a.tick);
}

// ---------------------------------------------------------------------
// Single-CTA level-synchronous sweeps for systems whose binary64 vector
// fits in shared memory (n*8 B real, n*16 B complex <= 227 KB): the whole
// forward/backward solve runs in ONE thread block; the vector lives in
// SMEM (z overwrites y in place: backward row i reads its own y_i first,
// and only z_j of earlier backward levels), levels are separated by
// __syncthreads (~tens of ns) instead of L2 round trips, and each row's
// entries are fetched from L2 in independent batches.  Per-row operation
// order is the reference's, so results are bitwise identical.
// ---------------------------------------------------------------------
constexpr int kSmemThreads = 1024;

template <bool CX>
__device__ __forceinline__ void sm_ld(const double *sv, int j, double &r,
                                      double &m) {
  if constexpr (CX) {
    const double2 w = reinterpret_cast<const double2 *>(sv)[j];
    r = w.x;
    m = w.y;
  } else {
    r = sv[j];
    m = 0.0;
  }
}
template <bool CX>
__device__ __forceinline__ void sm_st(double *sv, int j, double r, double m) {
  if constexpr (CX)
    reinterpret_cast<double2 *>(sv)[j] = make_double2(r, m);
  else
    sv[j] = r;
}

// acc -= val[q] * sv[col[q]], q = lo..hi-1 in order, entries batch-loaded
template <bool CX, bool CONJ>
__device__ __forceinline__ void sm_chain(double &ar, double &ai,
                                         const int *col, const double *val,
                                         const double *sv, int lo, int hi) {
  for (int p0 = lo; p0 < hi; p0 += 8) {
    int c[8];
    double lr[8], li[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      c[q] = 0;
      lr[q] = li[q] = 0.0;
      if (p0 + q < hi) {
        c[q] = col[p0 + q];
        ldval<CX>(val, p0 + q, lr[q], li[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (p0 + q < hi) {
        double vr, vi;
        sm_ld<CX>(sv, c[q], vr, vi);
        mulsub<CX, CONJ>(ar, ai, lr[q], li[q], vr, vi);
      }
    }
  }
}

template <bool CX, bool ADJ>
__global__ void __launch_bounds__(kSmemThreads, 1)
    sweep_smem_kernel(SweepArgs a) {
  if (a.done && *a.done) return;
  extern __shared__ double sv[];
  const int tid = threadIdx.x;
  for (int L = 0; L < a.nlev_f; ++L) {
    const int r1 = a.lev_f[L + 1];
    for (int r = a.lev_f[L] + tid; r < r1; r += kSmemThreads) {
      const int i = a.ord_f[r];
      double ar, ai;
      load_in<CX>(a, i, ar, ai);
      if constexpr (!ADJ) {
        sm_chain<CX, false>(ar, ai, a.ci, a.lu, sv, a.rp[i], a.dp[i]);
        sm_st<CX>(sv, i, ar, ai);
      } else {
        sm_chain<CX, true>(ar, ai, a.ut_ci, a.ut_val, sv, a.ut_rp[i],
                           a.ut_rp[i + 1]);
        double dr, di, qr, qi;
        ldval<CX>(a.lu, a.dp[i], dr, di);
        if constexpr (CX) {
          py_cdiv(ar, ai, dr, -di, qr, qi);
        } else {
          qr = ddiv(ar, dr);
          qi = 0.0;
        }
        sm_st<CX>(sv, i, qr, qi);
      }
    }
    __syncthreads();
  }
  bool bad = false;
  for (int L = 0; L < a.nlev_b; ++L) {
    const int r1 = a.lev_b[L + 1];
    for (int r = a.lev_b[L] + tid; r < r1; r += kSmemThreads) {
      const int i = a.ord_b[r];
      double ar, ai, qr, qi;
      sm_ld<CX>(sv, i, ar, ai);
      if constexpr (!ADJ) {
        const int d = a.dp[i];
        sm_chain<CX, false>(ar, ai, a.ci, a.lu, sv, d + 1, a.rp[i + 1]);
        double dr, di;
        ldval<CX>(a.lu, d, dr, di);
        if constexpr (CX) {
          py_cdiv(ar, ai, dr, di, qr, qi);
        } else {
          qr = ddiv(ar, dr);
          qi = 0.0;
        }
      } else {
        sm_chain<CX, true>(ar, ai, a.lt_ci, a.lt_val, sv, a.lt_rp[i],
                           a.lt_rp[i + 1]);
        qr = ar;
        qi = ai;
      }
      bad = bad || !isfin(qr) || !isfin(qi);
      sm_st<CX>(sv, i, qr, qi);
      if constexpr (CX)
        reinterpret_cast<double2 *>(a.z)[i] = make_double2(qr, qi);
      else
        a.z[i] = qr;
    }
    __syncthreads();
  }
  if (bad) atomicOr(a.err, 1);
}

// ---------------------------------------------------------------------
// Prefetched single-CTA sweep over level-ordered sweep matrices.  Row
// descriptors, the first kPE entries, the right-hand side and the divisor
// of the NEXT level are loaded into registers before the current level is
// computed, so a level's critical path is SMEM reads + the FP64 chain +
// one __syncthreads, not a chain of dependent L2 loads.
// ---------------------------------------------------------------------
constexpr int kPE = 6;             // entries per row held in registers
constexpr int kMatsThreads = 768;  // 85 registers/thread

// Entries + divisor of one row, fetched one level ahead.
template <bool CX>
struct RowEnt {
  int col[kPE];
  double vr[kPE], vi[CX ? kPE : 1];
  double dr, di[CX ? 1 : 1];
};

template <bool CX, bool ADJ>
__device__ __forceinline__ void ent_load(RowEnt<CX> &E, const SweepPhase &ph,
                                         const int4 d, int r, bool fwd) {
#pragma unroll
  for (int q = 0; q < kPE; ++q) {
    int c = 0;
    double lr = 0.0, li = 0.0;
    if (q < d.z) {
      c = ph.col[d.y + q];
      ldval<CX>(ph.val, d.y + q, lr, li);
    }
    E.col[q] = c;
    E.vr[q] = lr;
    if constexpr (CX) E.vi[q] = li;
  }
  double d0 = 1.0, d1 = 0.0;
  if (fwd == ADJ && r >= 0) ldval<CX>(ph.dval, r, d0, d1);
  E.dr = d0;
  E.di[0] = d1;
}

// Process one row: acc = (fwd ? rhs : y_i) - sum val*v[col] in order,
// then the divisor (forward adjoint: conj(U_ii); backward plain: U_ii).
template <bool CX, bool ADJ>
__device__ __forceinline__ void row_run(const int4 d, const RowEnt<CX> &E,
                                        const SweepPhase &ph,
                                        const SweepArgs &a, double *sv,
                                        bool fwd, bool &bad) {
  const int i = d.x;
  double ar, ai;
  sm_ld<CX>(sv, i, ar, ai);  // forward: rhs preloaded; backward: y_i
#pragma unroll
  for (int q = 0; q < kPE; ++q) {
    if (q < d.z) {
      double vr, vi;
      sm_ld<CX>(sv, E.col[q], vr, vi);
      if constexpr (CX)
        mulsub<CX, ADJ>(ar, ai, E.vr[q], E.vi[q], vr, vi);
      else
        mulsub<CX, ADJ>(ar, ai, E.vr[q], 0.0, vr, vi);
    }
  }
  for (int e = d.y + kPE; e < d.y + d.z; ++e) {
    double lr, li, vr, vi;
    ldval<CX>(ph.val, e, lr, li);
    sm_ld<CX>(sv, ph.col[e], vr, vi);
    mulsub<CX, ADJ>(ar, ai, lr, li, vr, vi);
  }
  double qr = ar, qi = ai;
  if (fwd == ADJ) {
    if constexpr (CX) {
      py_cdiv(ar, ai, E.dr, ADJ ? -E.di[0] : E.di[0], qr, qi);
    } else {
      qr = ddiv(ar, E.dr);
    }
  }
  sm_st<CX>(sv, i, qr, qi);
  if (!fwd) {
    bad = bad || !isfin(qr) || !isfin(qi);
    if constexpr (CX)
      reinterpret_cast<double2 *>(a.z)[i] = make_double2(qr, qi);
    else
      a.z[i] = qr;
  }
}

// global level index g -> (phase, level) helpers over [fwd levels | bwd levels]
struct GLev {
  const int *fl, *bl;
  int nf, nb;
  __device__ __forceinline__ bool fwd(int g) const { return g < nf; }
  __device__ __forceinline__ int lo(int g) const {
    return g < nf ? fl[g] : bl[g - nf];
  }
  __device__ __forceinline__ int hi(int g) const {
    return g < nf ? fl[g + 1] : bl[g - nf + 1];
  }
};

template <bool CX, bool ADJ>
__global__ void __launch_bounds__(kMatsThreads, 1)
    sweep_mats_kernel(SweepArgs a, SweepMats m) {
  if (a.done && *a.done) return;
  extern __shared__ double sv[];
  const int tid = threadIdx.x;
  const int n = a.n, nf = m.fwd.nlev, nb = m.bwd.nlev, nl = nf + nb;
  int *fl = reinterpret_cast<int *>(sv + (size_t)n * (CX ? 2 : 1));
  int *bl = fl + nf + 1;
  const int T = blockDim.x;  // sized to the widest level (<= kMatsThreads)
  for (int t = tid; t <= nf; t += T) fl[t] = m.fwd.lev[t];
  for (int t = tid; t <= nb; t += T) bl[t] = m.bwd.lev[t];
  // forward right-hand side (demoted input) preloaded into the vector slots
  for (int i = tid; i < n; i += T) {
    double r, mm;
    load_in<CX>(a, i, r, mm);
    sm_st<CX>(sv, i, r, mm);
  }
  __syncthreads();
  const GLev gl{fl, bl, nf, nb};
  bool bad = false;
  // pipeline registers: descriptor of levels g+1, g+2 and entries of g, g+1
  const int4 none = make_int4(0, 0, 0, -1);
  auto desc_at = [&](int g) -> int4 {
    if (g >= nl) return none;
    const int r = gl.lo(g) + tid;
    if (r >= gl.hi(g)) return none;
    int4 d = (gl.fwd(g) ? m.fwd : m.bwd).desc[r];
    d.w = r;
    return d;
  };
  int4 d0 = desc_at(0), d1 = desc_at(1), d2;
  RowEnt<CX> e0, e1;
  if (d0.w >= 0) ent_load<CX, ADJ>(e0, gl.fwd(0) ? m.fwd : m.bwd, d0, d0.w, gl.fwd(0));
  for (int g = 0; g < nl; ++g) {
    const bool fwd = gl.fwd(g);
    const SweepPhase &ph = fwd ? m.fwd : m.bwd;
    // stage 1: descriptor two levels ahead; stage 2: entries one ahead
    d2 = desc_at(g + 2);
    if (d1.w >= 0)
      ent_load<CX, ADJ>(e1, gl.fwd(g + 1) ? m.fwd : m.bwd, d1, d1.w,
                        gl.fwd(g + 1));
    if (d0.w >= 0) row_run<CX, ADJ>(d0, e0, ph, a, sv, fwd, bad);
    const int s = gl.lo(g), e = gl.hi(g);
    for (int r = s + tid + T; r < e; r += T) {
      int4 dx = ph.desc[r];
      RowEnt<CX> ex;
      ent_load<CX, ADJ>(ex, ph, dx, r, fwd);
      row_run<CX, ADJ>(dx, ex, ph, a, sv, fwd, bad);
    }
    __syncthreads();
    d0 = d1;
    e0 = e1;
    d1 = d2;
  }
  if (bad) atomicOr(a.err, 1);
}

// Level-synchronous single-CTA factorization (small n): rows of one level
// are independent; __syncthreads orders the global-memory factor values
// between levels within the block, so no per-row flags are needed.
template <bool CX>
__device__ void factor_row_nowait(const FactorArgs &a, int i) {
  const int lo = a.rp[i], hi = a.rp[i + 1], d = a.dp[i];
  double2 *lu2 = reinterpret_cast<double2 *>(a.lu);
  for (int t = lo; t < d; ++t) {
    const int kc = a.ci[t];
    const int uk = a.dp[kc];
    const int kend = a.rp[kc + 1];
    if constexpr (!CX) {
      const double l = ddiv(a.lu[t], a.lu[uk]);
      a.lu[t] = l;
      int q = t + 1;
      for (int s = uk + 1; s < kend; ++s) {
        const int col = a.ci[s];
        while (q < hi && a.ci[q] < col) ++q;
        if (q < hi && a.ci[q] == col) a.lu[q] = dsub(a.lu[q], dmul(l, a.lu[s]));
      }
    } else {
      const double2 at = lu2[t];
      const double2 ukk = lu2[uk];
      double lr, li;
      py_cdiv(at.x, at.y, ukk.x, ukk.y, lr, li);
      lu2[t] = make_double2(lr, li);
      int q = t + 1;
      for (int s = uk + 1; s < kend; ++s) {
        const int col = a.ci[s];
        while (q < hi && a.ci[q] < col) ++q;
        if (q < hi && a.ci[q] == col) {
          const double2 u = lu2[s];
          double pr, pi;
          py_cmul(lr, li, u.x, u.y, pr, pi);
          const double2 v = lu2[q];
          lu2[q] = make_double2(dsub(v.x, pr), dsub(v.y, pi));
        }
      }
    }
  }
  bool zero, fin = true;
  if constexpr (!CX) {
    zero = a.lu[d] == 0.0;
    for (int p = lo; p < hi; ++p) fin = fin && isfin(a.lu[p]);
  } else {
    zero = (lu2[d].x == 0.0) && (lu2[d].y == 0.0);
    for (int p = lo; p < hi; ++p) fin = fin && isfin(lu2[p].x) && isfin(lu2[p].y);
  }
  if (zero) atomicMin(a.bad_row, i);
  if (!fin) atomicOr(a.nonfinite, 1);
}

template <bool CX>
__global__ void __launch_bounds__(kSmemThreads, 1)
    factor_smem_kernel(FactorArgs a) {
  for (int L = 0; L < a.nlev; ++L) {
    const int r1 = a.lev[L + 1];
    for (int r = a.lev[L] + threadIdx.x; r < r1; r += kSmemThreads)
      factor_row_nowait<CX>(a, a.ord[r]);
    __syncthreads();
  }
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

// ---------------------------------------------------------------------
// cluster sweep (ilu.cuh CSweep): DSMEM-resident vector, TMA-bulk staged
// entries, one cluster barrier per level
// ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_map(uint32_t a, uint32_t rank) {
  uint32_t o;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(rank));
  return o;
}
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// values of earlier levels are immutable within a level: plain (reorderable)
// loads; the barrier asm above carries the memory clobber
__device__ __forceinline__ double cl_ld1(uint32_t a) {
  double v;
  asm("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void cl_ld2(uint32_t a, double &x, double &y) {
  asm("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ void cl_st1(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_st2(uint32_t a, double x, double y) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x),
               "d"(y)
               : "memory");
}
__device__ __forceinline__ int cl_ldi(uint32_t a) {
  int v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t *b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)),
               "r"(cnt)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "CSW_WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra CSW_WAIT%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src,
                                         uint32_t bytes, uint64_t *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

constexpr int kCsBatch = 16;  // entries whose loads are issued together

template <bool CX, bool ADJ>
__global__ void __launch_bounds__(1024, 1)
    csweep_kernel(SweepArgs a, CSweep p) {
  constexpr int ESZ = CX ? 16 : 8;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tid = threadIdx.x, T = blockDim.x;
  const uint32_t rank = cl_rank();
  const int C = p.C, nl = p.nl, nf = p.nf, NB = p.nbuf;
  const bool repl = p.repl != 0;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smraw);  // NB <= 8 mbarriers
  int *flag = reinterpret_cast<int *>(smraw + 64);
  int4 *seg = reinterpret_cast<int4 *>(smraw + 80);     // nl own segments
  unsigned char *q = smraw + 80 + (size_t)nl * 16;
  double *vec = reinterpret_cast<double *>(q);
  q += ((size_t)p.maxslots * ESZ + 15) / 16 * 16;
  unsigned char *stage = q;  // NB x maxseg
  const uint32_t vbase = smem_u32(vec);

  if (tid == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
    flag[0] = (a.done && *a.done) ? 1 : 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  for (int g = tid; g < nl; g += T) seg[g] = p.seg[(size_t)g * C + rank];
  // forward right-hand side (demoted input) preloaded into the slots: all
  // rows (replicated) or the own slots (distributed)
  const int s0 = repl ? 0 : p.slot_off[rank];
  const int s1 = repl ? a.n : p.slot_off[rank + 1];
  for (int s = s0 + tid; s < s1; s += T) {
    double r, m;
    load_in<CX>(a, repl ? s : p.slot_row[s], r, m);
    vec[(s - s0) * (CX ? 2 : 1)] = r;
    if constexpr (CX) vec[(s - s0) * 2 + 1] = m;
  }
  __syncthreads();
  // every CTA of the cluster is running and initialised; one uniform
  // decision on the solver's done flag (rank 0's read)
  cl_arrive();
  cl_wait();
  const bool skip = cl_ldi(cl_map(smem_u32(flag), 0)) != 0;
  if (skip) {
    cl_arrive();  // rank 0's flag must outlive the readers
    cl_wait();
    return;
  }
  auto issue = [&](int g) {
    const int b = g % NB;
    const int4 sg = seg[g];
    if (sg.y == 0) {
      mbar_arrive(&bar[b]);
      return;
    }
    mbar_arrive_tx(&bar[b], (uint32_t)sg.y);
    bulk_g2s(stage + (size_t)b * p.maxseg, p.stream + ((size_t)sg.x << 4),
             (uint32_t)sg.y, &bar[b]);
  };
  if (tid == 0)
    for (int g = 0; g < NB - 1 && g < nl; ++g) issue(g);
  // distributed: DSMEM address of a packed slot reference
  auto addr = [&](int pk) -> uint32_t {
    return cl_map(vbase + (uint32_t)(pk & 0xFFFFFF) * ESZ, (uint32_t)pk >> 24);
  };
  auto ldv = [&](int ref, double &r, double &m) {
    if (repl) {
      r = vec[ref * (CX ? 2 : 1)];
      m = CX ? vec[ref * 2 + 1] : 0.0;
    } else if constexpr (CX) {
      cl_ld2(addr(ref), r, m);
    } else {
      r = cl_ld1(addr(ref));
      m = 0.0;
    }
  };
#ifdef MPK_CSWEEP_PROF
  // per-level phase times of CTA 0 (diagnostic build only)
  long long *prof_sm = reinterpret_cast<long long *>(smraw + 72);
  if (tid == 0) prof_sm[0] = 0;
  long long pa[4] = {0, 0, 0, 0}, plast = clock64();
  __syncthreads();
#endif
  for (int g = 0; g < nl; ++g) {
    const int b = g % NB;
    mbar_wait(&bar[b], (uint32_t)((g / NB) & 1));
#ifdef MPK_CSWEEP_PROF
    const long long tq0 = clock64();
#endif
    const int4 sg = seg[g];
    const unsigned char *base = stage + (size_t)b * p.maxseg;
    const CSDesc *D = reinterpret_cast<const CSDesc *>(base);
    const int *refs = reinterpret_cast<const int *>(base + 16 * (size_t)sg.z);
    const double *vals = reinterpret_cast<const double *>(
        base + 16 * (size_t)sg.z + (((size_t)sg.w * 4 + 15) / 16) * 16);
    for (int r = tid; r < sg.z; r += T) {
      const CSDesc d = D[r];
      double ar, ai;
      ldv(d.row, ar, ai);
      for (int e = 0; e < d.cnt; e += kCsBatch) {
        double lr[kCsBatch], li[kCsBatch], vr[kCsBatch], vi[kCsBatch];
#pragma unroll
        for (int t = 0; t < kCsBatch; ++t) {
          vr[t] = vi[t] = lr[t] = li[t] = 0.0;
          if (e + t < d.cnt) {
            const int x = d.e0 + e + t;
            lr[t] = vals[x * (CX ? 2 : 1)];
            if constexpr (CX) li[t] = vals[2 * x + 1];
            ldv(refs[x], vr[t], vi[t]);
          }
        }
#pragma unroll
        for (int t = 0; t < kCsBatch; ++t)
          if (e + t < d.cnt) mulsub<CX, ADJ>(ar, ai, lr[t], li[t], vr[t], vi[t]);
      }
      double qr = ar, qi = ai;
      if (d.hasdiv & 1) {
        const int x = d.e0 + d.cnt;
        if constexpr (CX)
          py_cdiv(ar, ai, vals[2 * x], ADJ ? -vals[2 * x + 1] : vals[2 * x + 1], qr, qi);
        else
          qr = ddiv(ar, vals[x]);
      }
      if (repl) {
        // own copy + every peer's copy
        const uint32_t la = vbase + (uint32_t)d.row * ESZ;
        if constexpr (CX) {
          vec[2 * d.row] = qr;
          vec[2 * d.row + 1] = qi;
        } else {
          vec[d.row] = qr;
        }
        for (int k = 1; k < C; ++k) {
          const uint32_t rr = (rank + (uint32_t)k) % (uint32_t)C;
          if constexpr (CX)
            cl_st2(cl_map(la, rr), qr, qi);
          else
            cl_st1(cl_map(la, rr), qr);
        }
      } else if constexpr (CX) {
        cl_st2(addr(d.row), qr, qi);
      } else {
        cl_st1(addr(d.row), qr);
      }
    }
    // no global stores inside the level loop: the release of the cluster
    // barrier would have to wait for their acknowledgements
#ifdef MPK_CSWEEP_PROF
    const long long tq1 = clock64();
    atomicMax(reinterpret_cast<unsigned long long *>(prof_sm),
              (unsigned long long)(tq1 - tq0));
#endif
    cl_arrive();
#ifdef MPK_CSWEEP_PROF
    const long long tq2 = clock64();
#endif
    // buffer (g+NB-1)%NB was last read at level g-1, which every CTA finished
    if (tid == 0 && g + NB - 1 < nl) issue(g + NB - 1);
    cl_wait();
#ifdef MPK_CSWEEP_PROF
    if (tid == 0) {
      const long long tq3 = clock64();
      pa[0] += tq0 - plast;  // staging wait
      pa[1] += prof_sm[0];   // slowest thread's rows
      pa[2] += tq2 - tq1;    // arrive (release: drains the stores)
      pa[3] += tq3 - tq2;    // wait for the cluster
      plast = tq3;
      prof_sm[0] = 0;
    }
#endif
  }
#ifdef MPK_CSWEEP_PROF
  if (tid == 0 && rank == 0)
    printf("csweep prof C=%d repl=%d levels %d: staging %lld rows(max) %lld arrive %lld wait %lld cycles\n",
           C, p.repl, nl, pa[0], pa[1], pa[2], pa[3]);
#endif
  // every slot now holds the backward result z of its row: write out (the
  // replicated layout splits the rows over the CTAs) and check them
  bool bad = false;
  const int w0 = repl ? (int)rank : s0, w1 = repl ? a.n : s1, ws = repl ? C : 1;
  for (int s = w0 + tid * ws; s < w1; s += T * ws) {
    const int i = repl ? s : p.slot_row[s];
    const int v = repl ? s : s - s0;
    if constexpr (CX) {
      const double qr = vec[2 * v], qi = vec[2 * v + 1];
      bad = bad || !isfin(qr) || !isfin(qi);
      reinterpret_cast<double2 *>(a.z)[i] = make_double2(qr, qi);
    } else {
      const double qr = vec[v];
      bad = bad || !isfin(qr);
      a.z[i] = qr;
    }
  }
  if (bad) atomicOr(a.err, 1);
  // peers may still be pushing into this CTA's vector until they pass here
  cl_arrive();
  cl_wait();
}

// ---------------------------------------------------------------------
// dataflow cluster sweep (CSweep.dflow): replicated vector, no barrier per
// level.  Every CTA's copy starts as signalling-NaN sentinels; a row polls
// its dependencies in the LOCAL copy (volatile ld.shared, ~30 cycles) until
// the producer's push (st.shared::cluster) has replaced the sentinel, so
// the critical path is producer latency + DSMEM store latency per level.
// Deadlock-free: all threads of the cluster are resident, every thread
// processes its rows in level order, and a row only waits on lower levels.
// Cluster barriers: start (copies initialised), forward -> backward (all
// forward reads done; y_i of the own backward rows saved, copies reset) and
// end.  A producer warp streams the level segments through nbuf staging
// buffers (mbarriers full / empty) so warps of one CTA may be at different
// levels.
// ---------------------------------------------------------------------
__device__ __forceinline__ double lds_volatile(const double *p) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}

template <bool CX, bool ADJ>
__global__ void __launch_bounds__(1024, 1)
    dsweep_kernel(SweepArgs a, CSweep p) {
  constexpr int ESZ = CX ? 16 : 8;
  constexpr int BATCH = CX ? 4 : 8;
  constexpr int W = CX ? 2 : 1;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tid = threadIdx.x, T = blockDim.x, NC = T - 32;
  const uint32_t rank = cl_rank();
  const int C = p.C, nl = p.nl, nf = p.nf, NB = p.nbuf, n = a.n;
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);
  uint64_t *empty = full + 8;
  int *flag = reinterpret_cast<int *>(smraw + 128);
  int4 *seg = reinterpret_cast<int4 *>(smraw + 144);
  unsigned char *q = smraw + 144 + (size_t)nl * 16;
  double *vec = reinterpret_cast<double *>(q);
  q += ((size_t)n * ESZ + 15) / 16 * 16;
  double *init = reinterpret_cast<double *>(q);
  q += ((size_t)p.ninit * ESZ + 15) / 16 * 16;
  unsigned char *stage = q;
  const uint32_t vbase = smem_u32(vec);
  const double SENT = sent_val();

  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NC / 32);
    }
    flag[0] = (a.done && *a.done) ? 1 : 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  for (int g = tid; g < nl; g += T) seg[g] = p.seg[(size_t)g * C + rank];
  for (int s = tid; s < n * W; s += T) vec[s] = SENT;
  const int f0 = p.slot_off[rank], f1 = p.slot_off[rank + 1];
  for (int k = tid; k < f1 - f0; k += T) {
    double r, m;
    load_in<CX>(a, p.slot_row[f0 + k], r, m);
    init[k * W] = r;
    if constexpr (CX) init[k * 2 + 1] = m;
  }
  __syncthreads();
  cl_arrive();  // #1: every copy is initialised before anyone pushes
  cl_wait();
  const bool skip = cl_ldi(cl_map(smem_u32(flag), 0)) != 0;
  if (skip) {
    cl_arrive();
    cl_wait();
    return;
  }
  auto issue = [&](int g) {
    const int b = g % NB, k = g / NB;
    if (k > 0) mbar_wait(&empty[b], (uint32_t)((k - 1) & 1));
    const int4 sg = seg[g];
    if (sg.y == 0) {
      mbar_arrive(&full[b]);
      return;
    }
    mbar_arrive_tx(&full[b], (uint32_t)sg.y);
    bulk_g2s(stage + (size_t)b * p.maxseg, p.stream + ((size_t)sg.x << 4),
             (uint32_t)sg.y, &full[b]);
  };
  if (tid >= NC) {
    // producer warp: lane 0 streams the segments; the whole warp takes part
    // in the cluster barriers
    const int gb = nl < nf + NB - 1 ? nl : nf + NB - 1;
    if (tid == NC)
      for (int g = 0; g < gb; ++g) issue(g);
    __syncwarp();
    cl_arrive();  // #2 forward done
    cl_wait();
    cl_arrive();  // #3 copies reset
    cl_wait();
    if (tid == NC)
      for (int g = gb; g < nl; ++g) issue(g);
    __syncwarp();
    cl_arrive();  // #4 end
    cl_wait();
    return;
  }
  const int lane = tid & 31;
  for (int g = 0; g < nl; ++g) {
    if (g == nf) {
      // forward -> backward: everyone is done reading y; save y of the own
      // backward rows, reset the copy, and only then let pushes start
      cl_arrive();  // #2
      cl_wait();
      const int b0 = p.boff[rank], b1 = p.boff[rank + 1];
      for (int k = tid; k < b1 - b0; k += NC) {
        const int i = p.brow[b0 + k];
        init[k * W] = vec[i * W];
        if constexpr (CX) init[k * 2 + 1] = vec[i * 2 + 1];
      }
      named_bar(1, NC);
      for (int s = tid; s < n * W; s += NC) vec[s] = SENT;
      cl_arrive();  // #3
      cl_wait();
    }
    const int b = g % NB;
    mbar_wait(&full[b], (uint32_t)((g / NB) & 1));
    const int4 sg = seg[g];
    const unsigned char *base = stage + (size_t)b * p.maxseg;
    const CSDesc *D = reinterpret_cast<const CSDesc *>(base);
    const int *refs = reinterpret_cast<const int *>(base + 16 * (size_t)sg.z);
    const double *vals = reinterpret_cast<const double *>(
        base + 16 * (size_t)sg.z + (((size_t)sg.w * 4 + 15) / 16) * 16);
    for (int r = tid; r < sg.z; r += NC) {
      const CSDesc d = D[r];
      const int k = d.hasdiv >> 1;
      double ar = init[k * W], ai = CX ? init[k * 2 + 1] : 0.0;
      for (int e = 0; e < d.cnt; e += BATCH) {
        double lr[BATCH], li[BATCH], vr[BATCH], vi[BATCH];
        int jj[BATCH];
#pragma unroll
        for (int t = 0; t < BATCH; ++t) {
          vr[t] = vi[t] = lr[t] = li[t] = 0.0;
          jj[t] = 0;
          if (e + t < d.cnt) {
            const int x = d.e0 + e + t;
            lr[t] = vals[x * W];
            if constexpr (CX) li[t] = vals[2 * x + 1];
            jj[t] = refs[x];
            vr[t] = lds_volatile(vec + jj[t] * W);
            if constexpr (CX) vi[t] = lds_volatile(vec + jj[t] * 2 + 1);
          }
        }
#pragma unroll
        for (int t = 0; t < BATCH; ++t) {
          if (e + t < d.cnt) {
            while (is_sent(vr[t]) || (CX && is_sent(vi[t]))) {
              vr[t] = lds_volatile(vec + jj[t] * W);
              if constexpr (CX) vi[t] = lds_volatile(vec + jj[t] * 2 + 1);
            }
            mulsub<CX, ADJ>(ar, ai, lr[t], li[t], vr[t], vi[t]);
          }
        }
      }
      double qr = ar, qi = ai;
      if (d.hasdiv & 1) {
        const int x = d.e0 + d.cnt;
        if constexpr (CX)
          py_cdiv(ar, ai, vals[2 * x], ADJ ? -vals[2 * x + 1] : vals[2 * x + 1], qr, qi);
        else
          qr = ddiv(ar, vals[x]);
      }
      // a value carrying the sentinel pattern (only a copied input can) is
      // published as a quiet NaN, so no consumer waits on it forever
      qr = unsent(qr);
      if constexpr (CX) qi = unsent(qi);
      // push to every peer first, then the own copy
      const uint32_t la = vbase + (uint32_t)d.row * ESZ;
      for (int kk = 1; kk < C; ++kk) {
        const uint32_t rr = (rank + (uint32_t)kk) % (uint32_t)C;
        if constexpr (CX)
          cl_st2(cl_map(la, rr), qr, qi);
        else
          cl_st1(cl_map(la, rr), qr);
      }
      if constexpr (CX) {
        vec[2 * d.row] = qr;
        vec[2 * d.row + 1] = qi;
      } else {
        vec[d.row] = qr;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
  }
  if (nf == nl) {  // no backward phase (never for ILU): keep barriers paired
    cl_arrive();
    cl_wait();
    cl_arrive();
    cl_wait();
  }
  cl_arrive();  // #4: every z is pushed everywhere
  cl_wait();
  bool bad = false;
  for (int s = (int)rank + tid * C; s < n; s += NC * C) {
    if constexpr (CX) {
      const double qr = vec[2 * s], qi = vec[2 * s + 1];
      bad = bad || !isfin(qr) || !isfin(qi);
      reinterpret_cast<double2 *>(a.z)[s] = make_double2(qr, qi);
    } else {
      const double qr = vec[s];
      bad = bad || !isfin(qr);
      a.z[s] = qr;
    }
  }
  if (bad) atomicOr(a.err, 1);
}

__global__ void gather_csweep_kernel(const double *lu, CSweep p, int cx) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= p.nval) return;
  double *st = reinterpret_cast<double *>(p.stream);
  const int s = p.esrc[t];
  const long long o = p.eoff[t];
  if (cx) {
    const double2 v = reinterpret_cast<const double2 *>(lu)[s];
    st[o] = v.x;
    st[o + 1] = v.y;
  } else {
    st[o] = lu[s];
  }
}

// ---------------------------------------------------------------------
// ring sweep (ilu.cuh RSweep): vector resident in shared memory, rows and
// entries streamed by a producer warp through a ring of TMA-filled slots
// ---------------------------------------------------------------------


template <bool CX, bool ADJ>
__global__ void __launch_bounds__(1024, 1) rsweep_kernel(SweepArgs a, RSweep p) {
  constexpr int ESZ = CX ? 16 : 8;
  constexpr int kRsBatch = CX ? 4 : 8;  // entries whose loads issue together
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tid = threadIdx.x, T = blockDim.x, NC = T - 32;
  const int S = p.S, nch = p.nchunks, n = a.n;
  uint64_t *full = reinterpret_cast<uint64_t *>(smraw);
  uint64_t *empty = full + S;
  int *flag = reinterpret_cast<int *>(empty + S);
  int2 *tab = reinterpret_cast<int2 *>(smraw + ((16 * S + 16 + 15) / 16) * 16);
  double *vec = reinterpret_cast<double *>(
      reinterpret_cast<unsigned char *>(tab) + ((8 * (size_t)nch + 15) / 16) * 16);
  unsigned char *ring =
      reinterpret_cast<unsigned char *>(vec) + (((size_t)n * ESZ + 15) / 16) * 16;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC / 32);
    }
    flag[0] = (a.done && *a.done) ? 1 : 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  for (int c = tid; c < nch; c += T) {
    const RChunk m = p.chunks[c];
    tab[c] = make_int2((int)(m.off >> 4), m.bytes);
  }
  // forward right-hand side (demoted input) preloaded into the vector
  for (int i = tid; i < n; i += T) {
    double r, m;
    load_in<CX>(a, i, r, m);
    if constexpr (CX) {
      vec[2 * i] = r;
      vec[2 * i + 1] = m;
    } else {
      vec[i] = r;
    }
  }
  __syncthreads();
  if (flag[0]) return;  // uniform: read once, after the barrier
  if (tid >= NC) {
    // producer warp: lane 0 keeps up to S chunks in flight
    if (tid == NC) {
      for (int c = 0; c < nch; ++c) {
        const int s = c % S, k = c / S;
        if (k > 0) mbar_wait(&empty[s], (uint32_t)((k - 1) & 1));
        const int2 m = tab[c];
        mbar_arrive_tx(&full[s], (uint32_t)m.y);
        bulk_g2s(ring + (size_t)s * p.slot, p.stream + ((size_t)m.x << 4),
                 (uint32_t)m.y, &full[s]);
      }
    }
    return;
  }
  const int lane = tid & 31;
  for (int c = 0; c < nch; ++c) {
    const int s = c % S;
    mbar_wait(&full[s], (uint32_t)((c / S) & 1));
    const unsigned char *base = ring + (size_t)s * p.slot;
    const int4 h = *reinterpret_cast<const int4 *>(base);  // nrows nent end fwd
    const RDesc *D = reinterpret_cast<const RDesc *>(base + 16);
    const int *cols = reinterpret_cast<const int *>(base + 16 + 32 * (size_t)h.x);
    const double *vals = reinterpret_cast<const double *>(
        base + 16 + 32 * (size_t)h.x + (((size_t)h.y * 4 + 15) / 16) * 16);
    for (int r = tid; r < h.x; r += NC) {
      const RDesc d = D[r];
      double ar, ai = 0.0;
      if constexpr (CX) {
        ar = vec[2 * d.row];
        ai = vec[2 * d.row + 1];
      } else {
        ar = vec[d.row];
      }
      for (int e = 0; e < d.cnt; e += kRsBatch) {
        double lr[kRsBatch], li[kRsBatch], vr[kRsBatch], vi[kRsBatch];
#pragma unroll
        for (int t = 0; t < kRsBatch; ++t) {
          vr[t] = vi[t] = lr[t] = li[t] = 0.0;
          if (e + t < d.cnt) {
            const int q = d.e0 + e + t;
            const int j = cols[q];
            if constexpr (CX) {
              lr[t] = vals[2 * q];
              li[t] = vals[2 * q + 1];
              vr[t] = vec[2 * j];
              vi[t] = vec[2 * j + 1];
            } else {
              lr[t] = vals[q];
              vr[t] = vec[j];
            }
          }
        }
#pragma unroll
        for (int t = 0; t < kRsBatch; ++t)
          if (e + t < d.cnt) mulsub<CX, ADJ>(ar, ai, lr[t], li[t], vr[t], vi[t]);
      }
      double qr = ar, qi = ai;
      if (d.hasdiv) {
        if constexpr (CX)
          py_cdiv(ar, ai, d.dr, ADJ ? -d.di : d.di, qr, qi);
        else
          qr = ddiv(ar, d.dr);
      }
      if constexpr (CX) {
        vec[2 * d.row] = qr;
        vec[2 * d.row + 1] = qi;
      } else {
        vec[d.row] = qr;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (h.z) named_bar(1, NC);  // level complete: its values are readable
  }
  // z = the vector after the backward phase; non-finite -> breakdown
  bool bad = false;
  for (int i = tid; i < n; i += NC) {
    if constexpr (CX) {
      const double qr = vec[2 * i], qi = vec[2 * i + 1];
      bad = bad || !isfin(qr) || !isfin(qi);
      reinterpret_cast<double2 *>(a.z)[i] = make_double2(qr, qi);
    } else {
      const double qr = vec[i];
      bad = bad || !isfin(qr);
      a.z[i] = qr;
    }
  }
  if (bad) atomicOr(a.err, 1);
}

__global__ void gather_rsweep_kernel(const double *lu, RSweep p, int cx) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double *st = reinterpret_cast<double *>(p.stream);
  if (t < p.nent) {
    const int s = p.esrc[t];
    const long long o = p.eoff[t];
    if (cx) {
      const double2 v = reinterpret_cast<const double2 *>(lu)[s];
      st[o] = v.x;
      st[o + 1] = v.y;
    } else {
      st[o] = lu[s];
    }
  }
  if (t < p.ndesc) {
    const int s = p.dsrc[t];
    if (s >= 0) {
      const long long o = p.doff[t];
      if (cx) {
        const double2 v = reinterpret_cast<const double2 *>(lu)[s];
        st[o] = v.x;
        st[o + 1] = v.y;
      } else {
        st[o] = lu[s];
      }
    }
  }
}

int sweep_grid(int n) {
  // enough resident warps to expose the DAG's width; extra warps idle out
  long long warps = (2LL * n + 31) / 32;
  long long blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks < 1) blocks = 1;
  if (blocks > sm_count() * 6) blocks = sm_count() * 6;
  return (int)blocks;
}

}  // namespace

// Sweep variant (A/B measured on B200): MPK_SWEEP_VAR
// 0 = one dependency load at a time (volatile), 1 = batches of 8
// (volatile), 2 = batches of 8 (relaxed.gpu), 3 = one at a time (relaxed).
static int sweep_variant() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("MPK_SWEEP_VAR");
    v = e ? atoi(e) : 3;
    if (v < 0 || v > 3) v = 3;
  }
  return v;
}

template <bool CX, bool ADJ>
static void launch_sweep_t(const SweepArgs &a, int g, cudaStream_t st) {
  switch (sweep_variant()) {
    case 0: sweep_kernel<CX, ADJ, 1, false><<<g, kBlock, 0, st>>>(a); break;
    case 1: sweep_kernel<CX, ADJ, 8, false><<<g, kBlock, 0, st>>>(a); break;
    case 2: sweep_kernel<CX, ADJ, 8, true><<<g, kBlock, 0, st>>>(a); break;
    default: sweep_kernel<CX, ADJ, 1, true><<<g, kBlock, 0, st>>>(a); break;
  }
}

static bool env_on(const char *name, bool dflt) {
  const char *e = getenv(name);
  if (!e) return dflt;
  return e[0] != '0';
}

constexpr size_t kSmemMax = 227 * 1024;

template <bool CX, bool ADJ>
static void launch_sweep_smem(const SweepArgs &a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sweep_smem_kernel<CX, ADJ>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemMax);
    attr = true;
  }
  const size_t bytes = (size_t)a.n * (CX ? 16 : 8);
  sweep_smem_kernel<CX, ADJ><<<1, kSmemThreads, bytes, st>>>(a);
}

template <bool CX, bool ADJ>
static void launch_sweep_mats_t(const SweepArgs &a, const SweepMats &m,
                                cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sweep_mats_kernel<CX, ADJ>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemMax);
    attr = true;
  }
  const size_t bytes = (size_t)a.n * (CX ? 16 : 8) +
                       sizeof(int) * (m.fwd.nlev + m.bwd.nlev + 2);
  int T = ((std::max(m.fwd.maxw, m.bwd.maxw) + 31) / 32) * 32;
  T = T < 32 ? 32 : (T > kMatsThreads ? kMatsThreads : T);
  sweep_mats_kernel<CX, ADJ><<<1, T, bytes, st>>>(a, m);
}

void launch_sweep_mats(const SweepArgs &a, const SweepMats &m, bool cx,
                       bool adjoint, cudaStream_t st) {
  ++tl_launches;
  if (!cx && !adjoint) launch_sweep_mats_t<false, false>(a, m, st);
  if (!cx && adjoint) launch_sweep_mats_t<false, true>(a, m, st);
  if (cx && !adjoint) launch_sweep_mats_t<true, false>(a, m, st);
  if (cx && adjoint) launch_sweep_mats_t<true, true>(a, m, st);
}

size_t csweep_smem_limit() { return kSmemMax; }

template <bool CX, bool ADJ>
static void launch_csweep_t(const SweepArgs &a, const CSweep &p,
                            cudaStream_t st) {
  static bool attr[2] = {false, false};
  auto kfn = p.dflow ? dsweep_kernel<CX, ADJ> : csweep_kernel<CX, ADJ>;
  if (!attr[p.dflow]) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemMax);
    cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr[p.dflow] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.C);
  cfg.blockDim = dim3(p.T);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kfn, a, p);
}

void launch_csweep(const SweepArgs &a, const CSweep &p, bool cx, bool adjoint,
                   cudaStream_t st) {
  ++tl_launches;
  if (!cx && !adjoint) launch_csweep_t<false, false>(a, p, st);
  if (!cx && adjoint) launch_csweep_t<false, true>(a, p, st);
  if (cx && !adjoint) launch_csweep_t<true, false>(a, p, st);
  if (cx && adjoint) launch_csweep_t<true, true>(a, p, st);
}

void gather_csweep(const double *lu, const CSweep &p, bool cx,
                   cudaStream_t st) {
  const long long m = p.nval;
  if (p.C == 0 || m <= 0) return;
  ++tl_launches;
  gather_csweep_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(lu, p,
                                                                    cx ? 1 : 0);
}

template <bool CX, bool ADJ>
static void launch_rsweep_t(const SweepArgs &a, const RSweep &p,
                            cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rsweep_kernel<CX, ADJ>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemMax);
    attr = true;
  }
  rsweep_kernel<CX, ADJ><<<1, p.T, p.smem, st>>>(a, p);
}

void launch_rsweep(const SweepArgs &a, const RSweep &p, bool cx, bool adjoint,
                   cudaStream_t st) {
  ++tl_launches;
  if (!cx && !adjoint) launch_rsweep_t<false, false>(a, p, st);
  if (!cx && adjoint) launch_rsweep_t<false, true>(a, p, st);
  if (cx && !adjoint) launch_rsweep_t<true, false>(a, p, st);
  if (cx && adjoint) launch_rsweep_t<true, true>(a, p, st);
}

void gather_rsweep(const double *lu, const RSweep &p, bool cx,
                   cudaStream_t st) {
  const long long m = p.nent > p.ndesc ? p.nent : p.ndesc;
  if (p.nchunks == 0 || m <= 0) return;
  ++tl_launches;
  gather_rsweep_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(lu, p,
                                                                    cx ? 1 : 0);
}

bool sweep_uses_smem(int n, bool cx) {
  return env_on("MPK_SWEEP_SMEM", true) &&
         (size_t)n * (cx ? 16 : 8) + 16384 <= kSmemMax;
}

void launch_sweep(const SweepArgs &a, bool cx, bool adjoint,
                  cudaStream_t st) {
  ++tl_launches;
  if (a.lev_f && a.lev_b && sweep_uses_smem(a.n, cx)) {
    if (!cx && !adjoint) launch_sweep_smem<false, false>(a, st);
    if (!cx && adjoint) launch_sweep_smem<false, true>(a, st);
    if (cx && !adjoint) launch_sweep_smem<true, false>(a, st);
    if (cx && adjoint) launch_sweep_smem<true, true>(a, st);
    return;
  }
  SweepArgs b = a;  // multi-CTA sync-free kernel: natural row order
  b.ord_f = b.ord_b = nullptr;
  const int g = sweep_grid(a.n);
  if (!cx && !adjoint) launch_sweep_t<false, false>(b, g, st);
  if (!cx && adjoint) launch_sweep_t<false, true>(b, g, st);
  if (cx && !adjoint) launch_sweep_t<true, false>(b, g, st);
  if (cx && adjoint) launch_sweep_t<true, true>(b, g, st);
}

void launch_sweep_reset(double *y, double *z, int n, bool cx,
                        const int *done, cudaStream_t st) {
  const int g = grid_for(n);
  ++tl_launches;
  if (cx)
    sweep_reset_kernel<true><<<g, kBlock, 0, st>>>(y, z, n, done);
  else
    sweep_reset_kernel<false><<<g, kBlock, 0, st>>>(y, z, n, done);
}

__global__ void fill_sentinel_kernel(double *p, long long n) {
  const double s = sent_val();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = s;
}
void launch_fill_sentinel(double *p, long long n, cudaStream_t st) {
  ++tl_launches;
  long long g = (n + 255) / 256;
  if (g > sm_count() * 8) g = sm_count() * 8;
  if (g < 1) g = 1;
  fill_sentinel_kernel<<<(int)g, 256, 0, st>>>(p, n);
}

void launch_factor(const FactorArgs &a, bool cx, cudaStream_t st) {
  ++tl_launches;
  if (a.lev && a.n <= 65536 && env_on("MPK_FACTOR_SMEM", false)) {
    if (cx)
      factor_smem_kernel<true><<<1, kSmemThreads, 0, st>>>(a);
    else
      factor_smem_kernel<false><<<1, kSmemThreads, 0, st>>>(a);
    return;
  }
  // Multi-CTA sync-free kernel.  Ticket t -> row: natural order (t), or the
  // level order of the L DAG (a.ord).  In natural order the 32 rows of a warp
  // are usually chained (a grid stencil's row i needs row i-1), so the lanes
  // of one warp wait on each other and every DAG level costs a divergent
  // spin hand-off (cfg4: 6142 levels x 16 us).  In level order a warp's rows
  // are independent and only wait on rows of lower levels, held by other
  // (resident, lower-ticket) warps -- every level is padded to a multiple of
  // 32 tickets (FactorArgs::ordp), else the warp straddling a level boundary
  // would chain its lanes again.  Deep DAGs take the level order; shallow
  // ones (random patterns: tens of levels, rows of a level scattered over
  // the matrix) keep the natural order and its coalesced row reads.
  // MPK_FACTOR_ORDER = natural | level overrides.
  FactorArgs b = a;
  bool level = a.ordp != nullptr;
  if (const char *e = getenv("MPK_FACTOR_ORDER")) level = a.ordp != nullptr && e[0] == 'l';
  b.ord = level ? a.ordp : nullptr;
  long long warps = ((level ? a.nt : a.n) + 31) / 32;
  long long blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks < 1) blocks = 1;
  int per_sm = level ? 1 : 6;  // level order: fewer pollers, shorter hand-off (measured)
  if (const char *e = getenv("MPK_FACTOR_BLOCKS")) per_sm = atoi(e) > 0 ? atoi(e) : per_sm;
  if (blocks > (long long)sm_count() * per_sm) blocks = (long long)sm_count() * per_sm;
  if (const char *e = getenv("MPK_FACTOR_GRID"))
    if (atoi(e) > 0 && atoi(e) < blocks) blocks = atoi(e);
  if (cx)
    factor_kernel<true><<<(int)blocks, kBlock, 0, st>>>(b);
  else
    factor_kernel<false><<<(int)blocks, kBlock, 0, st>>>(b);
}

}  // namespace mpk
