// wf.cu -- lane-chunk wavefront sweep plan (see wf.cuh for the scheme).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ilu.cuh"

namespace mpk {

namespace {

constexpr unsigned kFullW = 0xffffffffu;

__device__ __forceinline__ uint32_t wf_smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void wf_mbar_init(uint64_t *b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(wf_smem_u32(b)),
               "r"(cnt)
               : "memory");
}
__device__ __forceinline__ void wf_mbar_arrive_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   wf_smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void wf_mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WF_WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WF_WAIT%=;\n}\n" ::"r"(wf_smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void wf_bulk(void *dst, const void *src,
                                        uint32_t bytes, uint64_t *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(wf_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(wf_smem_u32(b))
      : "memory");
}

template <bool CX>
__device__ __forceinline__ void wf_ld(const double *buf, int j, double &r,
                                      double &m) {
  if constexpr (CX) {
    const double2 w = ld_relaxed2(reinterpret_cast<const double2 *>(buf) + j);
    r = w.x;
    m = w.y;
  } else {
    r = ld_relaxed(buf + j);
    m = 0.0;
  }
}
__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(wf_smem_u32(dst)),
               "l"(src)
               : "memory");
}
template <bool CX>
__device__ __forceinline__ void cp_async_v(double *dst, const double *src) {
  if constexpr (CX)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(wf_smem_u32(dst)),
                 "l"(src)
                 : "memory");
  else
    cp_async8(dst, src);
}
// sentinel test on the high word only: 0x7FF40000 is a signalling NaN no
// binary64 operation produces and published values are never signalling
// with that payload (wf_pub), so the low word need not be compared
__device__ __forceinline__ bool wf_hi_sent(double v) {
  return __double2hiint(v) == (int)(kSentBits >> 32);
}
template <bool CX>
__device__ __forceinline__ bool wf_sent(double r, double m) {
  return wf_hi_sent(r) || (CX && wf_hi_sent(m));
}
template <bool CX>
__device__ __forceinline__ void wf_poll(const double *buf, int j, double &r,
                                        double &m) {
  wf_ld<CX>(buf, j, r, m);
  while (wf_sent<CX>(r, m)) {
    __nanosleep(32);
    wf_ld<CX>(buf, j, r, m);
  }
}
__device__ __forceinline__ double wf_unsent(double v) {
  return wf_hi_sent(v) ? __longlong_as_double((long long)kQNaNBits) : v;
}
template <bool CX>
__device__ __forceinline__ void wf_pub(double *buf, int j, double r, double m) {
  if constexpr (CX) {
    const double2 v = make_double2(wf_unsent(r), wf_unsent(m));
    asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(
                     reinterpret_cast<double2 *>(buf) + j),
                 "d"(v.x), "d"(v.y));
  } else {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(buf + j),
                 "d"(wf_unsent(r)));
  }
}

// acc -= l * v in the reference's order (real a - l*u; complex CPython)
template <bool CX>
__device__ __forceinline__ void wf_mulsub(double &ar, double &ai, double lr,
                                          double li, double vr, double vi) {
  if constexpr (CX) {
    double pr, pi;
    py_cmul(lr, li, vr, vi, pr, pi);
    ar = dsub(ar, pr);
    ai = dsub(ai, pi);
  } else {
    ar = dsub(ar, dmul(lr, vr));
  }
}

__device__ long long wf_dbg2[4096];  // clock64 per step of group 0 (dbg 2)
__device__ int wf_dbg3[8192];        // slow-path steps per group (dbg)
__device__ long long wf_dbg4[4096];  // clock per step of group 1 (dbg 2)
__device__ __forceinline__ long long wf_gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// a / d on the critical path of a backward row: reciprocal (independent of
// a, off the chain) + Markstein correction, then an exact residual test
// that PROVES the result equals RN(a / d) (= __ddiv_rn): with e = a - q*d
// exact (fma; q within an ulp of a/d), q == RN(a/d) iff |a/d - q| < ulp(q)/2
// i.e. |e| < |d| * ulp(q)/2 (ties cannot occur in this range).  Outside
// the safe exponent range, for q a power of two (asymmetric ulp) or when
// the test fails, ok = false and the caller divides with __ddiv_rn.
__device__ __forceinline__ double wf_fast_div(double a, double d, double r, bool &ok) {
  // r = __drcp_rn(d), precomputed per factorization (wf_gather_kernel)
  const double q0 = __dmul_rn(a, r);
  const double e0 = fma(-q0, d, a);
  const double q2 = fma(e0, r, q0);   // one Markstein correction
  const double e2 = fma(-q2, d, a);   // exact residual of the candidate
  const unsigned long long qb = (unsigned long long)__double_as_longlong(q2);
  const unsigned long long ab = (unsigned long long)__double_as_longlong(a);
  const unsigned long long db = (unsigned long long)__double_as_longlong(d);
  const int eq = (int)((qb >> 52) & 0x7ff), ea = (int)((ab >> 52) & 0x7ff),
            ed = (int)((db >> 52) & 0x7ff);
  const double half_ulp = __longlong_as_double((long long)(eq - 53) << 52);
  ok = eq > 256 && eq < 1792 && ea > 256 && ea < 1792 && ed > 256 && ed < 1792 &&
       (qb & 0xFFFFFFFFFFFFFull) != 0 && fabs(e2) < __dmul_rn(fabs(d), half_ulp);
  return q2;
}

// Shared-memory layout of one CTA (= one group at a time, two warps:
// warp 0 computes, warp 1 stages remote values), byte offsets; the host
// analysis encodes value sources as such offsets:
//   [0, 128) mbarriers | [128, 144) zero slot | ring [H][32] |
//   stage [NS][T][EM+2][32] | NB record buffers
// Record of one (group, step):
//   int32 off[EM][32] (value source: ring / stage / zero slot) |
//   int32 col[EM][32] (global row for stage-sourced values, else -1) |
//   value[EM][32] | divisor[32] (backward)
constexpr int kWfNS = 3;  // stage chunks (helper lead)
template <bool CX>
struct WfLayout {
  static constexpr int VB = CX ? 16 : 8;        // value bytes
  static constexpr int kZero = 128;
  static constexpr int kRingOff = 256;
  static constexpr int kRing = 32 * kWfH * VB;
  static constexpr int kStageOff = kRingOff + kRing;
  static constexpr int kStage = kWfNS * kWfT * (kWfEM + 2) * 32 * VB;
  // rhs ring [4 chunks][2 planes][32 lanes][10 f64]: a lane's T values of
  // a chunk are contiguous (16-byte copies), lane stride 80 B (2-way banks)
  static constexpr int kRhsOff = kStageOff + kStage;
  static constexpr int kRhs = 4 * 2 * 32 * 80;
  static constexpr int kBufOff = kRhsOff + kRhs;
  static __host__ __device__ constexpr int rhs_base(int c, int plane, int j) {
    return kRhsOff + (((c & 3) * 2 + plane) * 32 + j) * 80;
  }
  static constexpr int kOffB = kWfEM * 32 * 4;  // off block bytes
  static constexpr int kValOff = 2 * kOffB;     // values after off + col
  static constexpr int kVal = kWfEM * 32 * VB;
  static __host__ __device__ constexpr int ring_slot(int sq, int jq) {
    return kRingOff + ((sq & (kWfH - 1)) * 32 + jq) * VB;
  }
  // step s of a group (chunks restart at stage buffer 0 for every group)
  static __host__ __device__ constexpr int stage_slot(int s, int slot, int j) {
    return kStageOff +
           ((((s / kWfT) % kWfNS) * kWfT + (s % kWfT)) * (kWfEM + 2) + slot) * 32 * VB +
           j * VB;
  }
};

// barriers: rec_full[NB] at 0
__device__ __forceinline__ uint64_t *wf_bar(unsigned char *base, int i) {
  return reinterpret_cast<uint64_t *>(base) + i;
}

// One group (32 lanes) of one phase, run by one warp.  Chunk c (T steps):
// its step records arrive by TMA bulk copies NB chunks ahead; the remote
// values of chunk c + 1 (right-hand sides, dependencies the ring does not
// hold) are requested by cp.async at the top of chunk c.  Per step the lane's row is a
// branch-free chain: every entry reads its value through a precomputed
// shared-memory offset (ring, stage, or the zero slot for padding: acc -
// 0*0 == acc bit for bit); a staged value still carrying the sentinel (not
// yet published when requested) is re-polled with an L1-bypassing load.
// L1-cached cp.async copies are safe: L1 starts every launch invalidated
// and a published slot only changes sentinel -> final value, so a stale
// copy can only be a sentinel.
template <bool CX, bool FWD>
__device__ __forceinline__ void wf_group(const SweepArgs &a, const WPhase &P,
                                         int gl, unsigned char *wbase,
                                         int bufsz, bool dbgstep, bool dbgcnt,
                                         int dbgg) {
  using Lt = WfLayout<CX>;
  constexpr int VW = CX ? 2 : 1;
  const int j = threadIdx.x & 31;
  const int n = a.n, S = P.S, rs = P.recsz, Lc = P.Lc, lag = P.lag;
  const int nch = S / kWfT;
  const unsigned char *src = P.rec + (size_t)gl * nch * P.chunkb;
  const int p0 = (gl * 32 + j) * Lc - lag * j;  // n < 2^31 (C ABI check)
  const int pos0 = -lag * j;
  double *glob = FWD ? a.y : a.z;
  unsigned char *buf = wbase + Lt::kBufOff;
  const uint32_t cb = (uint32_t)P.chunkb;
  if (j == 0) {
    const int first = nch < kWfNB ? nch : kWfNB;
    for (int c = 0; c < first; ++c) {
      wf_mbar_arrive_tx(wf_bar(wbase, c), cb);
      wf_bulk(buf + (size_t)c * bufsz, src + (size_t)c * cb, cb, wf_bar(wbase, c));
    }
  }
  auto recp = [&](int s) -> const unsigned char * {
    return buf + (size_t)((s / kWfT) % kWfNB) * bufsz + (size_t)(s % kWfT) * rs;
  };
  auto rec_wait = [&](int c) {
    if (c < nch) wf_mbar_wait(wf_bar(wbase, c % kWfNB), (c / kWfNB) & 1);
  };
  // cp.async of chunk c's remote dependency values (one commit group per
  // chunk, maybe empty): the chunk's fetch table spreads them over the 32
  // lanes ({global row, shared offset} items, row -1 = none)
  // Register path (kmax <= kWfRegItems): the items of chunk c are LOADED at
  // the top of chunk c-1 with L1-bypassing relaxed loads (an L1-cached copy
  // of the line, fetched while neighbouring values were still sentinels,
  // would keep re-serving the sentinel) and stored to their stage slots at
  // the top of chunk c.  The cp.async group of the chunk is then empty.
  constexpr int kWfRegItems = 4;
  const bool regpath = P.kmax <= kWfRegItems;
  double dvr[kWfRegItems], dvi[kWfRegItems];
  int dvo[kWfRegItems];
  auto deps_load = [&](int c) {
#pragma unroll
    for (int r = 0; r < kWfRegItems; ++r) {
      dvo[r] = -1;
      if (c < nch && r < P.kmax) {
        const int2 it = reinterpret_cast<const int2 *>(
            buf + (size_t)(c % kWfNB) * bufsz + (size_t)kWfT * rs)[r * 32 + j];
        if (it.x >= 0) {
          dvo[r] = it.y;
          wf_ld<CX>(glob, it.x, dvr[r], dvi[r]);
        }
      }
    }
  };
  auto deps_store = [&]() {
#pragma unroll
    for (int r = 0; r < kWfRegItems; ++r)
      if (dvo[r] >= 0) {
        double *d = reinterpret_cast<double *>(wbase + dvo[r]);
        d[0] = dvr[r];
        if constexpr (CX) d[1] = dvi[r];
      }
  };
  auto deps_issue = [&](int c) {
    if (c < nch && !regpath) {
      const int2 *ft = reinterpret_cast<const int2 *>(
          buf + (size_t)(c % kWfNB) * bufsz + (size_t)kWfT * rs);
      for (int r = 0; r < P.kmax; ++r) {
        const int2 it = ft[r * 32 + j];
        if (it.x >= 0)
          cp_async_v<CX>(reinterpret_cast<double *>(wbase + it.y), glob + (size_t)it.x * VW);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // chunk c's right-hand sides (static input / forward results, requested
  // 3 chunks ahead): a lane's T rows are consecutive, 4 x 16-byte copies
  // when aligned and all active, else one 8-byte copy per active step
  auto rhs_issue = [&](int c) {
    if (c < nch) {
      const int s0 = c * kWfT;
      const int pa = p0 + s0;
      const bool full = (unsigned)(s0 + pos0) < (unsigned)Lc &&
                        (unsigned)(s0 + pos0 + kWfT - 1) < (unsigned)Lc &&
                        pa + kWfT - 1 < n;
      double *d0 = reinterpret_cast<double *>(wbase + Lt::rhs_base(c, 0, j));
      if (!CX && P.rhs16 && full) {
        const double *g0 = FWD ? a.in_re + pa : a.y + (n - kWfT - pa);
#pragma unroll
        for (int q = 0; q < kWfT / 2; ++q)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(wf_smem_u32(d0 + 2 * q)),
                       "l"(g0 + 2 * q)
                       : "memory");
      } else {
        double *d1 = reinterpret_cast<double *>(wbase + Lt::rhs_base(c, 1, j));
#pragma unroll
        for (int t = 0; t < kWfT; ++t) {
          const int s = s0 + t;
          const int pp = p0 + s;
          if ((unsigned)(s + pos0) < (unsigned)Lc && pp < n) {
            const int row = FWD ? pp : n - 1 - pp;
            const int ix = FWD ? t : kWfT - 1 - t;
            if constexpr (FWD) {
              cp_async8(d0 + ix, a.in_re + row);
              if constexpr (CX) cp_async8(d1 + ix, a.in_im + row);
            } else {
              cp_async8(d0 + ix, a.y + (size_t)row * VW);
              if constexpr (CX) cp_async8(d1 + ix, a.y + (size_t)row * VW + 1);
            }
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int off[kWfEM];
  double lr[kWfEM], li[kWfEM];
  auto load_rec = [&](int s) {
    const unsigned char *rec = recp(s);
#pragma unroll
    for (int e = 0; e < kWfEM; ++e) {
      off[e] = reinterpret_cast<const int *>(rec)[e * 32 + j];
      const double *val = reinterpret_cast<const double *>(rec + Lt::kValOff);
      lr[e] = val[(e * 32 + j) * VW];
      li[e] = CX ? val[(e * 32 + j) * VW + 1] : 0.0;
    }
  };
  // commit order per chunk c: deps(c + 1), rhs(c + 3); at the top of chunk
  // c the three most recent groups (rhs(c+3), deps(c+1), rhs(c+2)) may
  // still be pending: deps(c) and rhs(c) are complete
  rec_wait(0);
  if constexpr (!FWD) {
    // the backward right-hand sides are forward results: request them once
    // the forward phase's last row (the sink of its DAG for grid stencils)
    // is published, instead of re-polling stale requests row by row
    if (j == 0) {
      double r0, m0;
      wf_poll<CX>(a.y, n - 1, r0, m0);
    }
    __syncwarp();
  }
  deps_issue(0);
  rhs_issue(0);
  rhs_issue(1);
  rhs_issue(2);
  load_rec(0);
  if (regpath && P.kmax > 0 && nch > 1) {
    // Start at the steady-state lag: wait until every remote value of
    // chunk 1 is published, so that from here on each chunk's values
    // (requested one chunk ahead) are ready when requested.  Starting
    // earlier only ends in per-step polls that overshoot the lag.
    rec_wait(1);
    const int2 *ft = reinterpret_cast<const int2 *>(
        buf + (size_t)(1 % kWfNB) * bufsz + (size_t)kWfT * rs);
    for (int r = 0; r < P.kmax; ++r) {
      const int2 it = ft[r * 32 + j];
      if (it.x >= 0) {
        double vr0, vi0;
        wf_poll<CX>(glob, it.x, vr0, vi0);
      }
    }
    __syncwarp();
  }
  if (regpath) deps_load(0);
  const bool dbc = dbgstep && j == 0;
  for (int c = 0; c < nch; ++c) {
    if (dbc && c < 256) wf_dbg2[3072 + 4 * c] = clock64();
    rec_wait(c + 1);
    if (regpath) {
      deps_store();     // chunk c's remote values (loaded one chunk ago)
      deps_load(c + 1);
    }
    if (dbc && c < 256) wf_dbg2[3072 + 4 * c + 1] = clock64();
    deps_issue(c + 1);
    if (dbc && c < 256) wf_dbg2[3072 + 4 * c + 2] = clock64();
    rhs_issue(c + 3);
    if (dbc && c < 256) wf_dbg2[3072 + 4 * c + 3] = clock64();
    asm volatile("cp.async.wait_group 3;" ::: "memory");  // deps(c), rhs(c) landed
#pragma unroll
    for (int t = 0; t < kWfT; ++t) {
      const int s = c * kWfT + t;
      if (dbgstep && j == 0 && s < 3072) wf_dbg2[s] = wf_gtime();
      if (dbgcnt && dbgg == (FWD ? 1 : P.ngroups) && j == 0 && s < 3072) wf_dbg4[s] = wf_gtime();
      const int pp = p0 + s;
      const bool act = (unsigned)(s + pos0) < (unsigned)Lc && pp < n;
      double vr[kWfEM], vi[kWfEM], cl[kWfEM], cm[kWfEM];
      bool bad = false;
#pragma unroll
      for (int e = 0; e < kWfEM; ++e) {
        const double *vp = reinterpret_cast<const double *>(wbase + off[e]);
        vr[e] = vp[0];
        vi[e] = CX ? vp[1] : 0.0;
        cl[e] = lr[e];
        cm[e] = li[e];
        bad |= wf_sent<CX>(vr[e], vi[e]);
      }
      const int rix = FWD ? t : kWfT - 1 - t;
      const double *rh = reinterpret_cast<const double *>(wbase + Lt::rhs_base(c, 0, j)) + rix;
      const double *rh1 = reinterpret_cast<const double *>(wbase + Lt::rhs_base(c, 1, j)) + rix;
      double ar, ai;
      if constexpr (FWD && CX) {
        const double re0 = rh[0];
        const double im0 = rh1[0];
        ar = dadd(re0, dsub(dmul(0.0, im0), 0.0));  // numpy re + 1j*im
        ai = dadd(0.0, im0);
      } else {
        ar = rh[0];
        ai = CX ? rh1[0] : 0.0;
        if (!FWD) bad |= wf_sent<CX>(ar, ai);
      }
      double dr = 0.0, di = 0.0, drc = 0.0;
      if constexpr (!FWD) {
        const double *dv =
            reinterpret_cast<const double *>(recp(s) + Lt::kValOff + Lt::kVal);
        dr = dv[j * VW];
        di = CX ? dv[j * VW + 1] : 0.0;
        if constexpr (!CX) drc = dv[32 + j];  // reciprocal block follows
      }
      if (s + 1 < S) load_rec(s + 1);  // read ahead
      // common path: the chain on the staged values (no branch before it)
      double xr = ar, xi = ai;
#pragma unroll
      for (int e = 0; e < kWfEM; ++e) wf_mulsub<CX>(xr, xi, cl[e], cm[e], vr[e], vi[e]);
      bool slow = act && bad;
      if constexpr (!FWD) {
        if constexpr (CX) {
          double qr, qi;
          py_cdiv(xr, xi, dr, di, qr, qi);
          xr = qr;
          xi = qi;
        } else {
          bool ok;
          xr = wf_fast_div(xr, dr, drc, ok);
          slow |= act && !ok;
        }
      }
      if (slow && dbgcnt) atomicAdd(&wf_dbg3[dbgg], bad ? 1 : 65536);
      if (slow) {  // a staged value was requested before it was published,
                   // or the fast quotient is not provably RN: redo the row
        const int row = FWD ? pp : n - 1 - pp;
        const int *col = reinterpret_cast<const int *>(recp(s) + Lt::kOffB);
#pragma unroll
        for (int e = 0; e < kWfEM; ++e)
          if (wf_sent<CX>(vr[e], vi[e])) wf_poll<CX>(glob, col[e * 32 + j], vr[e], vi[e]);
        if (!FWD && wf_sent<CX>(ar, ai)) wf_poll<CX>(a.y, row, ar, ai);
        xr = ar;
        xi = ai;
#pragma unroll
        for (int e = 0; e < kWfEM; ++e) wf_mulsub<CX>(xr, xi, cl[e], cm[e], vr[e], vi[e]);
        if constexpr (!FWD) {
          if constexpr (CX) {
            double qr, qi;
            py_cdiv(xr, xi, dr, di, qr, qi);
            xr = qr;
            xi = qi;
          } else {
            xr = ddiv(xr, dr);
          }
        }
      }
      ar = xr;
      ai = xi;
      if constexpr (!FWD) {
        if (act && (!isfin(ar) || !isfin(ai))) atomicOr(a.err, 1);
      }
      if (act) {
        double *rg = reinterpret_cast<double *>(wbase + Lt::ring_slot(s, j));
        rg[0] = ar;
        if constexpr (CX) rg[1] = ai;
        wf_pub<CX>(glob, FWD ? pp : n - 1 - pp, ar, ai);
      }
      __syncwarp();
    }
    // record chunk c consumed: refill its buffer with chunk c + NB
    if (j == 0 && c + kWfNB < nch) {
      const int b = c % kWfNB;
      wf_mbar_arrive_tx(wf_bar(wbase, b), cb);
      wf_bulk(buf + (size_t)b * bufsz, src + (size_t)(c + kWfNB) * cb, cb,
              wf_bar(wbase, b));
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// diagnostics (MPK_WF_DEBUG=1): globaltimer at start / end of every group
__device__ long long wf_dbg[2 * 8192];


template <bool CX>
__global__ void __launch_bounds__(32, 1)
    wsweep_kernel(SweepArgs a, WPhase F, WPhase B, int bufsz, int dbg) {
  {  // stopped solve: skip, but count this CTA out (ticket reset)
    int d = 0;
    if (threadIdx.x == 0 && a.done) d = *(volatile const int *)a.done;
    if (__shfl_sync(kFullW, d, 0)) {
      if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&a.tick[1], 1) == (int)gridDim.x - 1) {
          atomicExch(&a.tick[0], 0);
          atomicExch(&a.tick[1], 0);
        }
      }
      return;
    }
  }
  using Lt = WfLayout<CX>;
  extern __shared__ __align__(128) unsigned char wsm[];
  const int j = threadIdx.x & 31;
  unsigned char *base = wsm;
  if (j < 4) reinterpret_cast<double *>(base + Lt::kZero)[j & 1] = 0.0;
  const int gtot = F.ngroups + B.ngroups;
  for (;;) {
    int g = 0;
    if (j == 0) {
      g = atomicAdd(a.tick, 1);
      // fresh barriers per group (no copy is pending here)
      for (int b = 0; b < kWfNB; ++b) wf_mbar_init(wf_bar(base, b), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    g = __shfl_sync(kFullW, g, 0);
    __syncwarp();
    if (g >= gtot) break;
    if (dbg && j == 0 && g < 8192) wf_dbg[2 * g] = wf_gtime();
    if (g < F.ngroups)
      wf_group<CX, true>(a, F, g, base, bufsz, dbg == 2 && g == 0, dbg != 0, g & 8191);
    else
      wf_group<CX, false>(a, B, g - F.ngroups, base, bufsz, false, dbg != 0, g & 8191);
    if (dbg && j == 0 && g < 8192) wf_dbg[2 * g + 1] = wf_gtime();
    __syncwarp();
  }
  // last CTA out resets the ticket for the next launch / graph replay
  if (j == 0) {
    __threadfence();
    if (atomicAdd(&a.tick[1], 1) == (int)gridDim.x - 1) {
      atomicExch(&a.tick[0], 0);
      atomicExch(&a.tick[1], 0);
    }
  }
}

__global__ void wf_gather_kernel(const double *lu, WPhase P, int cx) {
  const int VB = cx ? 16 : 8;
  const int kCode = 2 * kWfEM * 32 * 4, kVal = kWfEM * 32 * VB;
  const long long tot = P.nslots + P.ndslots;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    int srcp;
    unsigned char *dst;
    if (i < P.nslots) {
      const long long gs = i / (kWfEM * 32);
      const int rem = (int)(i % (kWfEM * 32));
      srcp = P.esrc[i];
      dst = P.rec + (gs / kWfT) * P.chunkb + (gs % kWfT) * P.recsz + kCode + (size_t)rem * VB;
    } else {
      const long long d = i - P.nslots;
      srcp = P.dsrc[d];
      const long long gs = d / 32;
      dst = P.rec + (gs / kWfT) * P.chunkb + (gs % kWfT) * P.recsz + kCode + kVal + (d % 32) * VB;
    }
    if (cx) {
      const double2 v = srcp >= 0 ? reinterpret_cast<const double2 *>(lu)[srcp]
                                  : make_double2(0.0, 0.0);
      *reinterpret_cast<double2 *>(dst) = v;
    } else {
      const double v = srcp >= 0 ? lu[srcp] : 0.0;
      *reinterpret_cast<double *>(dst) = v;
      if (i >= P.nslots)  // backward divisor: its RN reciprocal follows the block
        *reinterpret_cast<double *>(dst + 32 * 8) = __drcp_rn(v);
    }
  }
}

// Host analysis of one phase.  Positions p = 0..n-1 (forward: row p;
// backward: row n-1-p); dependencies of a row = its L (forward) or U
// (backward) entries in reference order.
struct HostPhase {
  int Lc = 0, lag = 0, nlanes = 0, ngroups = 0, S = 0;
  long long cost = LLONG_MAX;
};

template <class Deps>
static HostPhase choose_phase(int n, Deps deps) {
  // D = max distance back to a dependency
  long long D = 0;
  for (int p = 0; p < n; ++p)
    deps(p, [&](int pq, int) {
      if (p - pq > D) D = p - pq;
    });
  HostPhase best;
  if (D < 2) return best;
  const long long cands[] = {D - 1, D, D + 1, D - 2};
  for (long long Lc : cands) {
    if (Lc < 2 || Lc > n) continue;
    const long long nl = (n + Lc - 1) / Lc;
    if (nl < 8) continue;
    long long lag = 1;
    for (int p = 0; p < n; ++p) {
      const long long l = p / Lc, pos = p % Lc;
      deps(p, [&](int pq, int) {
        const long long lq = pq / Lc, posq = pq % Lc;
        if (lq == l) return;
        // need posq + lag*lq < pos + lag*l
        const long long need = (posq - pos) / (l - lq) + 1;
        const long long nd = (posq - pos) >= 0 ? need : 1;
        if (nd > lag) lag = nd;
      });
      if (lag > 64) break;
    }
    if (lag > 64) continue;
    const long long ng = (nl + 31) / 32;
    const long long S = Lc + lag * 31;
    const long long cost = (ng - 1) * (32 * lag + 24) + S;
    if (cost < best.cost) {
      best.Lc = (int)Lc;
      best.lag = (int)lag;
      best.nlanes = (int)nl;
      best.ngroups = (int)ng;
      best.S = (int)((S + kWfT - 1) / kWfT * kWfT);
      best.cost = cost;
    }
  }
  return best;
}

template <class Deps, class Div>
static bool build_phase_wf(WPhase &ph, int n, bool cx, bool fwd,
                           const HostPhase &hp, Deps deps, Div div,
                           cudaStream_t st) {
  const int VB = cx ? 16 : 8;
  ph.fwd = fwd ? 1 : 0;
  ph.Lc = hp.Lc;
  ph.lag = hp.lag;
  ph.nlanes = hp.nlanes;
  ph.ngroups = hp.ngroups;
  ph.S = hp.S;
  ph.cost = hp.cost;
  // backward: divisors [32] (+ their reciprocals [32], real field)
  ph.recsz = 2 * kWfEM * 32 * 4 + kWfEM * 32 * VB + (fwd ? 0 : 32 * VB + (cx ? 0 : 32 * 8));
  const long long nsteps = (long long)ph.ngroups * ph.S;
  ph.nslots = nsteps * kWfEM * 32;
  ph.ndslots = fwd ? 0 : nsteps * 32;
  std::vector<unsigned char> rec((size_t)nsteps * ph.recsz, 0);
  std::vector<int> esrc((size_t)ph.nslots, -1), dsrc((size_t)ph.ndslots, -1);
  // shared-memory offsets of the value sources (WfLayout<CX>)
  auto ring_slot = [&](long long sq, long long jq) {
    return cx ? WfLayout<true>::ring_slot((int)sq, (int)jq)
              : WfLayout<false>::ring_slot((int)sq, (int)jq);
  };
  auto stage_slot = [&](long long s, int e, long long j) {
    return cx ? WfLayout<true>::stage_slot((int)s, e, (int)j)
              : WfLayout<false>::stage_slot((int)s, e, (int)j);
  };
  const int zero = WfLayout<false>::kZero;
  for (long long gs = 0; gs < nsteps; ++gs) {
    int *off = reinterpret_cast<int *>(rec.data() + gs * ph.recsz);
    int *col = off + kWfEM * 32;
    for (int q = 0; q < kWfEM * 32; ++q) {
      off[q] = zero;
      col[q] = -1;
    }
  }
  const long long Lc = ph.Lc, lag = ph.lag;
  bool ok = true;
  for (int p = 0; p < n && ok; ++p) {
    const long long l = p / Lc, pos = p % Lc;
    const long long g = l / 32, j = l % 32;
    const long long s = pos + lag * j;  // step within the group
    const long long gs = g * ph.S + s;
    int *off = reinterpret_cast<int *>(rec.data() + gs * ph.recsz);
    int *colv = off + kWfEM * 32;
    int e = 0;
    deps(p, [&](int pq, int lu_idx) {
      if (e >= kWfEM) {
        ok = false;
        return;
      }
      const long long lq = pq / Lc, posq = pq % Lc;
      const int col = fwd ? pq : n - 1 - pq;
      bool ring = false;
      long long sq = 0, jq = 0;
      if (lq / 32 == g) {
        jq = lq % 32;
        sq = posq + lag * jq;
        if (sq >= s) {
          ok = false;  // schedule violated (cannot happen for a valid lag)
          return;
        }
        ring = s - sq <= kWfH - 1;
      }
      if (ring) {
        off[e * 32 + j] = ring_slot(sq, jq);
      } else {
        off[e * 32 + j] = stage_slot(s, e, j);
        colv[e * 32 + j] = col;
      }
      esrc[(size_t)((gs * kWfEM + e) * 32 + j)] = lu_idx;
      ++e;
    });
    if (!fwd) dsrc[(size_t)(gs * 32 + j)] = div(p);
  }
  if (!ok) return false;
  // fetch tables: the staged values of each chunk spread over the 32 lanes
  const long long nchunks = nsteps / kWfT;
  std::vector<std::vector<int2>> items((size_t)nchunks);
  int kmax = 0;
  for (long long ch = 0; ch < nchunks; ++ch) {
    for (int t = 0; t < kWfT; ++t) {
      const int *off = reinterpret_cast<const int *>(rec.data() + (ch * kWfT + t) * ph.recsz);
      const int *colv = off + kWfEM * 32;
      for (int q = 0; q < kWfEM * 32; ++q)
        if (colv[q] >= 0) items[(size_t)ch].push_back(make_int2(colv[q], off[q]));
    }
    kmax = std::max(kmax, (int)((items[(size_t)ch].size() + 31) / 32));
  }
  ph.kmax = kmax;
  ph.chunkb = kWfT * ph.recsz + kmax * 32 * 8;
  ph.rhs16 = (!cx && ph.Lc % 2 == 0 && ph.lag % 2 == 0 && (fwd || n % 2 == 0)) ? 1 : 0;
  std::vector<unsigned char> packed((size_t)nchunks * ph.chunkb, 0);
  for (long long ch = 0; ch < nchunks; ++ch) {
    unsigned char *dst = packed.data() + ch * ph.chunkb;
    memcpy(dst, rec.data() + ch * kWfT * ph.recsz, (size_t)kWfT * ph.recsz);
    int2 *ft = reinterpret_cast<int2 *>(dst + (size_t)kWfT * ph.recsz);
    for (int q = 0; q < kmax * 32; ++q)
      ft[q] = q < (int)items[(size_t)ch].size() ? items[(size_t)ch][(size_t)q]
                                                 : make_int2(-1, 0);
  }
  rec.swap(packed);
  auto up = [&](void **d, const void *h, size_t bytes) {
    if (cudaMalloc(d, bytes < 16 ? 16 : bytes) != cudaSuccess) return false;
    return cudaMemcpyAsync(*d, h, bytes, cudaMemcpyHostToDevice, st) ==
           cudaSuccess;
  };
  bool good = up((void **)&ph.rec, rec.data(), rec.size()) &&
              up((void **)&ph.esrc, esrc.data(), esrc.size() * sizeof(int));
  if (!fwd) good = good && up((void **)&ph.dsrc, dsrc.data(), dsrc.size() * sizeof(int));
  cudaStreamSynchronize(st);
  return good;
}

static void free_phase_wf(WPhase &ph) {
  if (ph.rec) cudaFree(ph.rec);
  if (ph.esrc) cudaFree(ph.esrc);
  if (ph.dsrc) cudaFree(ph.dsrc);
  ph = WPhase{};
}

static size_t wf_per_warp(const WSweep &w, bool cx) {
  const int VB = cx ? 16 : 8;
  const int maxchunk = std::max(w.f.chunkb, w.b.chunkb);
  (void)VB;
  const size_t bo = cx ? WfLayout<true>::kBufOff : WfLayout<false>::kBufOff;
  return bo + (size_t)kWfNB * maxchunk;
}

}  // namespace

void free_wsweep(WSweep &w) {
  free_phase_wf(w.f);
  free_phase_wf(w.b);
  w = WSweep{};
}

bool build_wsweep(WSweep &w, int n, bool cx, const int *rp, const int *ci,
                  const int *dp, int nlev_f, int nlev_b, cudaStream_t st) {
  const char *ev = getenv("MPK_WSWEEP");
  if ((ev && ev[0] == '0') || n < 256) return false;
  auto fdeps = [&](int p, auto cb) {
    const int i = p;
    const int hi = dp[i] < 0 ? rp[i] : dp[i];
    for (int q = rp[i]; q < hi; ++q) cb(ci[q], q);
  };
  auto bdeps = [&](int p, auto cb) {
    const int i = n - 1 - p;
    const int lo = dp[i] < 0 ? rp[i + 1] : dp[i] + 1;
    for (int q = lo; q < rp[i + 1]; ++q) cb(n - 1 - ci[q], q);
  };
  // rows with more than kWfEM entries in a phase: no plan
  for (int i = 0; i < n; ++i) {
    const int d = dp[i];
    const int nl = (d < 0 ? rp[i] : d) - rp[i];
    const int nu = rp[i + 1] - (d < 0 ? rp[i + 1] : d + 1);
    if (nl > kWfEM || nu > kWfEM) return false;
  }
  const HostPhase hf = choose_phase(n, fdeps);
  const HostPhase hb = choose_phase(n, bdeps);
  if (hf.Lc == 0 || hb.Lc == 0) return false;
  // the modelled critical path must not be far above the level count
  // (then the level-synchronous plans win)
  const long long lim = 3LL * (nlev_f + nlev_b) + 512;
  if (hf.cost + hb.cost > lim) return false;
  WSweep t;
  if (!build_phase_wf(t.f, n, cx, true, hf, fdeps, [](int) { return -1; }, st) ||
      !build_phase_wf(t.b, n, cx, false, hb, bdeps,
                      [&](int p) { return dp[n - 1 - p]; }, st)) {
    free_wsweep(t);
    return false;
  }
  const size_t pw = wf_per_warp(t, cx);
  if (pw > 220 * 1024) {
    free_wsweep(t);
    return false;
  }
  t.wpb = 1;  // one warp = one group per CTA
  t.smem = pw;
  t.on = 1;
  w = t;
  return true;
}

void gather_wsweep(const double *lu, const WSweep &w, bool cx,
                   cudaStream_t st) {
  if (!w.on) return;
  for (const WPhase *P : {&w.f, &w.b}) {
    const long long tot = P->nslots + P->ndslots;
    if (tot <= 0) continue;
    ++tl_launches;
    long long g = (tot + 255) / 256;
    if (g > sm_count() * 16) g = sm_count() * 16;
    wf_gather_kernel<<<(unsigned)g, 256, 0, st>>>(lu, *P, cx ? 1 : 0);
  }
}

void launch_wsweep(const SweepArgs &a, const WSweep &w, bool cx,
                   cudaStream_t st) {
  ++tl_launches;
  static const int dbg = getenv("MPK_WF_DEBUG") ? atoi(getenv("MPK_WF_DEBUG")) : 0;
  const int bufsz = std::max(w.f.chunkb, w.b.chunkb);
  const int gtot = w.f.ngroups + w.b.ngroups;
  int grid = gtot;
  if (grid > sm_count()) grid = sm_count();
  if (cx) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(wsweep_kernel<true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      attr = true;
    }
    wsweep_kernel<true><<<grid, 32 * w.wpb, w.smem, st>>>(a, w.f, w.b, bufsz, dbg);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(wsweep_kernel<false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      attr = true;
    }
    wsweep_kernel<false><<<grid, 32 * w.wpb, w.smem, st>>>(a, w.f, w.b, bufsz, dbg);
  }
}

}  // namespace mpk

// diagnostics for tools/: per-group globaltimer stamps of the last launch
extern "C" int mpk_wf_debug3(int *out, int reset) {
  if (reset) {
    static int z[8192];
    return cudaMemcpyToSymbol(mpk::wf_dbg3, z, sizeof(z)) == cudaSuccess ? 0 : 4;
  }
  return cudaMemcpyFromSymbol(out, mpk::wf_dbg3, sizeof(int) * 8192) == cudaSuccess ? 0 : 4;
}
extern "C" int mpk_wf_debug4(long long *out) {
  return cudaMemcpyFromSymbol(out, mpk::wf_dbg4, sizeof(long long) * 4096) == cudaSuccess ? 0 : 4;
}
extern "C" int mpk_wf_debug2(long long *out) {
  return cudaMemcpyFromSymbol(out, mpk::wf_dbg2, sizeof(long long) * 4096) == cudaSuccess ? 0 : 4;
}
extern "C" int mpk_wf_debug(long long *out, int n) {
  if (n > 2 * 8192) n = 2 * 8192;
  return cudaMemcpyFromSymbol(out, mpk::wf_dbg, sizeof(long long) * n) == cudaSuccess ? 0 : 4;
}
