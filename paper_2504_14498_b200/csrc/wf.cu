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
template <bool CX>
__device__ __forceinline__ bool wf_sent(double r, double m) {
  return is_sent(r) || (CX && is_sent(m));
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
template <bool CX>
__device__ __forceinline__ void wf_pub(double *buf, int j, double r, double m) {
  if constexpr (CX) {
    const double2 v = make_double2(unsent(r), unsent(m));
    asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(
                     reinterpret_cast<double2 *>(buf) + j),
                 "d"(v.x), "d"(v.y));
  } else {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(buf + j),
                 "d"(unsent(r)));
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

// Per-warp shared-memory layout (byte offsets from the warp's base; the
// host analysis encodes value sources as such offsets):
//   [0, 64) mbarriers | [64, 80) zero slot | [128, +kRing) ring [H][32] |
//   stage [PG][EM+2][32] | NB record buffers
// Record of one (group, step):
//   int32 off[EM][32] (value source: ring / stage / zero slot) |
//   int32 col[EM][32] (global row for stage-sourced values, else -1) |
//   value[EM][32] | divisor[32] (backward)
template <bool CX>
struct WfLayout {
  static constexpr int VB = CX ? 16 : 8;        // value bytes
  static constexpr int PG = CX ? 4 : 8;         // global-value prefetch depth
  static constexpr int kZero = 64;
  static constexpr int kRingOff = 128;
  static constexpr int kRing = 32 * kWfH * VB;
  static constexpr int kStageOff = kRingOff + kRing;
  static constexpr int kStage = PG * (kWfEM + 2) * 32 * VB;
  static constexpr int kBufOff = kStageOff + kStage;
  static constexpr int kOffB = kWfEM * 32 * 4;  // off block bytes
  static constexpr int kValOff = 2 * kOffB;     // values after off + col
  static constexpr int kVal = kWfEM * 32 * VB;
  static __host__ __device__ constexpr int ring_slot(int sq, int jq) {
    return kRingOff + ((sq & (kWfH - 1)) * 32 + jq) * VB;
  }
  static __host__ __device__ constexpr int stage_slot(int u, int slot, int j) {
    return kStageOff + ((u * (kWfEM + 2) + slot) * 32 + j) * VB;
  }
};

// One group (32 lanes) of one phase, run by the calling warp.  Per step the
// lane's row is a branch-free chain: every entry reads its value through a
// precomputed shared-memory offset (ring, prefetched stage, or the zero slot
// for padding: acc - 0*0 == acc bit for bit), one rarely taken branch
// re-polls stage values that were still sentinels when prefetched.
template <bool CX, bool FWD>
__device__ __forceinline__ void wf_group(const SweepArgs &a, const WPhase &P,
                                         int gl, unsigned &cc, uint64_t *bar,
                                         unsigned char *wbase, int bufsz,
                                         bool dbgstep) {
  using Lt = WfLayout<CX>;
  constexpr int PG = Lt::PG;
  constexpr int VW = CX ? 2 : 1;
  const int j = threadIdx.x & 31;
  const int n = a.n, S = P.S, rs = P.recsz, Lc = P.Lc, lag = P.lag;
  const int nch = S / kWfT;
  const unsigned char *src = P.rec + (size_t)gl * S * rs;
  const long long p0 = ((long long)gl * 32 + j) * Lc - (long long)lag * j;
  const int pos0 = -lag * j;
  double *glob = FWD ? a.y : a.z;
  unsigned char *buf = wbase + Lt::kBufOff;
  const uint32_t cb = (uint32_t)(kWfT * rs);
  if (j == 0) {
    const int first = nch < kWfNB ? nch : kWfNB;
    for (int c = 0; c < first; ++c) {
      const int b = (int)((cc + c) % kWfNB);
      wf_mbar_arrive_tx(&bar[b], cb);
      wf_bulk(buf + (size_t)b * bufsz, src + (size_t)c * cb, cb, &bar[b]);
    }
  }
  auto recp = [&](int s) -> const unsigned char * {
    const unsigned c = (unsigned)(s / kWfT);
    return buf + (size_t)((cc + c) % kWfNB) * bufsz + (size_t)(s % kWfT) * rs;
  };
  // lane active at step s: 0 <= s + pos0 < Lc and position < n
  auto active = [&](int s, long long &pp) -> bool {
    pp = p0 + s;
    return (unsigned)(s + pos0) < (unsigned)Lc && pp < n;
  };
  // PG steps ahead: cp.async of the rhs and of stage-sourced values (L1
  // may serve a stale copy only as a sentinel, see wf_poll below)
  // cp.async of step s's rhs / stage-sourced values (col: the record's
  // global rows, read ahead by the caller)
  auto prefetch = [&](int s, int u, const int (&col)[kWfEM]) {
    long long pp;
    if (s < S && active(s, pp)) {
      const int row = FWD ? (int)pp : (int)(n - 1 - pp);
      double *rh = reinterpret_cast<double *>(wbase + Lt::stage_slot(u, kWfEM, j));
      if constexpr (FWD) {
        cp_async8(rh, a.in_re + row);
        if constexpr (CX)
          cp_async8(reinterpret_cast<double *>(wbase + Lt::stage_slot(u, kWfEM + 1, j)),
                    a.in_im + row);
      } else {
        cp_async_v<CX>(rh, a.y + (size_t)row * VW);
      }
#pragma unroll
      for (int e = 0; e < kWfEM; ++e)
        if (col[e] >= 0)
          cp_async_v<CX>(reinterpret_cast<double *>(wbase + Lt::stage_slot(u, e, j)),
                         glob + (size_t)col[e] * VW);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto load_cols = [&](int s, int (&col)[kWfEM]) {
    const int *colp = reinterpret_cast<const int *>(recp(s) + Lt::kOffB);
#pragma unroll
    for (int e = 0; e < kWfEM; ++e) col[e] = s < S ? colp[e * 32 + j] : -1;
  };
  // record fields of a step, read one step ahead
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
  wf_mbar_wait(&bar[cc % kWfNB], (cc / kWfNB) & 1);
  if (nch > 1) wf_mbar_wait(&bar[(cc + 1) % kWfNB], ((cc + 1) / kWfNB) & 1);
#pragma unroll
  for (int u = 0; u < PG; ++u) {
    int col[kWfEM];
    load_cols(u, col);
    prefetch(u, u, col);
  }
  load_rec(0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      const unsigned q = cc + c + 1;
      wf_mbar_wait(&bar[q % kWfNB], (q / kWfNB) & 1);
    }
#pragma unroll
    for (int t = 0; t < kWfT; ++t) {
      const int s = c * kWfT + t;
      const int u = t % PG;
      if (dbgstep && j == 0 && s < 1024) wf_dbg2[4 * s] = clock64();
      asm volatile("cp.async.wait_group %0;" ::"n"(PG - 1) : "memory");
      if (dbgstep && j == 0 && s < 1024) wf_dbg2[4 * s + 1] = clock64();
      long long pp;
      const bool act = active(s, pp);
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
      const double *rh = reinterpret_cast<const double *>(wbase + Lt::stage_slot(u, kWfEM, j));
      double ar, ai;
      if constexpr (FWD) {
        if constexpr (CX) {
          const double re0 = rh[0];
          const double im0 = *reinterpret_cast<const double *>(
              wbase + Lt::stage_slot(u, kWfEM + 1, j));
          ar = dadd(re0, dsub(dmul(0.0, im0), 0.0));  // numpy re + 1j*im
          ai = dadd(0.0, im0);
        } else {
          ar = rh[0];
          ai = 0.0;
        }
      } else {
        ar = rh[0];
        ai = CX ? rh[1] : 0.0;
        bad |= wf_sent<CX>(ar, ai);
      }
      double dr = 0.0, di = 0.0;
      if constexpr (!FWD) {
        const double *dv =
            reinterpret_cast<const double *>(recp(s) + Lt::kValOff + Lt::kVal);
        dr = dv[j * VW];
        di = CX ? dv[j * VW + 1] : 0.0;
      }
      // read ahead: the next step's record, the cols of step s + PG
      if (s + 1 < S) load_rec(s + 1);
      int coln[kWfEM];
      load_cols(s + PG, coln);
      if (dbgstep && j == 0 && s < 1024) wf_dbg2[4 * s + 2] = clock64();
      if (act && bad) {  // a prefetched value was not yet published
        const int row = FWD ? (int)pp : (int)(n - 1 - pp);
        const int *col = reinterpret_cast<const int *>(recp(s) + Lt::kOffB);
#pragma unroll
        for (int e = 0; e < kWfEM; ++e)
          if (wf_sent<CX>(vr[e], vi[e])) wf_poll<CX>(glob, col[e * 32 + j], vr[e], vi[e]);
        if (!FWD && wf_sent<CX>(ar, ai)) wf_poll<CX>(a.y, row, ar, ai);
      }
#pragma unroll
      for (int e = 0; e < kWfEM; ++e) wf_mulsub<CX>(ar, ai, cl[e], cm[e], vr[e], vi[e]);
      if constexpr (!FWD) {
        if constexpr (CX) {
          double qr, qi;
          py_cdiv(ar, ai, dr, di, qr, qi);
          ar = qr;
          ai = qi;
        } else {
          ar = ddiv(ar, dr);
        }
        if (act && (!isfin(ar) || !isfin(ai))) atomicOr(a.err, 1);
      }
      if (act) {
        double *rg = reinterpret_cast<double *>(wbase + Lt::ring_slot(s, j));
        rg[0] = ar;
        if constexpr (CX) rg[1] = ai;
        wf_pub<CX>(glob, FWD ? (int)pp : (int)(n - 1 - pp), ar, ai);
      }
      if (dbgstep && j == 0 && s < 1024) wf_dbg2[4 * s + 3] = clock64();
      prefetch(s + PG, u, coln);
      __syncwarp();
    }
    // chunk c consumed: refill its buffer with chunk c + NB
    if (j == 0 && c + kWfNB < nch) {
      const int b = (int)((cc + c) % kWfNB);
      wf_mbar_arrive_tx(&bar[b], cb);
      wf_bulk(buf + (size_t)b * bufsz, src + (size_t)(c + kWfNB) * cb, cb,
              &bar[b]);
    }
    __syncwarp();
  }
  cc += (unsigned)nch;
}

// diagnostics (MPK_WF_DEBUG=1): globaltimer at start / end of every group
__device__ long long wf_dbg[2 * 8192];

__device__ __forceinline__ long long wf_gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <bool CX>
__global__ void __launch_bounds__(128, 1)
    wsweep_kernel(SweepArgs a, WPhase F, WPhase B, int bufsz, int dbg) {
  if (a.done && *a.done) return;
  using Lt = WfLayout<CX>;
  extern __shared__ __align__(128) unsigned char wsm[];
  const int warp = threadIdx.x >> 5, j = threadIdx.x & 31;
  const size_t per_warp = Lt::kBufOff + (size_t)kWfNB * bufsz;
  unsigned char *base = wsm + (size_t)warp * per_warp;
  uint64_t *bar = reinterpret_cast<uint64_t *>(base);
  if (j == 0) {
    for (int b = 0; b < kWfNB; ++b) wf_mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (j < 4) reinterpret_cast<double *>(base + Lt::kZero)[j & 1] = 0.0;
  __syncwarp();
  unsigned cc = 0;
  const int gtot = F.ngroups + B.ngroups;
  for (;;) {
    int g = 0;
    if (j == 0) g = atomicAdd(a.tick, 1);
    g = __shfl_sync(kFullW, g, 0);
    if (g >= gtot) break;
    if (dbg && j == 0 && g < 8192) wf_dbg[2 * g] = wf_gtime();
    if (g < F.ngroups)
      wf_group<CX, true>(a, F, g, cc, bar, base, bufsz, dbg == 2 && g == 0);
    else
      wf_group<CX, false>(a, B, g - F.ngroups, cc, bar, base, bufsz, false);
    if (dbg && j == 0 && g < 8192) wf_dbg[2 * g + 1] = wf_gtime();
  }
  // last warp out resets the ticket for the next launch / graph replay
  __syncwarp();
  if (j == 0) {
    const int total = gridDim.x * (blockDim.x >> 5);
    __threadfence();
    if (atomicAdd(&a.tick[1], 1) == total - 1) {
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
      dst = P.rec + gs * P.recsz + kCode + (size_t)rem * VB;
    } else {
      const long long d = i - P.nslots;
      srcp = P.dsrc[d];
      dst = P.rec + (d / 32) * P.recsz + kCode + kVal + (d % 32) * VB;
    }
    if (cx) {
      const double2 v = srcp >= 0 ? reinterpret_cast<const double2 *>(lu)[srcp]
                                  : make_double2(0.0, 0.0);
      *reinterpret_cast<double2 *>(dst) = v;
    } else {
      *reinterpret_cast<double *>(dst) = srcp >= 0 ? lu[srcp] : 0.0;
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
  ph.recsz = 2 * kWfEM * 32 * 4 + kWfEM * 32 * VB + (fwd ? 0 : 32 * VB);
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
    const int PG = cx ? WfLayout<true>::PG : WfLayout<false>::PG;
    return cx ? WfLayout<true>::stage_slot((int)(s % PG), e, (int)j)
              : WfLayout<false>::stage_slot((int)(s % PG), e, (int)j);
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
  const int maxrec = std::max(w.f.recsz, w.b.recsz);
  (void)VB;
  const size_t bo = cx ? WfLayout<true>::kBufOff : WfLayout<false>::kBufOff;
  return bo + (size_t)kWfNB * kWfT * maxrec;
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
  const size_t lim_smem = 220 * 1024;
  int wpb = (int)std::min<size_t>(4, lim_smem / pw);
  if (wpb < 1) {
    free_wsweep(t);
    return false;
  }
  t.wpb = wpb;
  t.smem = pw * wpb;
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
    if (g > 148 * 16) g = 148 * 16;
    wf_gather_kernel<<<(unsigned)g, 256, 0, st>>>(lu, *P, cx ? 1 : 0);
  }
}

void launch_wsweep(const SweepArgs &a, const WSweep &w, bool cx,
                   cudaStream_t st) {
  ++tl_launches;
  static const int dbg = getenv("MPK_WF_DEBUG") ? atoi(getenv("MPK_WF_DEBUG")) : 0;
  const int bufsz = kWfT * std::max(w.f.recsz, w.b.recsz);
  const int gtot = w.f.ngroups + w.b.ngroups;
  int grid = (gtot + w.wpb - 1) / w.wpb;
  if (grid > 148) grid = 148;
  if (cx) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(wsweep_kernel<true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr = true;
    }
    wsweep_kernel<true><<<grid, 32 * w.wpb, w.smem, st>>>(a, w.f, w.b, bufsz, dbg);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(wsweep_kernel<false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr = true;
    }
    wsweep_kernel<false><<<grid, 32 * w.wpb, w.smem, st>>>(a, w.f, w.b, bufsz, dbg);
  }
}

}  // namespace mpk

// diagnostics for tools/: per-group globaltimer stamps of the last launch
extern "C" int mpk_wf_debug2(long long *out) {
  return cudaMemcpyFromSymbol(out, mpk::wf_dbg2, sizeof(long long) * 4096) == cudaSuccess ? 0 : 4;
}
extern "C" int mpk_wf_debug(long long *out, int n) {
  if (n > 2 * 8192) n = 2 * 8192;
  return cudaMemcpyFromSymbol(out, mpk::wf_dbg, sizeof(long long) * n) == cudaSuccess ? 0 : 4;
}
