// swf.cu -- shuffle-wavefront ("SWF") sweep plan for stencil-structured
// ILU(0) DAGs (real binary64 factors).
//
// Reference: ilu.py:322-343 (_sweep_forward / _sweep_backward) and
// :448-458 (the mixed apply): per row acc = rhs; acc = acc - L_ij*y_j over
// the row's entries in ascending column order; backward: acc / U_ii.  Each
// row is computed by one thread in exactly that order with _rn operations,
// so the result is bit for bit every other sweep path's (and the
// reference's); only the schedule is new.
//
// Schedule.  As in wf.cu the phase order (forward: rows ascending;
// backward: rows descending) is cut into "lines" of Lc consecutive
// positions, lane l runs line l in order, skewed `lag` steps behind lane
// l-1, 32 lanes per warp ("group").  The plan applies when every
// dependency of a row lies on the SAME line or on the PREVIOUS line, at
// most 4 steps back in the lane schedule -- a 5- or 9-point grid stencil
// in natural order (cfg1, cfg4).  Then a row's inputs are all in
// registers:
//   o[(s-d)&3]  the lane's own output of step s-d,
//   q[(s-d)&3]  the previous line's output of step s-d, delivered by one
//               __shfl_up per step (lane 0: from the previous warp's lane 31
//               through a shared-memory ring, or -- first warp of a CTA --
//               from global memory, prefetched a chunk ahead),
// and the entries of a row map to a fixed "key" list (previous-or-own line,
// steps back) in reference order, a compile-time pattern.  Entries a row
// lacks (grid boundary) read a slot whose source position is inactive
// (outside its line), which holds +0, with a 0 factor value: acc - 0*(+0)
// == acc bit for bit (the host analysis proves this for every row, else no
// plan).  Per step a lane then executes ~25 instructions: 2 LDS.128 of its
// row's factor values (staged per 8-step chunk by one TMA bulk copy per
// warp), one LDS of its right-hand side (cp.async 3 chunks ahead), the
// reference's multiply-subtract chain, the shuffle, one global store.  The
// critical path per step is shuffle + the entries that depend on the
// previous step (forward: 2 mul-sub; backward: 3 mul-sub + the division,
// Markstein-corrected from the precomputed RN reciprocal and proven RN by
// an exact residual test, else __ddiv_rn).
//
// CTAs of W warps (W consecutive groups, one warp per SM sub-partition)
// are claimed in order through a ticket: a CTA only waits on lower
// tickets, which are resident or done (deadlock-free for any grid).
// Inside a CTA the lane-31 -> lane-0 hand-off is a single-producer /
// single-consumer shared-memory ring whose empty slots hold the sentinel;
// across CTAs the consumer polls the previous line in global memory (values
// there start as the sentinel, set by the kernel that produced the input).
// Forward and backward phases are two launches, so the backward phase
// reads the forward result (its right-hand side) without polling.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "ilu.cuh"

namespace mpk {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kT = kSwfT;     // steps per chunk (record copy granularity)
constexpr int kNB = 3;        // record buffers per warp
constexpr int kR = 128;       // previous-line ring slots (power of two)
constexpr int kNF = 32;       // "producer chunk done" mbarriers per warp (power of two)

__device__ __forceinline__ uint32_t s_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void s_mbar_init(uint64_t *b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(cnt)
               : "memory");
}
__device__ __forceinline__ void s_mbar_arrive_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void s_mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "SWF_WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra SWF_WAIT%=;\n}\n" ::"r"(s_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void s_bulk(void *dst, const void *src, uint32_t bytes,
                                       uint64_t *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(b))
      : "memory");
}
__device__ __forceinline__ void s_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ double s_ldv(const double *p) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(s_u32(p)));
  return v;
}
__device__ __forceinline__ void s_stv(double *p, double v) {
  asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(s_u32(p)), "d"(v) : "memory");
}
__device__ __forceinline__ void s_mbar_arrive_rel(uint64_t *b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(s_u32(b))
               : "memory");
}
__device__ __forceinline__ int s_ldv_i(const int *p) {
  int v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(s_u32(p)));
  return v;
}
__device__ __forceinline__ void s_stv_i(int *p, int v) {
  asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(s_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ bool s_sent(double v) {
  return __double2hiint(v) == (int)(kSentBits >> 32);
}
__device__ __forceinline__ double g_poll(const double *p) {
  double v = ld_relaxed(p);
  while (s_sent(v)) {
    __nanosleep(40);
    v = ld_relaxed(p);
  }
  return v;
}
__device__ __forceinline__ void g_pub(double *p, double v) {
  // a result equal to the sentinel pattern (a NaN no operation produces
  // from finite data) is published as a quiet NaN
  const double w = s_sent(v) ? __longlong_as_double((long long)kQNaNBits) : v;
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(w) : "memory");
}

// a / d with the reference's RN semantics (= __ddiv_rn): Markstein
// correction of a * RN(1/d), then an exact residual test that proves the
// candidate is RN(a/d) (|a - q d| < |d| ulp(q)/2 with the residual exact by
// FMA); outside the safe exponent range, for q a power of two, or when the
// test fails the caller divides with __ddiv_rn.
__device__ __forceinline__ double s_fast_div(double a, double d, double r, bool &ok) {
  const double q0 = __dmul_rn(a, r);
  const double e0 = fma(-q0, d, a);
  const double q2 = fma(e0, r, q0);
  const double e2 = fma(-q2, d, a);
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

// a call the compiler cannot speculate across: keeps the exact re-run of a
// chunk on its (rare) branch instead of if-converted into every chunk
__device__ __noinline__ void swf_rerun_mark() { asm volatile("" ::: "memory"); }

// per-warp shared-memory region: record mbarriers | producer-chunk mbarriers
// | consumer progress | previous-line ring | rhs ring | records
constexpr int kRD = 3;            // rhs ring depth (chunks)
constexpr int kRhsRow = kT + 2;   // doubles per lane row (16-byte aligned)
struct SwfSmem {
  static constexpr int kBars = 0;
  static constexpr int kFull = 64;
  static constexpr int kProg = kFull + kNF * 8;
  static constexpr int kRing = kProg + 64;
  static constexpr int kRhs = kRing + kR * 8;
  static constexpr int kBuf = kRhs + kRD * 32 * kRhsRow * 8;
};

__host__ __device__ constexpr int swf_stepb(int nk, bool fwd) {
  return nk * 32 * 8 + (fwd ? 0 : 32 * 16);
}

// key e of a pattern: bit 2 = previous line, bits 0-1 = steps back - 1
template <int KEYS>
__host__ __device__ constexpr int key_of(int e) {
  return (KEYS >> (3 * e)) & 7;
}
// window depth: the most steps back any key reads
template <int NK, int KEYS>
__host__ __device__ constexpr int swf_depth() {
  int h = 1;
  for (int e = 0; e < NK; ++e)
    if ((key_of<KEYS>(e) & 3) + 1 > h) h = (key_of<KEYS>(e) & 3) + 1;
  return h;
}

// diagnostics (MPK_SWF_DEBUG=1): globaltimer at start / end of every group
__device__ long long swf_dbg[4 * 4096];
__device__ int swf_dbg_on;
__device__ int swf_dbgw[2][64];  // smid * 1000 + hardware warp slot of each group
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// chunk-level clock stamps of groups 0 and 1 (swf_dbg_on == 2): per chunk
// [top, after record wait, after rhs wait, after acquire, after steps, end]
__device__ long long swf_dbgc[2][2][512][6];

template <int NK, int KEYS, bool FWD>
__device__ __forceinline__ void swf_group(const SweepArgs &a, const SPhase &P, int g,
                                          int w, int W, unsigned char *wb,
                                          unsigned char *sm) {
  constexpr int STEPB = swf_stepb(NK, FWD);
  constexpr int H = swf_depth<NK, KEYS>();
  const int j = threadIdx.x & 31;
  const int n = a.n, Lc = P.Lc, lag = P.lag, nch = P.nch;
  const long long lbase = (long long)(g * 32 + j) * Lc;
  // active positions of this lane's line: [0, plim)
  const int plim = (g * 32 + j) < P.nlanes ? (int)min((long long)Lc, (long long)n - lbase) : 0;
  uint64_t *bars = reinterpret_cast<uint64_t *>(wb + SwfSmem::kBars);
  double *ring = reinterpret_cast<double *>(wb + SwfSmem::kRing);
  double *rhsb = reinterpret_cast<double *>(wb + SwfSmem::kRhs);
  unsigned char *buf = wb + SwfSmem::kBuf;
  const uint32_t cb = (uint32_t)P.chunkb;
  const unsigned char *src = P.rec + (size_t)g * nch * cb;
  double *out = FWD ? a.y : a.z;
  const double *rin = FWD ? a.in_re : a.y;
  // lane 31 feeds the next warp's ring when that group exists in this CTA:
  // every step it stores its result into the consumer's ring, and at the end
  // of each chunk it arrives on the consumer's "chunk done" mbarrier
  // (release); the consumer sleeps on it (try_wait).
  unsigned char *wnext = (w + 1 < W && g + 1 < P.ngroups)
                             ? sm + (size_t)(w + 1) * P.wbytes
                             : nullptr;
  double *ring_next = wnext ? reinterpret_cast<double *>(wnext + SwfSmem::kRing) : nullptr;
  uint64_t *full_next = wnext ? reinterpret_cast<uint64_t *>(wnext + SwfSmem::kFull) : nullptr;
  const int *prog_next = wnext ? reinterpret_cast<const int *>(wnext + SwfSmem::kProg) : nullptr;
  uint64_t *full_own = reinterpret_cast<uint64_t *>(wb + SwfSmem::kFull);
  int *prog_own = reinterpret_cast<int *>(wb + SwfSmem::kProg);
  const bool glob_prev = (w == 0);  // the previous line comes from global memory
  const bool has_prev = g > 0;
  const bool feed = (j == 31) && ring_next != nullptr;
  // global index of position p of the previous line (lane 0's view)
  const long long pbase = (long long)(g * 32 - 1) * Lc;
  auto prow = [&](int p) -> long long {
    const long long q = pbase + p;
    return FWD ? q : (long long)n - 1 - q;
  };
  auto prev_ok = [&](int p) { return has_prev && p >= 0 && p < Lc; };
  const bool r16 = P.rhs16 != 0;
  // producer chunk whose completion covers positions up to c*T + T - 1 + lag
  const int cshift = (32 * lag + kT - 1) / kT;

  // ---- record stream: kNB chunks in flight (TMA), L2 prefetch pf ahead ----
  const int pf = P.pf;
  auto rec_prefetch = [&](int c) {
    if (c < nch)
      for (int off = j * 128; off < (int)cb; off += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(src + (size_t)c * cb + off));
  };
  if (j == 0) {
    const int first = nch < kNB ? nch : kNB;
    for (int c = 0; c < first; ++c) {
      s_mbar_arrive_tx(bars + c, cb);
      s_bulk(buf + (size_t)c * cb, src + (size_t)c * cb, cb, bars + c);
    }
  }
  for (int c = kNB; c < pf; ++c) rec_prefetch(c);

  // ---- right-hand sides: chunk c's T positions of the lane, copied by
  // cp.async into a kRD-deep shared ring (one commit group per chunk, the
  // 16-byte copies of chunk c+2 spread over the steps of chunk c); position t
  // of a chunk sits at index t (forward) or T-1-t (backward: rows descend) ----
  auto rhs_slot = [&](int c) { return rhsb + ((c % kRD) * 32 + j) * kRhsRow; };
  auto rhs_full = [&](int c) {
    const int p0 = c * kT - lag * j;
    return r16 && c < nch && p0 >= 0 && p0 + kT <= plim;
  };
  auto rhs_gsrc = [&](int c) -> const double * {
    const int p0 = c * kT - lag * j;
    return FWD ? rin + lbase + p0 : rin + ((long long)n - kT - lbase - p0);
  };
  auto rhs_scalar = [&](int c) {  // partial / unaligned chunk: 8-byte copies
    if (c >= nch || rhs_full(c)) return;
    const int p0 = c * kT - lag * j;
    double *d0 = rhs_slot(c);
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int p = p0 + t;
      if (p >= 0 && p < plim) {
        const long long row = FWD ? lbase + p : (long long)n - 1 - lbase - p;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s_u32(d0 + (FWD ? t : kT - 1 - t))),
                     "l"(rin + row)
                     : "memory");
      }
    }
  };
  auto rhs_pair = [&](int c, int u) {  // 16-byte copy u of a full chunk
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s_u32(rhs_slot(c) + 2 * u)),
                 "l"(rhs_gsrc(c) + 2 * u)
                 : "memory");
  };
  auto rhs_issue_all = [&](int c) {
    if (rhs_full(c)) {
#pragma unroll
      for (int u = 0; u < kT / 2; ++u) rhs_pair(c, u);
    } else {
      rhs_scalar(c);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto rhs_prefetch = [&](int c) {
    const int p0 = c * kT - lag * j;
    if (c < nch && p0 + kT > 0 && p0 < plim) {
      const int pa = p0 < 0 ? 0 : p0;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(FWD ? rin + lbase + pa
                                                        : rin + ((long long)n - 1 - lbase - pa)));
    }
  };
  const int rpf = P.rpf;
  for (int c = 0; c < kRD - 1; ++c) rhs_issue_all(c);
  for (int c = kRD - 1; c <= rpf; ++c) rhs_prefetch(c);

  // ---- the previous line (lane 31 sends it to lane 0) ----
  // ring slot of position p: ring[p & (kR-1)].  Warp 0: lanes 0..T-1 load
  // chunk c+2's positions from global memory at the top of chunk c and store
  // them (checked: a sentinel is polled until published) at the top of chunk
  // c+1.  Other warps: the previous warp's lane 31 stores every result.
  double cv = 0.0;
  int cvp = -1;
  auto cross_load = [&](int c) {  // positions of chunk c: c*T + t + lag
    cvp = -1;
    if (glob_prev && has_prev && j < kT && c < nch) {
      const int p = c * kT + j + lag;
      if (p < Lc) {
        cvp = p;
        cv = ld_relaxed(out + prow(p));
      }
    }
  };
  auto cross_store = [&]() {  // the values loaded one chunk ago, checked
    if (cvp >= 0) {
      if (s_sent(cv)) {
        // not yet published when loaded: wait, and build slack by waiting
        // for the furthest position loaded so far too
        int pa = cvp + 2 * kT;
        if (pa >= Lc) pa = Lc - 1;
        g_poll(out + prow(pa));
        cv = g_poll(out + prow(cvp));
      }
      s_stv(ring + (cvp & (kR - 1)), cv);
    }
  };
  // consumer side (w >= 1): producer chunk cp done <=> its mbarrier phase cp
  auto wait_prod = [&](int cp) {
    if (cp >= nch) cp = nch - 1;
    if (!glob_prev && cp >= 0)
      s_mbar_wait(full_own + (cp & (kNF - 1)), (uint32_t)((cp / kNF) & 1));
  };
  double o[4] = {0.0, 0.0, 0.0, 0.0}, q[4] = {0.0, 0.0, 0.0, 0.0};
  if (glob_prev && has_prev) {
    // pre-roll (lag-H .. lag-1) and chunk 0 (lag .. lag+T-1), polled until
    // published; then wait 2 chunks further ahead so that the loads issued
    // from here on find published values
    const int p = lag - H + j;
    if (j < H + kT && prev_ok(p)) s_stv(ring + (p & (kR - 1)), g_poll(out + prow(p)));
    if (j == 0) {
      int pa = lag + 3 * kT - 1;
      if (pa >= Lc) pa = Lc - 1;
      g_poll(out + prow(pa));
    }
    cross_load(1);
  }
  wait_prod(cshift);  // the pre-roll and chunk 0's positions
  __syncwarp();
  {
    double pre[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int d = H; d >= 1; --d)
      if (prev_ok(lag - d)) pre[(4 - d) & 3] = s_ldv(ring + ((lag - d) & (kR - 1)));
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = j == 0 ? pre[u] : 0.0;
  }

  double lv[NK], dv = 1.0, dr = 1.0;
  auto load_step = [&](const unsigned char *rec, int t) {
#pragma unroll
    for (int e = 0; e < NK; e += 2) {
      const double2 v = reinterpret_cast<const double2 *>(rec + t * STEPB)[(e / 2) * 32 + j];
      lv[e] = v.x;
      lv[e + 1] = v.y;
    }
    if constexpr (!FWD) {
      const double2 v = reinterpret_cast<const double2 *>(rec + t * STEPB + NK * 32 * 8)[j];
      dv = v.x;
      dr = v.y;
    }
  };

  const bool dbc = swf_dbg_on == 2 && g < 2 && j == 0;
  long long *dbp = &swf_dbgc[FWD ? 0 : 1][g < 2 ? g : 0][0][0];
  for (int c = 0; c < nch; ++c) {
    const int p0 = c * kT - lag * j;  // this lane's position at step 0 of the chunk
    if (dbc && c < 512) dbp[c * 6] = clock64();
    s_mbar_wait(bars + (c % kNB), (uint32_t)((c / kNB) & 1));
    if (dbc && c < 512) dbp[c * 6 + 1] = clock64();
    asm volatile("cp.async.wait_group %0;" ::"n"(kRD - 2) : "memory");  // rhs(c) landed
    if (glob_prev && has_prev) {
      cross_store();  // chunk c+1's positions
      cross_load(c + 2);
    } else if (c > 0) {
      wait_prod(c + cshift);
    }
    if (pf) rec_prefetch(c + pf);
    if (rpf) rhs_prefetch(c + rpf);
    const bool fullnext = rhs_full(c + kRD - 1);
    if (!fullnext) rhs_scalar(c + kRD - 1);
    __syncwarp();
    if (dbc && c < 512) dbp[c * 6 + 2] = clock64();
    if (dbc && c < 512) dbp[c * 6 + 3] = clock64();
    const unsigned char *rec = buf + (size_t)(c % kNB) * cb;
    const double *rh = rhs_slot(c);
    double *op = out + (FWD ? lbase + p0 : (long long)n - 1 - lbase - p0);
    // lane 31: the previous line's value of step t (sent to lane 0)
    const int pc0 = c * kT + lag;
    // One chunk of T steps.  EXACT = false: the backward division uses the
    // Markstein quotient speculatively (its RN proof is accumulated in
    // `okall` off the critical path); the chunk's results are published
    // after the warp's proofs hold, else the chunk is re-run with EXACT =
    // true (__ddiv_rn) from the saved windows.  Stores and copies of other
    // chunks are interleaved into the steps' latency slots.
    auto run_chunk = [&](auto exact_tag, bool &okall, double (&xo)[kT], bool first) {
      constexpr bool EXACT = decltype(exact_tag)::value;
      load_step(rec, 0);
      double rr0 = 0.0, rr1 = 0.0;
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const bool act = (unsigned)(p0 + t) < (unsigned)plim;
        double l[NK];
#pragma unroll
        for (int e = 0; e < NK; ++e) l[e] = lv[e];
        const double d0 = dv, r0 = dr;
        if (t + 1 < kT) load_step(rec, t + 1);  // next step's values, off the chain
        if ((t & 1) == 0) {  // right-hand sides of steps t, t+1
          if constexpr (FWD) {  // position t at index t
            const double2 v = reinterpret_cast<const double2 *>(rh)[t / 2];
            rr0 = v.x;
            rr1 = v.y;
          } else {  // position t at index T-1-t
            const double2 v = reinterpret_cast<const double2 *>(rh)[(kT - 2 - t) / 2];
            rr0 = v.y;
            rr1 = v.x;
          }
        }
        if (first && fullnext && t < kT / 2) rhs_pair(c + kRD - 1, t);
        // previous line's value of this step, for lane 31 to send
        const int pc = pc0 + t;
        double av = 0.0;
        if (j == 31 && prev_ok(pc)) av = ring[pc & (kR - 1)];
        double acc = (t & 1) ? rr1 : rr0;
#pragma unroll
        for (int e = 0; e < NK; ++e) {
          const int key = key_of<KEYS>(e);
          const int d = (key & 3) + 1;
          const double v = (key & 4) ? q[(t - d) & 3] : o[(t - d) & 3];
          acc = __dsub_rn(acc, __dmul_rn(l[e], v));
        }
        double x = acc;
        if constexpr (!FWD) {
          if constexpr (EXACT) {
            x = __ddiv_rn(acc, d0);
          } else {
            bool ok;
            x = s_fast_div(acc, d0, r0, ok);
            okall &= ok || !act;
          }
        }
        const double xv = act ? x : 0.0;
        o[t & 3] = xv;
        q[t & 3] = __shfl_sync(kFull, (act && j != 31) ? x : av, (j + 31) & 31);
        if constexpr (FWD) {  // publish in the step's latency slots
          if (act) {
            asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(op + t), "d"(xv)
                         : "memory");
            if (feed) ring_next[(p0 + t) & (kR - 1)] = xv;
          }
        } else {
          xo[t] = xv;
        }
      }
    };
    bool okall = true;
    double xo[kT];
    if constexpr (FWD) {
      run_chunk(std::false_type{}, okall, xo, true);
    } else {
      double os[4], qs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        os[u] = o[u];
        qs[u] = q[u];
      }
      run_chunk(std::false_type{}, okall, xo, true);
      if (swf_dbg_on == 3) okall = false;  // test hook: force the exact re-run
      if (__any_sync(kFull, !okall)) {     // rare: some quotient not proven RN
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          o[u] = os[u];
          q[u] = qs[u];
        }
        swf_rerun_mark();
        run_chunk(std::true_type{}, okall, xo, false);
      }
      // publish the proven chunk (non-finite results: NumericBreakdownError)
      double nfin = 0.0;
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        if ((unsigned)(p0 + t) < (unsigned)plim) {
          asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(op - t), "d"(xo[t])
                       : "memory");
          if (feed) ring_next[(p0 + t) & (kR - 1)] = xo[t];
        }
        nfin = fma(xo[t], 0.0, nfin);
      }
      if (!isfinite(nfin)) atomicOr(a.err, 1);
    }
    if (dbc && c < 512) dbp[c * 6 + 4] = clock64();
    asm volatile("cp.async.commit_group;" ::: "memory");  // rhs(c + kRD - 1)
    if (feed) {
      // throttle: the consumer must have taken the ring slots the next
      // chunks overwrite, and must not fall kNF phases behind
      while (c + 1 > s_ldv_i(prog_next) + cshift + 6) __nanosleep(64);
      s_mbar_arrive_rel(full_next + (c & (kNF - 1)));
    }
    if (!glob_prev && j == 31) s_stv_i(prog_own, c);  // ring positions of chunk c consumed
    __syncwarp();
    if (dbc && c < 512) dbp[c * 6 + 5] = clock64();
    // record chunk c consumed: refill its buffer with chunk c + kNB
    if (j == 0 && c + kNB < nch) {
      const int b = c % kNB;
      s_mbar_arrive_tx(bars + b, cb);
      s_bulk(buf + (size_t)b * cb, src + (size_t)(c + kNB) * cb, cb, bars + b);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}


template <int NK, int KEYS, bool FWD>
__global__ void __launch_bounds__(32 * kSwfMaxW, 1)
    swf_kernel(SweepArgs a, SPhase P, int W) {
  __shared__ int s_tick;
  int *tick = a.tick;
  {  // stopped solve: skip, but count this CTA out (ticket reset)
    int d = 0;
    if (threadIdx.x == 0 && a.done) d = *(volatile const int *)a.done;
    d = __syncthreads_or(d);
    if (d) {
      if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&tick[1], 1) == (int)gridDim.x - 1) {
          atomicExch(&tick[0], 0);
          atomicExch(&tick[1], 0);
        }
      }
      return;
    }
  }
  extern __shared__ __align__(128) unsigned char sm[];
  const int w = threadIdx.x >> 5, j = threadIdx.x & 31;
  unsigned char *wb = sm + (size_t)w * P.wbytes;
  const int nct = (P.ngroups + W - 1) / W;
  for (;;) {
    if (threadIdx.x == 0) s_tick = atomicAdd(tick, 1);
    // fresh ring and barriers per ticket (no copy is pending here)
    double *ring = reinterpret_cast<double *>(wb + SwfSmem::kRing);
#pragma unroll
    for (int u = 0; u < kR / 32; ++u) ring[j + 32 * u] = sent_val();
    if (j == 0) {
      uint64_t *bars = reinterpret_cast<uint64_t *>(wb + SwfSmem::kBars);
      for (int b = 0; b < kNB; ++b) s_mbar_init(bars + b, 1);
      uint64_t *full = reinterpret_cast<uint64_t *>(wb + SwfSmem::kFull);
      for (int b = 0; b < kNF; ++b) s_mbar_init(full + b, 1);
      *reinterpret_cast<int *>(wb + SwfSmem::kProg) = -1;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const int t = s_tick;
    if (t >= nct) break;
    const int g = t * W + w;
    if (g < P.ngroups) {
      if (swf_dbg_on && j == 0 && g < 4096) {
        unsigned wid, smid;
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        swf_dbg[(FWD ? 0 : 2 * 4096) + 2 * g] = gtimer();
        if (g < 64) swf_dbgw[FWD ? 0 : 1][g] = (int)(smid * 1000 + wid);
      }
      swf_group<NK, KEYS, FWD>(a, P, g, w, W, wb, sm);
      if (swf_dbg_on && j == 0 && g < 4096)
        swf_dbg[(FWD ? 0 : 2 * 4096) + 2 * g + 1] = gtimer();
    }
    __syncthreads();
  }
  // last CTA out resets the ticket for the next launch / graph replay
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&tick[1], 1) == (int)gridDim.x - 1) {
      atomicExch(&tick[0], 0);
      atomicExch(&tick[1], 0);
    }
  }
}

// record values: esrc / dsrc -> chunk layout (see SPhase)
__global__ void swf_gather_kernel(const double *lu, SPhase P) {
  const int NK = P.nk;
  const int stepb = swf_stepb(NK, P.fwd != 0);
  const long long tot = P.nslots + P.ndslots;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    if (i < P.nslots) {
      const long long gs = i / (NK * 32);  // group * S + step
      const int rem = (int)(i % (NK * 32));
      const int e = rem / 32, jj = rem % 32;
      const long long g = gs / P.S;
      const int s = (int)(gs % P.S);
      unsigned char *dst = P.rec + ((size_t)g * P.nch + s / kT) * P.chunkb +
                           (size_t)(s % kT) * stepb;
      const int srcp = P.esrc[i];
      reinterpret_cast<double *>(dst)[((e / 2) * 32 + jj) * 2 + (e & 1)] =
          srcp >= 0 ? lu[srcp] : 0.0;
    } else {
      const long long d = i - P.nslots;
      const long long gs = d / 32;
      const int jj = (int)(d % 32);
      const long long g = gs / P.S;
      const int s = (int)(gs % P.S);
      unsigned char *dst = P.rec + ((size_t)g * P.nch + s / kT) * P.chunkb +
                           (size_t)(s % kT) * stepb + NK * 32 * 8;
      const int srcp = P.dsrc[d];
      const double v = srcp >= 0 ? lu[srcp] : 1.0;
      reinterpret_cast<double2 *>(dst)[jj] = make_double2(v, __drcp_rn(v));
    }
  }
}

// ------------------------------------------------------------------
// host analysis
// ------------------------------------------------------------------
// Canonical key lists of the instantiated patterns (reference entry order =
// ascending columns).  Key = 4 * previous_line + (steps_back - 1).
struct Pattern {
  int nk;
  int keys[4];
};
constexpr Pattern kPat[] = {
    {4, {4 + 2, 4 + 1, 4 + 0, 0}},  // 9-point forward: SW, S, SE, W
    {4, {0, 4 + 0, 4 + 1, 4 + 2}},  // 9-point backward: E, NW, N, NE
    {2, {4 + 0, 0, 0, 0}},          // 5-point forward: S, W
    {2, {0, 4 + 0, 0, 0}},          // 5-point backward: E, N
};
constexpr int kNPat = 4;

template <class Deps>
static bool analyse_phase(SPhase &ph, int n, bool fwd, Deps deps, long long &cost) {
  long long D = 0;
  for (int p = 0; p < n; ++p)
    deps(p, [&](int pq, int) {
      if (p - pq > D) D = p - pq;
    });
  if (D < 2) return false;
  bool found = false;
  cost = LLONG_MAX;
  for (long long Lc : {D - 1, D, D + 1, D - 2}) {
    if (Lc < 2 || Lc > n) continue;
    const long long nl = (n + Lc - 1) / Lc;
    if (nl < 2) continue;
    // lag: a previous-line dependency at posq needs posq - pos + lag >= 1
    long long lag = 1;
    bool ok = true;
    for (int p = 0; p < n && ok; ++p) {
      const long long l = p / Lc, pos = p % Lc;
      deps(p, [&](int pq, int) {
        const long long lq = pq / Lc, posq = pq % Lc;
        if (lq == l) return;
        if (lq != l - 1) {
          ok = false;
          return;
        }
        if (posq - pos + 1 > lag) lag = posq - pos + 1;
      });
    }
    if (!ok || lag > 3) continue;
    // the entries of every row must follow one pattern's key list
    int pat = -1;
    for (int k = 0; k < kNPat && pat < 0; ++k) {
      const Pattern &P = kPat[k];
      bool good = true;
      for (int p = 0; p < n && good; ++p) {
        const long long l = p / Lc, pos = p % Lc;
        int e = 0;  // next key of the pattern to match
        bool used[4] = {false, false, false, false};
        deps(p, [&](int pq, int) {
          if (!good) return;
          const long long lq = pq / Lc, posq = pq % Lc;
          const long long dl = l - lq;
          const long long ds = dl ? pos - posq + lag : pos - posq;
          if (ds < 1 || ds > 4) {
            good = false;
            return;
          }
          const int key = (int)(4 * dl + ds - 1);
          while (e < P.nk && P.keys[e] != key) ++e;
          if (e == P.nk) {
            good = false;
            return;
          }
          used[e++] = true;
        });
        // unused keys must read an inactive source (+0)
        for (int e2 = 0; e2 < P.nk && good; ++e2) {
          if (used[e2]) continue;
          const int dl = P.keys[e2] >> 2, ds = (P.keys[e2] & 3) + 1;
          const long long ls = l - dl;
          const long long posq = dl ? pos - ds + lag : pos - ds;
          const bool inactive = ls < 0 || posq < 0 || posq >= Lc || ls * Lc + posq >= n;
          if (!inactive) good = false;
        }
      }
      if (good) pat = k;
    }
    if (pat < 0) continue;
    const long long ng = (nl + 31) / 32;
    const long long S = Lc + lag * 31;
    const long long c = ng * 32 * lag + S;
    if (c < cost) {
      cost = c;
      found = true;
      ph.fwd = fwd ? 1 : 0;
      ph.Lc = (int)Lc;
      ph.lag = (int)lag;
      ph.nlanes = (int)nl;
      ph.ngroups = (int)ng;
      ph.S = (int)((S + kT - 1) / kT * kT);
      ph.nch = ph.S / kT;
      ph.pat = pat;
      ph.nk = kPat[pat].nk;
    }
  }
  return found;
}

template <class Deps, class Div>
static bool build_phase(SPhase &ph, int n, Deps deps, Div div, cudaStream_t st) {
  const bool fwd = ph.fwd != 0;
  const int NK = ph.nk;
  const Pattern &P = kPat[ph.pat];
  const long long nsteps = (long long)ph.ngroups * ph.S;
  ph.nslots = nsteps * NK * 32;
  ph.ndslots = fwd ? 0 : nsteps * 32;
  ph.chunkb = kT * swf_stepb(NK, fwd);
  ph.rhs16 = (ph.Lc % 2 == 0 && ph.lag % 2 == 0 && (fwd || n % 2 == 0)) ? 1 : 0;
  std::vector<int> esrc((size_t)ph.nslots, -1), dsrc((size_t)ph.ndslots, -1);
  const long long Lc = ph.Lc, lag = ph.lag;
  for (int p = 0; p < n; ++p) {
    const long long l = p / Lc, pos = p % Lc;
    const long long g = l / 32, j = l % 32;
    const long long s = pos + lag * j;
    const long long gs = g * ph.S + s;
    int e = 0;
    deps(p, [&](int pq, int lu_idx) {
      const long long lq = pq / Lc, posq = pq % Lc;
      const long long dl = l - lq;
      const long long ds = dl ? pos - posq + lag : pos - posq;
      const int key = (int)(4 * dl + ds - 1);
      while (P.keys[e] != key) ++e;  // analysed: always found
      esrc[(size_t)((gs * NK + e) * 32 + j)] = lu_idx;
      ++e;
    });
    if (!fwd) dsrc[(size_t)(gs * 32 + j)] = div(p);
  }
  auto up = [&](void **d, const void *h, size_t bytes) {
    if (cudaMalloc(d, bytes < 16 ? 16 : bytes) != cudaSuccess) return false;
    return cudaMemcpyAsync(*d, h, bytes, cudaMemcpyHostToDevice, st) == cudaSuccess;
  };
  const size_t recb = (size_t)ph.ngroups * ph.nch * ph.chunkb;
  bool good = cudaMalloc((void **)&ph.rec, recb) == cudaSuccess &&
              cudaMemsetAsync(ph.rec, 0, recb, st) == cudaSuccess &&
              up((void **)&ph.esrc, esrc.data(), esrc.size() * sizeof(int));
  if (!fwd) good = good && up((void **)&ph.dsrc, dsrc.data(), dsrc.size() * sizeof(int));
  cudaStreamSynchronize(st);
  return good;
}

static void free_phase(SPhase &ph) {
  if (ph.rec) cudaFree(ph.rec);
  if (ph.esrc) cudaFree(ph.esrc);
  if (ph.dsrc) cudaFree(ph.dsrc);
  ph = SPhase{};
}

template <int PAT, bool FWD>
static void launch_pat(const SweepArgs &a, const SPhase &P, int W, int grid, size_t smem,
                       cudaStream_t st) {
  constexpr Pattern pt = kPat[PAT];
  constexpr int KEYS =
      pt.keys[0] | (pt.keys[1] << 3) | (pt.keys[2] << 6) | (pt.keys[3] << 9);
  auto *fn = swf_kernel<pt.nk, KEYS, FWD>;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  fn<<<grid, 32 * W, smem, st>>>(a, P, W);
}

static void launch_phase(const SweepArgs &a, const SPhase &P, int W, int grid, size_t smem,
                         cudaStream_t st) {
  const bool f = P.fwd != 0;
  switch (P.pat) {
    case 0:
      f ? launch_pat<0, true>(a, P, W, grid, smem, st)
        : launch_pat<0, false>(a, P, W, grid, smem, st);
      break;
    case 1:
      f ? launch_pat<1, true>(a, P, W, grid, smem, st)
        : launch_pat<1, false>(a, P, W, grid, smem, st);
      break;
    case 2:
      f ? launch_pat<2, true>(a, P, W, grid, smem, st)
        : launch_pat<2, false>(a, P, W, grid, smem, st);
      break;
    default:
      f ? launch_pat<3, true>(a, P, W, grid, smem, st)
        : launch_pat<3, false>(a, P, W, grid, smem, st);
      break;
  }
}

}  // namespace

void free_ssweep(SSweep &w) {
  free_phase(w.f);
  free_phase(w.b);
  w = SSweep{};
}

bool build_ssweep(SSweep &w, int n, bool cx, const int *rp, const int *ci, const int *dp,
                  cudaStream_t st) {
  const char *ev = getenv("MPK_SSWEEP");
  if ((ev && ev[0] == '0') || cx || n < 256) return false;
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
  SSweep t;
  long long cf = 0, cbk = 0;
  if (!analyse_phase(t.f, n, true, fdeps, cf) || !analyse_phase(t.b, n, false, bdeps, cbk))
    return false;
  if (!build_phase(t.f, n, fdeps, [](int) { return -1; }, st) ||
      !build_phase(t.b, n, bdeps, [&](int p) { return dp[n - 1 - p]; }, st)) {
    free_ssweep(t);
    return false;
  }
  const char *ew = getenv("MPK_SSWEEP_W");
  int W = ew ? atoi(ew) : kSwfMaxW;
  if (W < 1) W = 1;
  if (W > kSwfMaxW) W = kSwfMaxW;
  const int maxg = std::max(t.f.ngroups, t.b.ngroups);
  if (W > maxg) W = maxg;
  const int chunkmax = std::max(t.f.chunkb, t.b.chunkb);
  const int wbytes = (SwfSmem::kBuf + kNB * chunkmax + 127) / 128 * 128;
  t.f.wbytes = t.b.wbytes = wbytes;
  t.W = W;
  t.smem = (size_t)W * wbytes;
  if (t.smem > 220 * 1024) {
    free_ssweep(t);
    return false;
  }
  const char *er = getenv("MPK_SWF_RPF");
  t.f.rpf = t.b.rpf = er ? atoi(er) : 4;
  const char *ep = getenv("MPK_SWF_PF");
  t.f.pf = t.b.pf = ep ? atoi(ep) : 8;
  t.cost = cf + cbk;
  t.on = 1;
  w = t;
  return true;
}

void gather_ssweep(const double *lu, const SSweep &w, cudaStream_t st) {
  if (!w.on) return;
  for (const SPhase *P : {&w.f, &w.b}) {
    const long long tot = P->nslots + P->ndslots;
    if (tot <= 0) continue;
    ++tl_launches;
    long long g = (tot + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    swf_gather_kernel<<<(unsigned)g, 256, 0, st>>>(lu, *P);
  }
}

void launch_ssweep(const SweepArgs &a, const SSweep &w, cudaStream_t st) {
  static const int only_g0 = getenv("MPK_SWF_ONLY_G0") ? atoi(getenv("MPK_SWF_ONLY_G0")) : 0;
  for (const SPhase *P : {&w.f, &w.b}) {
    ++tl_launches;
    SPhase Q = *P;
    if (only_g0) Q.ngroups = only_g0;  // diagnostics: timing of the first groups alone
    int grid = (Q.ngroups + w.W - 1) / w.W;
    if (grid > 148) grid = 148;
    launch_phase(a, Q, w.W, grid, w.smem, st);
  }
}

}  // namespace mpk

// diagnostics for tools/: per-group globaltimer stamps of the last launches
extern "C" int mpk_swf_debugw(int *out) {
  return cudaMemcpyFromSymbol(out, mpk::swf_dbgw, sizeof(int) * 128) == cudaSuccess ? 0 : 4;
}
extern "C" int mpk_swf_debugc(long long *out) {
  return cudaMemcpyFromSymbol(out, mpk::swf_dbgc, sizeof(long long) * 2 * 2 * 512 * 6) ==
                 cudaSuccess
             ? 0
             : 4;
}
extern "C" int mpk_swf_debug(long long *out, int on) {
  if (cudaMemcpyToSymbol(mpk::swf_dbg_on, &on, sizeof(int)) != cudaSuccess) return 4;
  if (!out) return 0;
  return cudaMemcpyFromSymbol(out, mpk::swf_dbg, sizeof(long long) * 4 * 4096) == cudaSuccess
             ? 0
             : 4;
}
