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
#include <atomic>
#include <thread>
#include <type_traits>
#include <vector>

#include "ilu.cuh"

namespace mpk {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kT = kSwfT;     // steps per chunk (record copy granularity)
constexpr int kNB = 4;        // record buffers (TMA) per group
constexpr int kR = 128;       // previous-line ring slots (power of two)

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
__device__ __forceinline__ uint32_t s_mapa(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(s_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void c_st_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void c_st_u32(uint32_t addr, int v) {
  asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v)
               : "memory");
}
__device__ __forceinline__ void c_arrive_rel(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
               : "memory");
}
__device__ __forceinline__ void s_mbar_wait_cl(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "SWF_WAITC%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra SWF_WAITC%=;\n}\n" ::"r"(s_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ int s_ld_acq_i(const int *p) {
  int v;
  // relaxed (an acquire at cluster scope costs a GPU-scope MEMBAR): the
  // consumer stores its progress after its ring reads have been used
  asm volatile("ld.relaxed.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(s_u32(p))
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
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

// Split form of s_fast_div: the Markstein candidate (on the dependency
// chain) and its RN proof (evaluated later, off the chain).
__device__ __forceinline__ double s_markstein(double a, double d, double r) {
  const double q0 = __dmul_rn(a, r);
  const double e0 = fma(-q0, d, a);
  return fma(e0, r, q0);
}
// Branch-free (no short circuits: the compiler must not put a branch
// between a step's quotient and its shuffle).  Exponent fields in
// (256, 1792): no under/overflow anywhere in the test; q not a power of
// two (symmetric ulp); then q == RN(a/d) iff |a - q d| < |d| ulp(q)/2.
__device__ __forceinline__ bool s_rn_proof(double a, double d, double q2) {
  const double e2 = fma(-q2, d, a);
  const unsigned qh = (unsigned)__double2hiint(q2), ql = (unsigned)__double2loint(q2);
  const unsigned ah = (unsigned)__double2hiint(a), dh = (unsigned)__double2hiint(d);
  const unsigned eq = (qh >> 20) & 0x7ff, ea = (ah >> 20) & 0x7ff, ed = (dh >> 20) & 0x7ff;
  const unsigned range = (unsigned)(eq - 257u < 1535u) & (unsigned)(ea - 257u < 1535u) &
                         (unsigned)(ed - 257u < 1535u);
  const unsigned frac = (unsigned)(((qh & 0xFFFFFu) | ql) != 0u);
  const double half_ulp = __hiloint2double((int)((eq - 53u) << 20), 0);
  const unsigned tight = (unsigned)(fabs(e2) < __dmul_rn(fabs(d), half_ulp));
  return (range & frac & tight) != 0u;
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

// Shared memory of one CTA (= one group: a compute warp and a helper warp):
// record mbarriers | ready / done mbarriers | previous-line ring | rhs
// staging | output staging | record buffers (TMA)
constexpr int kQ = 4;             // output staging depth / ready-done barriers (chunks)
constexpr int kQR = 6;            // rhs staging depth (chunks): requested kQR-1 ahead
constexpr int kNU = 16;           // upstream-chunk mbarriers (DSMEM hand-off)
constexpr int kRow = kT + 2;      // doubles per lane row (16-byte aligned)
struct SwfSmem {
  static constexpr int kRec = 0;                   // kNB mbarriers
  static constexpr int kReady = 64;                // kQ mbarriers
  static constexpr int kDone = kReady + kQ * 8;    // kQ mbarriers
  static constexpr int kUp = kDone + kQ * 8;       // kNU mbarriers (cluster hand-off)
  static constexpr int kProg = kUp + kNU * 8;      // downstream progress (int)
  static constexpr int kRing = (kProg + 8 + 127) / 128 * 128;
  static constexpr int kRhs = kRing + kR * 8;
  static constexpr int kOut = kRhs + kQR * 32 * kRow * 8;
  static constexpr int kBuf = (kOut + kQ * 32 * kRow * 8 + 127) / 128 * 128;
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
// chunk-level clock stamps of groups 0 and 1 (swf_dbg_on == 2), compute
// warp: [top, after ready wait, after record wait, after steps, after
// publish to staging, end]
__device__ long long swf_dbgc[2][2][512][6];

// Geometry of one group shared by its two warps.
struct SwfGeo {
  int n, Lc, lag, nch, g;
  int j;               // lane (= line within the group)
  long long lbase;     // global position of the lane's line start
  int plim;            // active positions of the line: [0, plim)
  bool has_prev;       // the group's first line has a predecessor
  long long pbase;     // global position of the previous line's start
  __device__ __forceinline__ SwfGeo(const SweepArgs &a, const SPhase &P, int g_) {
    n = a.n;
    Lc = P.Lc;
    lag = P.lag;
    nch = P.nch;
    g = g_;
    j = threadIdx.x & 31;
    lbase = (long long)(g * 32 + j) * Lc;
    plim = (g * 32 + j) < P.nlanes ? (int)min((long long)Lc, (long long)n - lbase) : 0;
    has_prev = g > 0;
    pbase = (long long)(g * 32 - 1) * Lc;
  }
};

// ---------------------------------------------------------------------
// compute warp: the rows of the group's 32 lines, T steps per chunk
// ---------------------------------------------------------------------
template <int NK, int KEYS, bool FWD>
__device__ __forceinline__ void swf_compute(const SweepArgs &a, const SPhase &P, int g,
                                            int rank, unsigned char *sm) {
  constexpr int STEPB = swf_stepb(NK, FWD);
  const SwfGeo G(a, P, g);
  const int j = G.j, lag = G.lag, nch = G.nch, Lc = G.Lc;
  // thread-block cluster hand-off (P.cl > 1): the previous group runs in
  // the CTA of cluster rank - 1 and stores its last line into this CTA's
  // ring (distributed shared memory), one mbarrier arrival per chunk; this
  // CTA's lane 31 feeds rank + 1 the same way.  Rank 0's previous line
  // comes from global memory (helper warp).
  const bool dsm_in = P.cl > 1 && rank > 0 && G.has_prev;
  uint64_t *up = reinterpret_cast<uint64_t *>(sm + SwfSmem::kUp);
  const int cshift = (32 * lag + kT - 1) / kT;  // upstream chunk covering a chunk's needs
  constexpr int HD = swf_depth<NK, KEYS>();
  uint32_t r_prog = 0;
  if (dsm_in) r_prog = s_mapa(sm + SwfSmem::kProg, (uint32_t)rank - 1);
  uint64_t *rec_bar = reinterpret_cast<uint64_t *>(sm + SwfSmem::kRec);
  uint64_t *ready = reinterpret_cast<uint64_t *>(sm + SwfSmem::kReady);
  uint64_t *done = reinterpret_cast<uint64_t *>(sm + SwfSmem::kDone);
  const double *ring = reinterpret_cast<const double *>(sm + SwfSmem::kRing);
  unsigned char *buf = sm + SwfSmem::kBuf;
  const uint32_t cb = (uint32_t)P.chunkb;
  double o[4] = {0.0, 0.0, 0.0, 0.0}, q[4] = {0.0, 0.0, 0.0, 0.0};
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
    const int sq = c % kQ;
    if (dbc && c < 512) dbp[c * 6] = clock64();
    s_mbar_wait(ready + sq, (uint32_t)((c / kQ) & 1));  // rhs(c) staged, ring(c) filled
    if (dsm_in) {  // the upstream chunk whose results cover this chunk
      const int cp = c + cshift < nch ? c + cshift : nch - 1;
      s_mbar_wait_cl(up + (cp % kNU), (uint32_t)((cp / kNU) & 1));
    }
    if (dbc && c < 512) dbp[c * 6 + 1] = clock64();
    if (c == 0) {
      // the window's previous-line entries before step 0 (pre-roll)
      double pre[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int d = HD; d >= 1; --d)
        pre[(4 - d) & 3] = (G.has_prev && lag - d >= 0) ? ring[(lag - d + 31 * lag) & (kR - 1)] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = j == 0 ? pre[u] : 0.0;
    }
    // (the records' TMA completion was observed by the helper before ready)
    if (dbc && c < 512) dbp[c * 6 + 2] = clock64();
    const unsigned char *rec = buf + (size_t)(c % kNB) * cb;
    const double *rh =
        reinterpret_cast<const double *>(sm + SwfSmem::kRhs) + ((c % kQR) * 32 + j) * kRow;
    double *ob = reinterpret_cast<double *>(sm + SwfSmem::kOut) + (sq * 32 + j) * kRow;
    const int pc0 = c * kT + lag;  // previous line's position of step 0 (lane 0's view)
    // One chunk of T steps.  EXACT = false: the backward division uses the
    // Markstein quotient speculatively (its RN proof is accumulated in
    // `okall` off the critical path); the results are handed to the helper
    // only after the warp's proofs hold, else the chunk is re-run with
    // EXACT = true (__ddiv_rn) from the saved windows.
    auto run_chunk = [&](auto exact_tag, bool &okall, double (&xo)[kT]) {
      constexpr bool EXACT = decltype(exact_tag)::value;
      load_step(rec, 0);
      double rr0 = 0.0, rr1 = 0.0;
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const bool act = (unsigned)(p0 + t) < (unsigned)G.plim;
        double l[NK];
#pragma unroll
        for (int e = 0; e < NK; ++e) l[e] = lv[e];
        const double d0 = dv, r0 = dr;
        if (t + 1 < kT) load_step(rec, t + 1);  // next step's values, off the chain
        if ((t & 1) == 0) {  // right-hand sides of steps t, t+1 (position order)
          const double2 v = reinterpret_cast<const double2 *>(rh)[t / 2];
          rr0 = v.x;
          rr1 = v.y;
        }
        // lane 31 sends the previous line's value of this step to lane 0
        const double av =
            (G.has_prev && (unsigned)(pc0 + t) < (unsigned)Lc) ? ring[(pc0 + t + 31 * lag) & (kR - 1)] : 0.0;
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
            x = s_markstein(acc, d0, r0);
          }
        }
        const double xv = act ? x : 0.0;
        o[t & 3] = xv;
        q[t & 3] = __shfl_sync(kFull, (act && j != 31) ? x : av, (j + 31) & 31);
        if constexpr (FWD) {
          ob[t] = xv;  // to the helper's output staging
        } else {
          xo[t] = xv;
          if constexpr (!EXACT) {
            // the RN proof of this step's quotient, after its shuffle: off
            // the dependency chain of the next step
            okall = okall & ((!act) | s_rn_proof(acc, d0, x));
          }
        }
      }
    };
    bool okall = true;
    double xo[kT];
    if constexpr (FWD) {
      run_chunk(std::false_type{}, okall, xo);
    } else {
      double os[4], qs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        os[u] = o[u];
        qs[u] = q[u];
      }
      run_chunk(std::false_type{}, okall, xo);
      if (swf_dbg_on == 3) okall = false;  // test hook: force the exact re-run
      if (__any_sync(kFull, !okall)) {     // rare: some quotient not proven RN
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          o[u] = os[u];
          q[u] = qs[u];
        }
        swf_rerun_mark();
        run_chunk(std::true_type{}, okall, xo);
      }
      double nfin = 0.0;  // NaN iff a result is non-finite (NumericBreakdownError)
#pragma unroll
      for (int t = 0; t < kT; t += 2) {
        reinterpret_cast<double2 *>(ob)[t / 2] = make_double2(xo[t], xo[t + 1]);
        nfin = fma(xo[t], 0.0, fma(xo[t + 1], 0.0, nfin));
      }
      if (!isfinite(nfin)) atomicOr(a.err, 1);
    }
    if (dbc && c < 512) dbp[c * 6 + 3] = clock64();
    if (dsm_in && j == 31) c_st_u32(r_prog, c);  // ring positions of chunk c consumed
    if (dbc && c < 512) dbp[c * 6 + 4] = clock64();
    s_mbar_arrive_rel(done + sq);  // (count 32) outputs staged, buffers free
    if (dbc && c < 512) dbp[c * 6 + 5] = clock64();
  }
}

// ---------------------------------------------------------------------
// helper warp: records (TMA), right-hand sides (cp.async), the previous
// line (polled in global memory), publication of the results
// ---------------------------------------------------------------------
template <bool FWD>
__device__ __forceinline__ void swf_helper(const SweepArgs &a, const SPhase &P, int g,
                                           int rank, unsigned char *sm) {
  const SwfGeo G(a, P, g);
  // previous line from the upstream CTA of the cluster (no polling here);
  // the group's last line sent to the downstream CTA of the cluster
  const bool dsm_in = P.cl > 1 && rank > 0 && G.has_prev;
  const bool dsm_out = P.cl > 1 && rank + 1 < P.cl && g + 1 < P.ngroups;
  uint32_t r_ring = 0, r_up = 0;
  if (dsm_out) {
    r_ring = s_mapa(sm + SwfSmem::kRing, (uint32_t)rank + 1);
    r_up = s_mapa(sm + SwfSmem::kUp, (uint32_t)rank + 1);
  }
  const int *prog = reinterpret_cast<const int *>(sm + SwfSmem::kProg);
  const int j = G.j, lag = G.lag, nch = G.nch, n = G.n, Lc = G.Lc;
  uint64_t *rec_bar = reinterpret_cast<uint64_t *>(sm + SwfSmem::kRec);
  uint64_t *ready = reinterpret_cast<uint64_t *>(sm + SwfSmem::kReady);
  uint64_t *done = reinterpret_cast<uint64_t *>(sm + SwfSmem::kDone);
  double *ring = reinterpret_cast<double *>(sm + SwfSmem::kRing);
  unsigned char *buf = sm + SwfSmem::kBuf;
  const uint32_t cb = (uint32_t)P.chunkb;
  const unsigned char *src = P.rec + (size_t)g * nch * cb;
  double *out = FWD ? a.y : a.z;
  const double *rin = FWD ? a.in_re : a.y;
  const bool r16 = P.rhs16 != 0;
  constexpr int HMAX = 4;

  // rows of the lane's positions p0 .. p0+T-1 of chunk c
  auto rowp = [&](int c) -> long long {
    const int p0 = c * kT - lag * j;
    return FWD ? G.lbase + p0 : (long long)n - kT - G.lbase - p0;  // lowest row (bwd)
  };
  auto full = [&](int c) {
    const int p0 = c * kT - lag * j;
    return p0 >= 0 && p0 + kT <= G.plim;
  };
  // chunk c's right-hand sides into staging slot c % kQ in POSITION order
  auto rhs_issue = [&](int c) {
    if (c < nch) {
      double *d0 = reinterpret_cast<double *>(sm + SwfSmem::kRhs) + ((c % kQR) * 32 + j) * kRow;
      const int p0 = c * kT - lag * j;
      if (FWD && r16 && full(c)) {
        const double *g0 = rin + rowp(c);
#pragma unroll
        for (int u = 0; u < kT / 2; ++u)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s_u32(d0 + 2 * u)),
                       "l"(g0 + 2 * u)
                       : "memory");
      } else {
#pragma unroll
        for (int t = 0; t < kT; ++t) {
          const int p = p0 + t;
          if (p >= 0 && p < G.plim) {
            const long long row = FWD ? G.lbase + p : (long long)n - 1 - G.lbase - p;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s_u32(d0 + t)),
                         "l"(rin + row)
                         : "memory");
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // previous line's value of position p (lane 0's view), polled until published
  auto prev_val = [&](int p) -> double {
    if (!G.has_prev || p < 0 || p >= Lc) return 0.0;
    const long long q = G.pbase + p;
    return g_poll(out + (FWD ? q : (long long)n - 1 - q));
  };
  // chunk c's previous-line positions (c*T + lag + t) into the ring; chunk
  // 0 also the pre-roll (lag - H .. lag - 1), polled until published
  auto ring_fill = [&](int c) {
    if (j < kT) {
      const int p = c * kT + lag + j;
      ring[(p + 31 * lag) & (kR - 1)] = prev_val(p);
    }
    if (c == 0 && j >= kT && j < kT + HMAX) {
      const int p = lag - (j - kT) - 1;
      ring[(p + 31 * lag) & (kR - 1)] = prev_val(p);
    }
  };
  // steady state: lanes 0..T-1 LOAD chunk c's positions one iteration
  // before they are stored (pv, pp) so the load latency overlaps the wait
  // for the compute warp; a value still holding the sentinel is polled, and
  // then the lane also waits for the furthest position of the next chunk to
  // build slack
  double pv = 0.0;
  int pp = -1;
  auto prev_load = [&](int c) {
    pp = -1;
    if (j < kT && c < nch && G.has_prev) {
      const int p = c * kT + lag + j;
      if (p < Lc) {
        const long long q = G.pbase + p;
        pp = p;
        pv = ld_relaxed(out + (FWD ? q : (long long)n - 1 - q));
      }
    }
  };
  auto prev_store = [&](int c) {
    if (j < kT) {
      const int p = c * kT + lag + j;
      double v = 0.0;
      if (pp == p) {
        v = pv;
        if (s_sent(v)) {
          int pa = p + kT;
          if (pa >= Lc) pa = Lc - 1;
          prev_val(pa);
          v = prev_val(p);
        }
      }
      ring[(p + 31 * lag) & (kR - 1)] = v;
    }
  };
  // publish chunk c's results (output staging slot c % kQ) to global memory
  auto publish = [&](int c) {
    const double *ob =
        reinterpret_cast<const double *>(sm + SwfSmem::kOut) + ((c % kQ) * 32 + j) * kRow;
    const int p0 = c * kT - lag * j;
    if (r16 && full(c)) {
      double *g0 = out + rowp(c);
#pragma unroll
      for (int u = 0; u < kT / 2; ++u) {
        const double2 v = reinterpret_cast<const double2 *>(ob)[u];
        // backward rows descend: memory pair u holds positions T-1-2u, T-2-2u
        const double lo = FWD ? v.x : ob[kT - 1 - 2 * u];
        const double hi = FWD ? v.y : ob[kT - 2 - 2 * u];
        asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(g0 + 2 * u), "d"(lo),
                     "d"(hi)
                     : "memory");
      }
    } else {
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int p = p0 + t;
        if (p >= 0 && p < G.plim)
          g_pub(out + (FWD ? G.lbase + p : (long long)n - 1 - G.lbase - p), ob[t]);
      }
    }
  };

  // prologue: records 0..kNB-1, right-hand sides 0..kQ-2, chunk 0 ready
  if (j == 0) {
    const int first = nch < kNB ? nch : kNB;
    for (int c = 0; c < first; ++c) {
      s_mbar_arrive_tx(rec_bar + c, cb);
      s_bulk(buf + (size_t)c * cb, src + (size_t)c * cb, cb, rec_bar + c);
    }
  }
#pragma unroll
  for (int c = 0; c < kQR - 1; ++c) rhs_issue(c);
  if (!dsm_in) {
    ring_fill(0);
    ring_fill(1);
    prev_load(2);
  }
  asm volatile("cp.async.wait_group %0;" ::"n"(kQR - 2) : "memory");  // rhs(0) landed
  s_mbar_wait(rec_bar, 0u);                                            // records(0)
  s_mbar_arrive_rel(ready + 0);
  constexpr int HD = 4;  // pre-roll bound of the throttle (window depth <= 4)
  for (int c = 0; c < nch; ++c) {
    // chunk c+1 ready: its right-hand sides, previous-line values, records
    if (c + 1 < nch) {
      if (c + 1 >= 2 && !dsm_in) {
        prev_store(c + 1);
        prev_load(c + 2);
      }
      asm volatile("cp.async.wait_group %0;" ::"n"(kQR - 3) : "memory");  // rhs(c+1)
      s_mbar_wait(rec_bar + (c + 1) % kNB, (uint32_t)(((c + 1) / kNB) & 1));
      // the output staging slot of chunk c+1 is the one chunk c+1-kQ sent
      // to the downstream CTA: that bulk copy (issued kQ-1 iterations ago;
      // the kQ-2 younger ones may still be in flight) must have read it
      if (dsm_out && j == 31)
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kQ - 2) : "memory");
      s_mbar_arrive_rel(ready + (c + 1) % kQ);
    }
    // chunk c computed
    s_mbar_wait(done + c % kQ, (uint32_t)((c / kQ) & 1));
    if (dsm_out && j == 31) {
      // the group's last line (output staging row 31) into the downstream
      // CTA's ring slots rslot(p0) .. +T-1 = c*T mod kR .. (contiguous), one
      // bulk copy completing the peer's mbarrier phase c, once the slots it
      // overwrites have been consumed there
      const int p0 = c * kT - lag * 31;
      const int pmax = p0 + kT - 1;
      for (;;) {
        const int pr = s_ld_acq_i(prog);
        const int consumed = pr < 0 ? lag - HD - 1 : pr * kT + kT - 1 + lag;
        if (pmax <= consumed + kR) break;
        __nanosleep(64);
      }
      const double *ob =
          reinterpret_cast<const double *>(sm + SwfSmem::kOut) + ((c % kQ) * 32 + 31) * kRow;
      const uint32_t bar = r_up + (uint32_t)((c % kNU) * 8);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      // relaxed: the data travels by the bulk copy, whose completion the
      // phase waits for (a release here costs a GPU-scope MEMBAR)
      asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar),
                   "r"((uint32_t)(kT * 8))
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              r_ring + (uint32_t)(((c * kT) & (kR - 1)) * 8)),
          "r"(s_u32(ob)), "r"((uint32_t)(kT * 8)), "r"(bar)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    publish(c);
    if (j == 0 && c + kNB < nch) {
      const int b = c % kNB;
      s_mbar_arrive_tx(rec_bar + b, cb);
      s_bulk(buf + (size_t)b * cb, src + (size_t)(c + kNB) * cb, cb, rec_bar + b);
    }
    rhs_issue(c + kQR - 1);  // slot (c - 1) % kQR: chunk c-1 is long done
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (dsm_out && j == 31) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int NK, int KEYS, bool FWD>
__global__ void __launch_bounds__(64, 1) swf_kernel(SweepArgs a, SPhase P) {
  __shared__ int s_tick;
  int *tick = a.tick;
  const bool clustered = P.cl > 1;
  {  // stopped solve: skip, but count this CTA out (ticket reset)
    int d = 0;
    if (threadIdx.x == 0 && a.done) d = *(volatile const int *)a.done;
    d = __syncthreads_or(d);
    if (d) {
      if (threadIdx.x == 0 && !clustered) {
        __threadfence();
        if (atomicAdd(&tick[1], 1) == (int)gridDim.x - 1) {
          atomicExch(&tick[0], 0);
          atomicExch(&tick[1], 0);
        }
      }
      return;
    }
  }
  if (!FWD && a.started && threadIdx.x == 0) atomicAdd(a.started, 1);
  extern __shared__ __align__(128) unsigned char sm[];
  const int w = threadIdx.x >> 5, j = threadIdx.x & 31;
  const int rank = clustered ? (int)cluster_rank() : 0;
  auto init = [&]() {
    if (threadIdx.x == 0) {
      // fresh barriers per group (no copy is pending here)
      uint64_t *rb = reinterpret_cast<uint64_t *>(sm + SwfSmem::kRec);
      for (int b = 0; b < kNB; ++b) s_mbar_init(rb + b, 1);
      uint64_t *ready = reinterpret_cast<uint64_t *>(sm + SwfSmem::kReady);
      uint64_t *done = reinterpret_cast<uint64_t *>(sm + SwfSmem::kDone);
      for (int b = 0; b < kQ; ++b) {
        s_mbar_init(ready + b, 32);
        s_mbar_init(done + b, 32);
      }
      uint64_t *up = reinterpret_cast<uint64_t *>(sm + SwfSmem::kUp);
      for (int b = 0; b < kNU; ++b) s_mbar_init(up + b, 1);
      *reinterpret_cast<int *>(sm + SwfSmem::kProg) = -1;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  };
  auto run = [&](int g) {
    if (swf_dbg_on && j == 0 && w == 0 && g < 4096) {
      unsigned wid, smid;
      asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      swf_dbg[(FWD ? 0 : 2 * 4096) + 2 * g] = gtimer();
      if (g < 64) swf_dbgw[FWD ? 0 : 1][g] = (int)(smid * 1000 + wid);
    }
    if (w == 0)
      swf_compute<NK, KEYS, FWD>(a, P, g, rank, sm);
    else
      swf_helper<FWD>(a, P, g, rank, sm);
    __syncthreads();
    if (swf_dbg_on && j == 0 && w == 0 && g < 4096)
      swf_dbg[(FWD ? 0 : 2 * 4096) + 2 * g + 1] = gtimer();
  };
  if (clustered) {
    // static mapping: group = CTA index (all clusters co-resident, checked
    // at plan build); peers' shared memory is live between the two syncs
    init();
    __syncthreads();
    cluster_sync();
    const int g = blockIdx.x;
    if (g < P.ngroups) run(g);
    cluster_sync();
    return;
  }
  for (;;) {
    if (threadIdx.x == 0) s_tick = atomicAdd(tick, 1);
    init();
    __syncthreads();
    const int g = s_tick;
    if (g >= P.ngroups) break;
    run(g);
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

// Row ranges of the host analysis on a few threads (the passes below read the
// pattern only; each thread reduces into its own slot).
static int par_threads(int n) {
  if (n < (1 << 16)) return 1;
  const unsigned hw = std::thread::hardware_concurrency();
  return (int)std::min<unsigned>(16u, hw ? hw : 1u);
}
template <class F>
static void par_rows(int n, int T, F f) {
  if (T <= 1) {
    f(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  const long long per = ((long long)n + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    const int lo = (int)std::min<long long>(n, per * t), hi = (int)std::min<long long>(n, per * (t + 1));
    th.emplace_back([=] { f(lo, hi, t); });
  }
  for (auto &x : th) x.join();
}

template <class Deps>
static bool analyse_phase(SPhase &ph, int n, bool fwd, Deps deps, long long &cost) {
  const int T = par_threads(n);
  long long D = 0;
  {
    std::vector<long long> dmax(T, 0);
    par_rows(n, T, [&](int lo, int hi, int t) {
      long long d = 0;
      for (int p = lo; p < hi; ++p)
        deps(p, [&](int pq, int) {
          if (p - pq > d) d = p - pq;
        });
      dmax[t] = d;
    });
    for (long long d : dmax) D = std::max(D, d);
  }
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
    {
      std::vector<long long> lags(T, 1);
      std::atomic<bool> okf{true};
      par_rows(n, T, [&](int lo, int hi, int t) {
        long long lg = 1;
        bool okt = true;
        for (int p = lo; p < hi && okt; ++p) {
          const long long l = p / Lc, pos = p % Lc;
          deps(p, [&](int pq, int) {
            const long long lq = pq / Lc, posq = pq % Lc;
            if (lq == l) return;
            if (lq != l - 1) {
              okt = false;
              return;
            }
            if (posq - pos + 1 > lg) lg = posq - pos + 1;
          });
          if ((p & 4095) == 0 && !okf.load(std::memory_order_relaxed)) break;
        }
        lags[t] = lg;
        if (!okt) okf.store(false, std::memory_order_relaxed);
      });
      ok = okf.load();
      for (long long lg : lags) lag = std::max(lag, lg);
    }
    if (!ok || lag > 3) continue;
    // the entries of every row must follow one pattern's key list
    int pat = -1;
    for (int k = 0; k < kNPat && pat < 0; ++k) {
      const Pattern &P = kPat[k];
      std::atomic<bool> goodf{true};
      par_rows(n, T, [&](int lo_, int hi_, int) {
      bool good = true;
      for (int p = lo_; p < hi_ && good; ++p) {
        if ((p & 4095) == 0 && !goodf.load(std::memory_order_relaxed)) break;
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
      if (!good) goodf.store(false, std::memory_order_relaxed);
      });
      if (goodf.load()) pat = k;
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
  par_rows(n, par_threads(n), [&](int lo_, int hi_, int) {  // rows own distinct slots
    for (int p = lo_; p < hi_; ++p) {
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
  });
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
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = smem;
  }
  if (P.cl > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)P.cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, fn, a, P);
  } else {
    fn<<<grid, 64, smem, st>>>(a, P);
  }
}

// thread-block clusters of `cl` CTAs that can be resident at once
template <int PAT, bool FWD>
static int max_clusters_pat(int cl, int grid, size_t smem) {
  constexpr Pattern pt = kPat[PAT];
  constexpr int KEYS =
      pt.keys[0] | (pt.keys[1] << 3) | (pt.keys[2] << 6) | (pt.keys[3] << 9);
  auto *fn = swf_kernel<pt.nk, KEYS, FWD>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int num = 0;
  const cudaError_t e = cudaOccupancyMaxActiveClusters(&num, fn, &cfg);
  if (getenv("MPK_VERBOSE"))
    fprintf(stderr, "[mpk] swf cluster query cl=%d grid=%d smem=%zu: %s, %d clusters\n", cl,
            grid, smem, cudaGetErrorString(e), num);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return num;
}
static int max_clusters(const SPhase &P, int cl, int grid, size_t smem) {
  const bool f = P.fwd != 0;
  switch (P.pat) {
    case 0: return f ? max_clusters_pat<0, true>(cl, grid, smem) : max_clusters_pat<0, false>(cl, grid, smem);
    case 1: return f ? max_clusters_pat<1, true>(cl, grid, smem) : max_clusters_pat<1, false>(cl, grid, smem);
    case 2: return f ? max_clusters_pat<2, true>(cl, grid, smem) : max_clusters_pat<2, false>(cl, grid, smem);
    default: return f ? max_clusters_pat<3, true>(cl, grid, smem) : max_clusters_pat<3, false>(cl, grid, smem);
  }
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
  // one group per CTA: a compute warp and a helper warp
  const int chunkmax = std::max(t.f.chunkb, t.b.chunkb);
  const int wbytes = (SwfSmem::kBuf + kNB * chunkmax + 127) / 128 * 128;
  t.f.wbytes = t.b.wbytes = wbytes;
  t.W = 1;
  t.smem = (size_t)wbytes;
  if (t.smem > 220 * 1024) {
    free_ssweep(t);
    return false;
  }
  // cluster hand-off between consecutive groups when every cluster of the
  // grid can be resident at once (static group -> CTA mapping)
  {
    const char *ec = getenv("MPK_SWF_CL");
    const int want = ec ? atoi(ec) : 16;
    for (SPhase *Q : {&t.f, &t.b}) {
      Q->cl = 1;
      for (int cl = want; cl >= 2; cl /= 2) {
        const int grid = (Q->ngroups + cl - 1) / cl * cl;
        if (grid > sm_count()) continue;
        if (max_clusters(*Q, cl, grid, t.smem) >= grid / cl) {
          Q->cl = cl;
          break;
        }
      }
    }
  }
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
    if (g > sm_count() * 16) g = sm_count() * 16;
    swf_gather_kernel<<<(unsigned)g, 256, 0, st>>>(lu, *P);
  }
}

void launch_ssweep(const SweepArgs &a, const SSweep &w, cudaStream_t st) {
  static const int only_g0 = getenv("MPK_SWF_ONLY_G0") ? atoi(getenv("MPK_SWF_ONLY_G0")) : 0;
  for (const SPhase *P : {&w.f, &w.b}) {
    ++tl_launches;
    SPhase Q = *P;
    if (only_g0) Q.ngroups = only_g0;  // diagnostics: timing of the first groups alone
    int grid = Q.ngroups;
    if (Q.cl > 1)
      grid = (Q.ngroups + Q.cl - 1) / Q.cl * Q.cl;
    else if (grid > sm_count())
      grid = sm_count();
    if (P == &w.b && tl_sweep_wait) cudaStreamWaitEvent(st, tl_sweep_wait, 0);
    launch_phase(a, Q, w.W, grid, w.smem, st);
    if (P == &w.f && tl_sweep_mid) cudaEventRecord(tl_sweep_mid, st);
  }
}

// CTAs of the backward phase (all resident at once in cluster mode)
int ssweep_bwd_ctas(const SSweep &w) {
  if (!w.on || w.b.cl <= 1) return 0;
  return (w.b.ngroups + w.b.cl - 1) / w.b.cl * w.b.cl;
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
