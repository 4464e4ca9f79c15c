// krylov.cu -- BiCG / CGS / BiCGSTAB / GPBiCG with binary64 ILU(0)-mixed
// preconditioning, entirely on the device.
//
// Reference: /root/reference/pkg/src/mpkrylov/solvers.py:183-412.  Every
// vector operation of the reference method bodies is executed with the
// same MC operation sequence per element (mc.cuh twins); consecutive
// element-wise operations are fused into one pass over HBM ("row
// kernels"), and each reduction is produced as block partials by the
// kernel that produces its operands, then folded by a one-block
// "finalize" kernel that also runs the scalar recurrence (alpha, beta,
// omega, zeta, eta; MC division on the device) and the stopping test.
// One iteration is captured once into a CUDA graph and replayed by a
// device-side WHILE conditional node: the host never synchronises inside
// the solve.
#include <cstdio>
#include <cstring>
#include <vector>

#include "krylov.cuh"
#include "rows.cuh"

namespace mpk {

// ---------------------------------------------------------------------
// scalar helpers run by thread 0 of a finalize kernel
// ---------------------------------------------------------------------
__device__ __forceinline__ void finish_state(State *S, long long it, int conv,
                                             int bd) {
  S->iterations = it;
  S->converged = conv;
  S->breakdown = bd;
  S->done = 1;
}

template <int K>
__device__ __forceinline__ void record(State *S, double *hist, const Sc &v) {
  if (S->hist_len < S->hist_cap) {
#pragma unroll
    for (int c = 0; c < K; ++c) hist[S->hist_len * K + c] = v.re[c];
  }
  S->hist_len++;
}

template <int K>
__device__ __noinline__ Sc sqrt_sc(const Sc &ss) {  // one copy per kernel (code size)
  Sc o = sc_zero();
  sqrt_mc<K>(R<K>(ss), R<K>(o));
  return o;
}

template <int K>
__device__ __forceinline__ bool lt(const Sc &a, const Sc &b) {
  return cmp<K>(R<K>(a), R<K>(b)) < 0;
}

// _Ctx.threshold solvers.py:146-149 and the r0 test; returns true if done
template <int K>
__device__ __forceinline__ bool setup_norm0(State *S, double *hist,
                                            const Sc &ss) {
  const Sc nrm0 = sqrt_sc<K>(ss);
  S->nrm0 = nrm0;
  S->nrm = nrm0;
  record<K>(S, hist, nrm0);
  Sc er = sc_zero(), ea = sc_zero(), t = sc_zero();
  er.re[0] = S->eps_rel;
  ea.re[0] = S->eps_abs;
  mul<K>(R<K>(er), R<K>(nrm0), R<K>(t));
  Sc thr = sc_zero();
  add<K>(R<K>(t), R<K>(ea), R<K>(thr));
  S->thr = thr;
  S->it = 1;
  if (lt<K>(nrm0, thr)) {
    S->have_nrm = 1;
    finish_state(S, 0, 1, kBdNone);
    return true;
  }
  if (S->max_iter < 1) {
    finish_state(S, S->max_iter < 0 ? 0 : S->max_iter, 0, kBdNone);
    return true;
  }
  return false;
}

// residual norm bookkeeping after norm2(r) / norm2(s); true if done
template <int K>
__device__ __forceinline__ bool check_nrm(State *S, double *hist,
                                          const Sc &ss) {
  const Sc nrm = sqrt_sc<K>(ss);
  S->nrm = nrm;
  S->have_nrm = 1;
  record<K>(S, hist, nrm);
  if (!is_finite<K>(R<K>(nrm))) {
    finish_state(S, S->it, 0, kBdNonfinite);
    return true;
  }
  if (lt<K>(nrm, S->thr)) {
    finish_state(S, S->it, 1, kBdNone);
    return true;
  }
  return false;
}

__device__ __forceinline__ void next_iter(State *S) {
  S->it++;
  if (S->it > S->max_iter) finish_state(S, S->max_iter, 0, kBdNone);
}

static __global__ void set_cond_kernel(cudaGraphConditionalHandle h, State *S,
                                       int count) {
  if (count) S->body_runs++;
  cudaGraphSetConditional(h, S->done ? 0u : 1u);
}

// report tail: final_recursive_relres = (nrm / nrm0).to_float()
template <int K>
__global__ void relres_kernel(State *S) {
  S->relres = NAN;
  if (S->have_nrm && !is_zero<K>(R<K>(S->nrm0))) {
    double q[K];
    div<K>(R<K>(S->nrm), R<K>(S->nrm0), q);
    S->relres = q[0];
  }
}

template <int K, bool CX>
__global__ void true_res_kernel_impl(State *S_, const double *pt_, int G_) {
  __shared__ double sm[kWarpsPerBlock * 16];
  Sc o[2];
  finalize_slots<K, false, false>(pt_, G_, sm, o);
  const Sc rr = o[0], bb = o[1];
  if (threadIdx.x == 0) {
    S_->true_relres = NAN;
    const Sc nb = sqrt_sc<K>(bb);
    if (!is_zero<K>(R<K>(nb))) {
      const Sc nr = sqrt_sc<K>(rr);
      double q[K];
      div<K>(R<K>(nr), R<K>(nb), q);
      S_->true_relres = q[0];
    }
  }
}


// BiCGSTAB: x = (x + alpha phat) + omega shat of the iteration recorded in
// S->xu_it (solvers.py:318), applied at the start of the NEXT body beside
// the forward phase of its first sweep, on the SMs the sweep leaves idle;
// also resets phat to the sentinel for that sweep's backward phase (this
// kernel is the last reader of the old phat).  Not skipped on the done flag:
// the pending update belongs to a completed iteration.  The last block out
// marks the update as applied.
template <int K, bool CX>
__global__ void __launch_bounds__(512, 2)
    xu_kernel(State *S, MV<K, CX> X, FV<CX> PH, FV<CX> SH, long long n) {
  const bool pend = S->xu_it != S->xu_done;
  const Sc al = S->alpha, om = S->omega;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (pend) {
      double xr[K], xi[K], fr[K], fi[K], tr[K], ti[K];
      X.load(i, xr, xi);
      PH.template load_mc<K>(i, fr, fi);
      e_axpy<K, CX>(al, fr, fi, xr, xi, tr, ti);
      SH.template load_mc<K>(i, fr, fi);
      e_axpy<K, CX>(om, fr, fi, tr, ti, xr, xi);
      X.store(i, xr, xi);
    }
    PH.set_sent(i);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&S->xu_cnt, 1) == (int)gridDim.x - 1) {
      if (pend) S->xu_done = S->xu_it;
      S->xu_cnt = 0;
    }
  }
}

// ---------------------------------------------------------------------
// solver object
// ---------------------------------------------------------------------
// A solver "plan": the per-(matrix, method, K, field) device workspace and
// the instantiated iteration graph.  Built on the first solve and cached on
// the matrix (DMat::plans), so repeated solves pay no allocation and no
// graph construction; every run-time parameter (eps, max_iter, scalars)
// lives in the device State the kernels read.
template <int K, bool CX>
struct Solver : PlanBase {
  using MVt = MV<K, CX>;
  using FVt = FV<CX>;
  DMat &A;
  DA da;
  SolveParams p;
  cudaStream_t st;
  int n;
  long long ld;
  int G;
  // row-block sharding (p.ex): rows [r0, r1) of blocks of nb, Gl blocks
  long long r0 = 0, r1 = 0, nb = 0;
  int gl = 0;
  // preconditioner 'none' (M = I): "applied" vectors are MC copies
  int nopre = 0;
  State *S = nullptr;
  double *part = nullptr;
  double *hist = nullptr;
  long long hist_cap = 0;
  const int *done = nullptr;
  int *err = nullptr;
  std::vector<void *> allocs;
  bool ok = true;
  char *errbuf;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  long long body_nodes = 0;
  bool cond_graph = true;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // side branch of the captured iteration (convergence tests overlapped
  // with the next sweep): its own stream, fork/join events, partials
  cudaStream_t st2 = nullptr, st3 = nullptr;
  cudaEvent_t evf = nullptr, evj = nullptr, evj3 = nullptr;
  double *part2 = nullptr;
  double *seqbuf = nullptr;  // twin-mode element terms [slot][i][2K]
  // MC-valued matrix (p.full_a): A x / A^H x of the next row kernel
  double *prebuf = nullptr, *prebuf_adj = nullptr;
  // sweep-pipelined SpMV (units.cu pspmv_kernel): the SpMV of a sweep's
  // output runs beside the sweep's backward phase on the SMs it leaves idle
  bool pipe_on = false;
  DA dap;  // da + the pipeline's result buffer and chunk flags
  cudaEvent_t evp_mid = nullptr, evp_join = nullptr;
  int *cur_started = nullptr;
  // deferred x update of BiCGSTAB (xu_kernel) beside the next forward phase
  bool xu_on = false;
  cudaEvent_t ev_xu0 = nullptr, ev_xu1 = nullptr;
  State *hp = nullptr;  // pinned host staging of the device State (x2)
  int *hpi = nullptr;

  void fork(bool third = false) {
    cudaEventRecord(evf, st);
    cudaStreamWaitEvent(st2, evf, 0);
    if (third) cudaStreamWaitEvent(st3, evf, 0);
  }
  void join(bool third = false) {
    cudaEventRecord(evj, st2);
    cudaStreamWaitEvent(st, evj, 0);
    if (third) {
      cudaEventRecord(evj3, st3);
      cudaStreamWaitEvent(st, evj3, 0);
    }
  }

  Solver(DMat &A_, const SolveParams &p_, cudaStream_t st_, char *eb)
      : A(A_), p(p_), st(st_), errbuf(eb) {
    nopre = p.precond_ilu == 1 ? 0 : 1;  // before any fv() allocation
    n = A.n;
    ld = plane_ld(n);
    // twin mode: element terms + ascending chains; finalize over 1 partial
    G = p.reduce_seq ? 1 : grid_for(n);
    if (p.ex) {  // row-block sharded (shard.cuh): W ranks x Gl blocks
      const int W = p.ex->world;
      gl = kMaxGrid / W;
      G = W * gl;
      nb = (n + W - 1) / W;
      r0 = (long long)p.ex->rank * nb;
      r1 = r0 + nb < n ? r0 + nb : n;
      if (r0 > n) r0 = n;
      if ((long long)W * nb > ld || p.reduce_seq || p.method != kBiCGSTAB ||
          !p.precond_ilu) {
        ok = false;
        snprintf(errbuf, 256,
                 "sharded solve: BiCGSTAB with tree reductions and W*ceil(n/W) <= "
                 "plane_ld(n) only");
      }
    }
    if (p.reduce_seq)
      seqbuf = (double *)dalloc(sizeof(double) * 8 * 2 * K * (size_t)(n > 0 ? n : 1));
    da = DA{A.n, A.rp, A.ci, A.val, A.at_rp, A.at_ci, A.at_val};
    if (p.full_a) {
      da.pre = prebuf = mc();
      if (p.method == kBiCG) da.pre_adj = prebuf_adj = mc();
    }
    dap = da;
    {
      const char *e = getenv("MPK_PIPE");
      pipe_on = A.pipe_order && !CX && p.precond_ilu == 1 && !p.ex && !p.full_a &&
                p.method != kBiCG && A.smat.ss.on && ssweep_bwd_ctas(A.smat.ss) > 0 &&
                !(e && e[0] == '0');
    }
    if (pipe_on) {
      dap.pre = prebuf = mc();
      dap.pflag = A.pipe_flag;
      cudaEventCreateWithFlags(&evp_mid, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&evp_join, cudaEventDisableTiming);
      const char *e = getenv("MPK_XU");
      xu_on = p.method == kBiCGSTAB && !(e && e[0] == '0');
      if (xu_on) {
        cudaEventCreateWithFlags(&ev_xu0, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_xu1, cudaEventDisableTiming);
        cudaFuncSetAttribute(xu_kernel<K, CX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kPipeSmem);
      }
    }
    S = (State *)dalloc(sizeof(State));
    part = (double *)dalloc(sizeof(double) * 6 * kMaxGrid * 8);
    hist_cap = p.hist_cap > 0 ? p.hist_cap : 1;
    hist = (double *)dalloc(sizeof(double) * K * hist_cap);
    fzero = fv();
    done = &S->done;
    err = A.err;
    switch (p.method) {
      case kBiCG: bicg_alloc(); break;
      case kCGS: cgs_alloc(); break;
      case kBiCGSTAB: bicgstab_alloc(); break;
      default: gpbicg_alloc(); break;
    }
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&st3, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&evf, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evj, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evj3, cudaEventDisableTiming);
    part2 = (double *)dalloc(sizeof(double) * 2 * kMaxGrid * 8);
    cudaMallocHost(&hp, sizeof(State) * 2);
    cudaMallocHost(&hpi, sizeof(int) * 4);
    *hpi = 0;
  }
  ~Solver() override {
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (evf) cudaEventDestroy(evf);
    if (evj) cudaEventDestroy(evj);
    if (st2) cudaStreamDestroy(st2);
    if (st3) cudaStreamDestroy(st3);
    if (evj3) cudaEventDestroy(evj3);
    if (evp_mid) cudaEventDestroy(evp_mid);
    if (evp_join) cudaEventDestroy(evp_join);
    if (ev_xu0) cudaEventDestroy(ev_xu0);
    if (ev_xu1) cudaEventDestroy(ev_xu1);
    if (hp) cudaFreeHost(hp);
    if (hpi) cudaFreeHost(hpi);
    for (void *q : allocs) cudaFree(q);
  }
  // MC-valued matrix: the SpMV the next row kernel consumes (sparse.py:
  // 414-451), x an F vector (xf) or a full MC vector
  void pre_spmv(const double *x_, bool xf, bool adjoint = false,
                bool after_loop = false) {
    if (!p.full_a) return;
    unit_spmv_full(A, K, adjoint, xf, x_, adjoint ? prebuf_adj : prebuf,
                   after_loop ? nullptr : done, st);
  }
  void zero_mc(double *q) {
    cudaMemsetAsync(q, 0, sizeof(double) * K * (CX ? 2 : 1) * ld, st);
  }
  void *dalloc(size_t bytes) {
    void *q = nullptr;
    if (cudaMalloc(&q, bytes < 16 ? 16 : bytes) != cudaSuccess) {
      ok = false;
      snprintf(errbuf, 256, "cudaMalloc(%zu) failed", bytes);
      return nullptr;
    }
    cudaMemsetAsync(q, 0, bytes < 16 ? 16 : bytes, st);
    allocs.push_back(q);
    return q;
  }
  double *mc() { return (double *)dalloc(sizeof(double) * K * (CX ? 2 : 1) * ld); }
  // F vector (head of an ILU(0)-mixed apply); none mode: a full MC vector
  double *fv() {
    return (double *)dalloc(sizeof(double) * (CX ? 2 : 1) * (nopre ? K : 1) * ld);
  }
  MVt mv(double *q) const { return MVt{q, ld}; }
  FVt fvv(double *q) const { return FVt{q, ld, nopre}; }

  // ILU(0)-mixed apply: z = promote(U^-1 L^-1 demote(in)).
  void sweep(const double *in_re, const double *in_im, double *y, double *z,
             bool adjoint, int which, bool after_loop = false) {
    if (nopre) {
      (void)in_im;
      if (p.precond_ilu == 2) {  // working-precision ILU(0) (ilu_mc.cu)
        mc_sweep(in_re, z, which, after_loop, st, adjoint);
        return;
      }
      // M = I (and M^H = I): the MC vector itself
      cudaMemcpyAsync(z, in_re, sizeof(double) * K * (CX ? 2 : 1) * ld,
                      cudaMemcpyDeviceToDevice, st);
      return;
    }
    if (p.ex) {
      // every rank sweeps the whole vector: gather the demoted input's rows
      // and reset all sentinels (the row kernels only touched own rows)
      p.ex->allgather_inplace(const_cast<double *>(in_re), (size_t)nb, st);
      if (in_im) p.ex->allgather_inplace(const_cast<double *>(in_im), (size_t)nb, st);
      launch_sweep_reset(y, z, n, CX, after_loop ? nullptr : done, st);
    }
    sweep_on(st, in_re, in_im, y, z, adjoint, which, after_loop);
  }
  // ILU(0)-mixed apply whose output z the next row kernel multiplies by A:
  // with a pipeline plan, A z is formed chunk by chunk beside the backward
  // phase (st3, released between the two phases of the sweep) into
  // `prebuf`; the row kernel then loads the flagged chunks (DA::pflag).
  void sweep_spmv(const double *in_re, const double *in_im, double *y, double *z,
                  cudaEvent_t before_bwd = nullptr) {
    if (!pipe_on) {
      sweep(in_re, in_im, y, z, false, 0);
      return;
    }
    launch_pipe_reset(A, st);
    tl_sweep_mid = evp_mid;
    tl_sweep_wait = before_bwd;
    cur_started = A.pipe_state + 1;
    sweep(in_re, in_im, y, z, false, 0);
    cur_started = nullptr;
    tl_sweep_mid = nullptr;
    tl_sweep_wait = nullptr;
    cudaStreamWaitEvent(st3, evp_mid, 0);
    launch_pspmv(A, K, z, prebuf, done, st3);
    cudaEventRecord(evp_join, st3);
    cudaStreamWaitEvent(st, evp_join, 0);
  }
  // deferred x update + phat sentinel reset (xu_kernel) on st3, released
  // when everything enqueued on st so far is done; ev_xu1 marks its end
  void launch_xu(bool side) {
    const MVt X = mv(x);
    const FVt PH = fvv(phat), SH = fvv(shat);
    ++tl_launches;
    if (side) {
      cudaEventRecord(ev_xu0, st);
      cudaStreamWaitEvent(st3, ev_xu0, 0);
      launch_pipe_delay(st3);  // the forward phase's clusters are placed first
      const int grid = (sm_count() - ssweep_bwd_ctas(A.smat.ss)) * 2;
      xu_kernel<K, CX><<<grid, 512, kPipeSmem, st3>>>(S, X, PH, SH, (long long)n);
      cudaEventRecord(ev_xu1, st3);
    } else {
      xu_kernel<K, CX><<<sm_count() * 2, 512, 0, st>>>(S, X, PH, SH, (long long)n);
    }
  }
  // z = U^-1 L^-1 in at working precision (real; planar K-component)
  void mc_sweep(const double *in, double *z, int which, bool after_loop,
                cudaStream_t s_, bool adjoint = false) {
    SweepMcArgs a{};
    a.adjoint = adjoint ? 1 : 0;
    a.cx = CX ? 1 : 0;
    a.ut_rp = A.ut_rp;
    a.ut_ci = A.ut_ci;
    a.ut_perm = A.ut_perm;
    a.lt_rp = A.lt_rp;
    a.lt_ci = A.lt_ci;
    a.lt_perm = A.lt_perm;
    a.ord_f = adjoint ? A.ord_fa : A.ord_f;
    a.ord_b = adjoint ? A.ord_ba : A.ord_b;
    a.n = n;
    a.ld = ld;
    a.rp = A.rp;
    a.ci = A.ci;
    a.dp = A.dp;
    a.lu = A.lu_mc;
    a.rcp = A.rcp_mc;
    a.in = in;
    a.y = which ? A.sw_mc2 : A.sw_mc;  // BiCG runs both applies concurrently
    a.z = z;
    a.tick = A.tick + 2 * which;
    a.err = A.err;
    a.done = after_loop ? nullptr : done;
    launch_sweep_mc(a, K, s_);
  }
  // all planes of an MC vector complete on every rank (sharded solve)
  void gather_mc(double *v) {
    if (!p.ex) return;
    for (int c = 0; c < K * (CX ? 2 : 1); ++c)
      p.ex->allgather_inplace(v + (size_t)c * ld, (size_t)nb, st);
  }
  void sweep_on(cudaStream_t s_, const double *in_re, const double *in_im,
                double *y, double *z, bool adjoint, int which,
                bool after_loop = false) {
    if (nopre) {
      if (p.precond_ilu == 2) {
        mc_sweep(in_re, z, which, after_loop, s_, adjoint);
        return;
      }
      cudaMemcpyAsync(z, in_re, sizeof(double) * K * (CX ? 2 : 1) * ld,
                      cudaMemcpyDeviceToDevice, s_);
      return;
    }
    SweepArgs a{};
    a.n = n;
    a.rp = A.rp;
    a.ci = A.ci;
    a.dp = A.dp;
    a.lu = A.lu;
    a.ut_rp = A.ut_rp;
    a.ut_ci = A.ut_ci;
    a.ut_val = A.ut_val;
    a.lt_rp = A.lt_rp;
    a.lt_ci = A.lt_ci;
    a.lt_val = A.lt_val;
    a.ord_f = adjoint ? A.ord_fa : A.ord_f;
    a.ord_b = adjoint ? A.ord_ba : A.ord_b;
    a.lev_f = adjoint ? A.lev_fa : A.lev_f;
    a.lev_b = adjoint ? A.lev_ba : A.lev_b;
    a.nlev_f = adjoint ? A.levels_fa : A.levels_f;
    a.nlev_b = adjoint ? A.levels_ba : A.levels_b;
    a.in_re = in_re;
    a.in_im = in_im;
    a.y = y;
    a.z = z;
    a.tick = A.tick + 2 * which;
    a.err = A.err;
    a.done = after_loop ? nullptr : done;
    a.started = cur_started;
    do_sweep(A, a, adjoint, s_);
  }
  const double *head_re(const double *v) const { return v; }
  const double *head_im(const double *v) const { return CX ? v + K * ld : nullptr; }

  // ---------------- BiCGSTAB (solvers.py:275-328) ----------------
  double *b, *x, *r, *rt0, *pp, *v, *s, *t, *phat, *shat, *fzero;
  double *u, *q, *w, *uhat, *whead;                 // CGS
  double *Bp, *Bt, *yv, *tpr, *zz, *yhat, *Mp, *Mt; // GPBiCG
  double *rt, *pt, *qv, *qt, *zf, *ztf;             // BiCG

  void alloc_common(const double *d_b) { b = const_cast<double *>(d_b); }

  // r = b - A*0 (the reference forms matvec(zeros), solvers.py:189 etc.),
  // plus partial norm2(r) [slot NH] and hdot(r, r) as rho [slot 0].
  void setup_residual(double *r_, double *r2_, bool with_rho) {
    const MVt B = mv(b), Rv = mv(r_), R2 = mv(r2_ ? r2_ : r_);
    const DA a = da;
    const double *fz = fzero;
    const long long L = ld;
    const int np_ = nopre;
    const bool two = r2_ != nullptr;
    pre_spmv(fzero, !nopre);
    rows<K, CX, 1, 1>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 1> &red) {
                        double axr[K], axi[K], br[K], bi[K], rr[K], ri[K];
                        spmv_fv<K, CX>(a, (int)i, fz, L, np_, axr, axi);
                        B.load(i, br, bi);
                        e_sub<K, CX>(br, bi, axr, axi, rr, ri);
                        Rv.store(i, rr, ri);
                        if (two) R2.store(i, rr, ri);
                        if (with_rho) acc_hdot<K, CX>(red.h[0], rr, ri, rr, ri);
                        acc_sumsq<K, CX>(red.nr[0], rr, ri);
                      });
    double *H = hist;
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          Sc o[2];
          finalize_slots<K, CX, false>(pt_, G_, sm, o);
          const Sc rho = o[0], ss = o[1];
          if (threadIdx.x == 0) {
            S_->rho = rho;
            setup_norm0<K>(S_, H, ss);
          }
        });
  }

  void bicgstab_alloc() {
    x = mc(); r = mc(); rt0 = mc(); pp = mc(); v = mc(); s = mc(); t = mc();
    phat = fv(); shat = fv();
  }
  void bicgstab_setup() {
    zero_mc(x);
    setup_residual(r, rt0, true);
  }

  void bicgstab_iter() {
    const MVt X = mv(x), Rr = mv(r), RT = mv(rt0), P = mv(pp), V = mv(v),
              Sv = mv(s), T = mv(t);
    const FVt PH = fvv(phat), SH = fvv(shat), Y = fvv(A.sw_y);
    State *Sd = S;
    double *H = hist;
    const DA a = pipe_on ? dap : da;
    const long long L = ld;
    const int np_ = nopre;
    const bool xu = xu_on;
    // F5+F1: [end of the previous iteration, deferred: rho_old = rho,
    // ||r|| record + tests, iteration count] then [this iteration: rho,
    // rho/omega zero tests, beta = (rho/rho_old)*(alpha/omega)].  The norm
    // test (warp 0) and the two quotients of beta (warps 1, 2) overlap; beta
    // is committed only if the solve continues.
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const bool pend = S_->pending != 0;
          Sc o[2];  // slot 1 (||r||) is only meaningful when pend
          finalize_slots<K, CX, false>(pt_, G_, sm, o);
          const Sc rho = o[0], ss = o[1];
          Sc *xs = reinterpret_cast<Sc *>(sm);
          if (threadIdx.x == 0) xs[2] = rho;
          __syncthreads();
          const long long itn = pend ? S_->it + 1 : S_->it;
          const Sc rold = pend ? S_->rho : S_->rho_old;
          const bool spec = itn > 1 && !s_is_zero<K, CX>(xs[2]) &&
                            !s_is_zero<K, CX>(S_->omega);
          if (spec && threadIdx.x == 32) xs[0] = s_div<K, CX>(xs[2], rold);
          if (spec && threadIdx.x == 64) xs[1] = s_div<K, CX>(S_->alpha, S_->omega);
          int *go = reinterpret_cast<int *>(xs + 3);
          if (threadIdx.x == 0) {
            *go = 0;
            bool stop = false;
            if (pend) {  // solvers.py:322-327
              S_->pending = 0;
              S_->rho_old = S_->rho;
              stop = check_nrm<K>(S_, H, ss);
              if (!stop) {
                next_iter(S_);
                stop = S_->done != 0;
              }
            }
            if (!stop) {  // solvers.py:291-300
              S_->rho = xs[2];
              if (s_is_zero<K, CX>(xs[2])) {
                finish_state(S_, S_->it, 0, kBdRhoZero);
              } else if (S_->it > 1 && s_is_zero<K, CX>(S_->omega)) {
                finish_state(S_, S_->it, 0, kBdOmegaZero);
              } else if (S_->it > 1) {
                *go = 1;
              }
            }
          }
          __syncthreads();
          if (*go && threadIdx.x == 0) S_->beta = s_mul<K, CX>(xs[0], xs[1]);
        });
    // K2: p = r (it 1) | p = r + beta*(p - omega*v); reset sweep buffers
    rows<K, CX, 0, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double rr[K], ri[K];
                        Rr.load(i, rr, ri);
                        if (Sd->it == 1) {
                          P.store(i, rr, ri);
                        } else {
                          double pr[K], pi[K], vr[K], vi[K], tr[K], ti[K];
                          P.load(i, pr, pi);
                          V.load(i, vr, vi);
                          const Sc mo = s_neg<K>(Sd->omega);
                          e_axpy<K, CX>(mo, vr, vi, pr, pi, tr, ti);
                          e_axpy<K, CX>(Sd->beta, tr, ti, rr, ri, pr, pi);
                          P.store(i, pr, pi);
                        }
                        Y.set_sent(i);
                        if (!xu) PH.set_sent(i);
                      });
    if (xu) launch_xu(true);
    sweep_spmv(head_re(pp), head_im(pp), A.sw_y, phat, xu ? ev_xu1 : nullptr);
    // K4: v = A phat ; sigma = hdot(rt0, v)
    const double *phc = phat;
    pre_spmv(phat, !nopre);
    rows<K, CX, 1, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 0> &red) {
                        double vr[K], vi[K], rr[K], ri[K];
                        spmv_fv<K, CX>(a, (int)i, phc, L, np_, vr, vi);
                        V.store(i, vr, vi);
                        RT.load(i, rr, ri);
                        acc_hdot<K, CX>(red.h[0], rr, ri, vr, vi);
                      });
    // F2: alpha
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc sg = finalize_slot<K, CX>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) {
            if (s_is_zero<K, CX>(sg)) {
              finish_state(S_, S_->it, 0, kBdSigmaZero);
              return;
            }
            S_->alpha = s_div<K, CX>(S_->rho, sg);
          }
        });
    // K5: s = r - alpha v ; norm2(s) (partials in part2 for the side branch)
    rows<K, CX, 0, 1>(n, done, part2, st,
                      [=] __device__(long long i, Red<K, CX, 0, 1> &red) {
                        double rr[K], ri[K], vr[K], vi[K], sr[K], si[K];
                        Rr.load(i, rr, ri);
                        V.load(i, vr, vi);
                        const Sc ma = s_neg<K>(Sd->alpha);
                        e_axpy<K, CX>(ma, vr, vi, rr, ri, sr, si);
                        Sv.store(i, sr, si);
                        acc_sumsq<K, CX>(red.nr[0], sr, si);
                        Y.set_sent(i);
                        SH.set_sent(i);
                      });
    // F3: half-step test on a side branch, overlapped with the sweep of s
    // and the SpMV that follow (they only touch shat / t / partials, which
    // are dead if F3 stops the solve; F4 and K8 run after the join and exit
    // on the done flag).  No sweep-error check here: that belongs to F4.
    fork();
    fin(S, nullptr, part2, G, st2,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc ss = finalize_slot<K, false>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) {
            if (check_nrm<K>(S_, H, ss) && S_->converged) S_->half_exit = 1;
          }
        });
    sweep_spmv(head_re(s), head_im(s), A.sw_y, shat);
    // K7: t = A shat ; tt = hdot(t,t), ts = hdot(t,s)
    const double *shc = shat;
    pre_spmv(shat, !nopre);
    rows<K, CX, 2, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 2, 0> &red) {
                        double tr[K], ti[K], sr[K], si[K];
                        spmv_fv<K, CX>(a, (int)i, shc, L, np_, tr, ti);
                        T.store(i, tr, ti);
                        Sv.load(i, sr, si);
                        acc_hdot<K, CX>(red.h[0], tr, ti, tr, ti);
                        acc_hdot<K, CX>(red.h[1], tr, ti, sr, si);
                      });
    join();
    // F4: omega
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          Sc o[2];
          finalize_slots<K, CX, CX>(pt_, G_, sm, o);
          const Sc tt = o[0], ts = o[1];
          if (threadIdx.x == 0) {
            if (s_is_zero<K, CX>(tt)) {
              finish_state(S_, S_->it, 0, kBdOmegaZero);
              return;
            }
            S_->omega = s_div<K, CX>(ts, tt);
            S_->pending = 1;  // K8 runs; its norm test happens in next F5+F1
          }
        });
    // K8: x = (x + alpha phat) + omega shat ; r = s - omega t ;
    //     norm2(r) [slot 1], next rho = hdot(rt0, r) [slot 0]
    rows<K, CX, 1, 1>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 1> &red) {
                        double tr[K], ti[K];
                        if (!xu) {
                          double xr[K], xi[K], fr[K], fi[K];
                          X.load(i, xr, xi);
                          PH.template load_mc<K>(i, fr, fi);
                          e_axpy<K, CX>(Sd->alpha, fr, fi, xr, xi, tr, ti);
                          SH.template load_mc<K>(i, fr, fi);
                          e_axpy<K, CX>(Sd->omega, fr, fi, tr, ti, xr, xi);
                          X.store(i, xr, xi);
                        } else if (i == 0) {
                          Sd->xu_it = Sd->it;  // applied by xu_kernel in the next body
                        }
                        double sr[K], si[K], rr[K], ri[K], qr[K], qi[K];
                        Sv.load(i, sr, si);
                        T.load(i, tr, ti);
                        const Sc mo = s_neg<K>(Sd->omega);
                        e_axpy<K, CX>(mo, tr, ti, sr, si, rr, ri);
                        Rr.store(i, rr, ri);
                        RT.load(i, qr, qi);
                        acc_hdot<K, CX>(red.h[0], qr, qi, rr, ri);
                        acc_sumsq<K, CX>(red.nr[0], rr, ri);
                      });
    // F5 (norm of r, rho_old = rho, iteration count) is deferred into the
    // next body's first finalize, where it runs concurrently with beta.
  }

  void bicgstab_finish(const State &hs) {
    // x update of the last completed iteration, if no later body applied it
    if (xu_on && hs.xu_it != hs.xu_done) launch_xu(false);
    if (hs.half_exit) {
      const MVt X = mv(x);
      const FVt PH = fvv(phat);
      State *Sd = S;
      rows<K, CX, 0, 0>(n, nullptr, part, st,
                        [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                          double xr[K], xi[K], fr[K], fi[K], tr[K], ti[K];
                          X.load(i, xr, xi);
                          PH.template load_mc<K>(i, fr, fi);
                          e_axpy<K, CX>(Sd->alpha, fr, fi, xr, xi, tr, ti);
                          X.store(i, tr, ti);
                        });
    }
  }

  // ---------------- CGS (solvers.py:229-272) ----------------
  void cgs_alloc() {
    x = mc(); r = mc(); rt0 = mc(); u = mc(); pp = mc(); q = mc(); v = mc();
    phat = fv(); uhat = fv();
    whead = (double *)dalloc(sizeof(double) * (nopre ? K * 2 : 2) * ld);
  }
  void cgs_setup() {
    zero_mc(x);
    setup_residual(r, rt0, true);
  }

  void cgs_iter() {
    const MVt X = mv(x), Rr = mv(r), RT = mv(rt0), U = mv(u), P = mv(pp),
              Q = mv(q), V = mv(v);
    const FVt PH = fvv(phat), UH = fvv(uhat), Y = fvv(A.sw_y);
    State *Sd = S;
    double *H = hist;
    const DA a = pipe_on ? dap : da;
    const long long L = ld;
    const int np_ = nopre;
    double *WH = whead;
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc rho = finalize_slot<K, CX>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) {
            S_->rho = rho;
            if (s_is_zero<K, CX>(rho)) {
              finish_state(S_, S_->it, 0, kBdRhoZero);
              return;
            }
            if (S_->it > 1) S_->beta = s_div<K, CX>(rho, S_->rho_old);
          }
        });
    // u = r + beta q ; p = u + beta (q + beta p)
    rows<K, CX, 0, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double rr[K], ri[K];
                        Rr.load(i, rr, ri);
                        if (Sd->it == 1) {
                          U.store(i, rr, ri);
                          P.store(i, rr, ri);
                        } else {
                          double qr[K], qi[K], ur[K], ui[K], pr[K], pi[K],
                              tr[K], ti[K];
                          Q.load(i, qr, qi);
                          P.load(i, pr, pi);
                          const Sc be = Sd->beta;
                          e_axpy<K, CX>(be, qr, qi, rr, ri, ur, ui);
                          e_axpy<K, CX>(be, pr, pi, qr, qi, tr, ti);
                          e_axpy<K, CX>(be, tr, ti, ur, ui, pr, pi);
                          U.store(i, ur, ui);
                          P.store(i, pr, pi);
                        }
                        Y.set_sent(i);
                        PH.set_sent(i);
                      });
    sweep_spmv(head_re(pp), head_im(pp), A.sw_y, phat);
    const double *phc = phat;
    pre_spmv(phat, !nopre);
    rows<K, CX, 1, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 0> &red) {
                        double vr[K], vi[K], rr[K], ri[K];
                        spmv_fv<K, CX>(a, (int)i, phc, L, np_, vr, vi);
                        V.store(i, vr, vi);
                        RT.load(i, rr, ri);
                        acc_hdot<K, CX>(red.h[0], rr, ri, vr, vi);
                      });
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc sg = finalize_slot<K, CX>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) {
            if (s_is_zero<K, CX>(sg)) {
              finish_state(S_, S_->it, 0, kBdSigmaZero);
              return;
            }
            S_->alpha = s_div<K, CX>(S_->rho, sg);
          }
        });
    // q = u - alpha v ; head(u + q) -> sweep input
    rows<K, CX, 0, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double ur[K], ui[K], vr[K], vi[K], qr[K], qi[K],
                            wr[K], wi[K];
                        U.load(i, ur, ui);
                        V.load(i, vr, vi);
                        const Sc ma = s_neg<K>(Sd->alpha);
                        e_axpy<K, CX>(ma, vr, vi, ur, ui, qr, qi);
                        Q.store(i, qr, qi);
                        e_add<K, CX>(ur, ui, qr, qi, wr, wi);
                        if (np_) {  // M = I: the whole u + q
#pragma unroll
                          for (int c = 0; c < K; ++c) {
                            WH[c * L + i] = wr[c];
                            if (CX) WH[(K + c) * L + i] = wi[c];
                          }
                        } else {
                          WH[i] = wr[0];
                          if (CX) WH[L + i] = wi[0];
                        }
                        Y.set_sent(i);
                        UH.set_sent(i);
                      });
    sweep_spmv(whead, CX ? whead + ld : nullptr, A.sw_y, uhat);
    // qhat = A uhat ; x += alpha uhat ; r -= alpha qhat ; norm2(r), rho
    const double *uhc = uhat;
    pre_spmv(uhat, !nopre);
    rows<K, CX, 1, 1>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 1> &red) {
                        double qr[K], qi[K], xr[K], xi[K], fr[K], fi[K],
                            tr[K], ti[K], rr[K], ri[K];
                        spmv_fv<K, CX>(a, (int)i, uhc, L, np_, qr, qi);
                        X.load(i, xr, xi);
                        UH.template load_mc<K>(i, fr, fi);
                        e_axpy<K, CX>(Sd->alpha, fr, fi, xr, xi, tr, ti);
                        X.store(i, tr, ti);
                        Rr.load(i, rr, ri);
                        const Sc ma = s_neg<K>(Sd->alpha);
                        e_axpy<K, CX>(ma, qr, qi, rr, ri, tr, ti);
                        Rr.store(i, tr, ti);
                        RT.load(i, qr, qi);
                        acc_hdot<K, CX>(red.h[0], qr, qi, tr, ti);
                        acc_sumsq<K, CX>(red.nr[0], tr, ti);
                      });
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc ss = finalize_slot<K, false>(pt_, 1, G_, sm);
          if (threadIdx.x == 0) {
            S_->rho_old = S_->rho;
            if (check_nrm<K>(S_, H, ss)) return;
            next_iter(S_);
          }
        });
  }

  // ---------------- GPBiCG (solvers.py:331-412) ----------------
  void gpbicg_alloc() {
    r = mc(); rt0 = mc(); u = mc(); zz = mc(); pp = mc(); Bp = mc();
    yv = mc(); t = mc(); Bt = mc(); w = mc(); tpr = mc(); yhat = mc();
    Mp = fv(); Mt = fv(); x = fv();
  }
  void gpbicg_setup() {
    // t_prev, w, u, z, yhat start at zero (solvers.py:341-352)
    zero_mc(u);
    zero_mc(zz);
    zero_mc(t);
    zero_mc(w);
    zero_mc(yhat);
    setup_residual(r, rt0, true);
  }

  void gpbicg_iter() {
    const MVt Rr = mv(r), RT = mv(rt0), U = mv(u), Z = mv(zz), P = mv(pp),
              BP = mv(Bp), YV = mv(yv), T = mv(t), BT = mv(Bt), W = mv(w),
              TPR = mv(tpr), YH = mv(yhat);
    const FVt MPv = fvv(Mp), MTv = fvv(Mt), Y = fvv(A.sw_y);
    State *Sd = S;
    double *H = hist;
    const DA a = pipe_on ? dap : da;
    const long long L = ld;
    const int np_ = nopre;
    // K2: w = Bt + beta Bp (end of previous iteration), p = r + beta (p - u)
    rows<K, CX, 0, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double rr[K], ri[K];
                        Rr.load(i, rr, ri);
                        if (Sd->it == 1) {
                          P.store(i, rr, ri);
                        } else {
                          double br[K], bi[K], tr[K], ti[K], pr[K], pi[K],
                              ur[K], ui[K];
                          BP.load(i, br, bi);
                          BT.load(i, tr, ti);
                          const Sc be = Sd->beta;
                          double wr[K], wi[K];
                          e_axpy<K, CX>(be, br, bi, tr, ti, wr, wi);
                          W.store(i, wr, wi);
                          P.load(i, pr, pi);
                          U.load(i, ur, ui);
                          e_sub<K, CX>(pr, pi, ur, ui, tr, ti);
                          e_axpy<K, CX>(be, tr, ti, rr, ri, pr, pi);
                          P.store(i, pr, pi);
                        }
                        Y.set_sent(i);
                        MPv.set_sent(i);
                      });
    sweep_spmv(head_re(pp), head_im(pp), A.sw_y, Mp);
    const double *mpc = Mp;
    pre_spmv(Mp, !nopre);
    rows<K, CX, 1, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 0> &red) {
                        double vr[K], vi[K], rr[K], ri[K];
                        spmv_fv<K, CX>(a, (int)i, mpc, L, np_, vr, vi);
                        BP.store(i, vr, vi);
                        RT.load(i, rr, ri);
                        acc_hdot<K, CX>(red.h[0], rr, ri, vr, vi);
                      });
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc sg = finalize_slot<K, CX>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) {
            if (s_is_zero<K, CX>(sg)) {
              finish_state(S_, S_->it, 0, kBdSigmaZero);
              return;
            }
            if (s_is_zero<K, CX>(S_->rho)) {
              finish_state(S_, S_->it, 0, kBdRhoZero);
              return;
            }
            S_->alpha = s_div<K, CX>(S_->rho, sg);
          }
        });
    // K5: tpr = t_prev - r ; y = tpr + alpha (Bp - w) ; t = r - alpha Bp
    rows<K, CX, 0, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double tr[K], ti[K], rr[K], ri[K], dr[K], di[K];
                        T.load(i, tr, ti);
                        Rr.load(i, rr, ri);
                        e_sub<K, CX>(tr, ti, rr, ri, dr, di);
                        TPR.store(i, dr, di);
                        double br[K], bi[K], wr[K], wi[K], gr[K], gi[K];
                        BP.load(i, br, bi);
                        W.load(i, wr, wi);
                        e_sub<K, CX>(br, bi, wr, wi, gr, gi);
                        double yr[K], yi[K];
                        e_axpy<K, CX>(Sd->alpha, gr, gi, dr, di, yr, yi);
                        YV.store(i, yr, yi);
                        const Sc ma = s_neg<K>(Sd->alpha);
                        e_axpy<K, CX>(ma, br, bi, rr, ri, tr, ti);
                        T.store(i, tr, ti);
                        Y.set_sent(i);
                        MTv.set_sent(i);
                      });
    sweep_spmv(head_re(t), head_im(t), A.sw_y, Mt);
    // K7: Bt = A Mt ; btbt, btt (+ yy, ybt, bty, yt when it > 1)
    const double *mtc = Mt;
    pre_spmv(Mt, !nopre);
    rows<K, CX, 6, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 6, 0> &red) {
                        double br[K], bi[K], tr[K], ti[K];
                        spmv_fv<K, CX>(a, (int)i, mtc, L, np_, br, bi);
                        BT.store(i, br, bi);
                        T.load(i, tr, ti);
                        acc_hdot<K, CX>(red.h[0], br, bi, br, bi);
                        acc_hdot<K, CX>(red.h[1], br, bi, tr, ti);
                        if (Sd->it > 1) {
                          double yr[K], yi[K];
                          YV.load(i, yr, yi);
                          acc_hdot<K, CX>(red.h[2], yr, yi, yr, yi);
                          acc_hdot<K, CX>(red.h[3], yr, yi, br, bi);
                          acc_hdot<K, CX>(red.h[4], br, bi, yr, yi);
                          acc_hdot<K, CX>(red.h[5], yr, yi, tr, ti);
                        }
                      });
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const bool more = S_->it > 1;  // uniform
          // all six slots side by side (slots 2-5 are stale when !more)
          Sc o[6];
          finalize_slots<K, CX, CX, CX, CX, CX, CX>(pt_, G_, sm, o);
          const Sc btbt = o[0], btt = o[1];
          Sc yy = sc_zero(), ybt = sc_zero(), bty = sc_zero(), yt = sc_zero();
          if (more) {
            yy = o[2];
            ybt = o[3];
            bty = o[4];
            yt = o[5];
          }
          if (!more) {
            if (threadIdx.x == 0) {
              if (s_is_zero<K, CX>(btbt)) {
                finish_state(S_, S_->it, 0, kBdLs);
                return;
              }
              S_->zeta = s_div<K, CX>(btt, btbt);
              S_->eta = sc_zero();
            }
            return;
          }
          // 2x2 least squares (solvers.py:384-392): the six products, the
          // three differences and the two quotients each run on their own
          // warp (independent MC operations -> latency of 1 mul + 1 sub +
          // 1 div instead of 6 + 3 + 2)
          Sc *xs = reinterpret_cast<Sc *>(sm);  // 6 slots (sm free here)
          if (threadIdx.x == 0) {
            xs[0] = yy;
            xs[1] = btbt;
            xs[2] = ybt;
            xs[3] = bty;
            xs[4] = yt;
            xs[5] = btt;
          }
          __syncthreads();
          Sc pr = sc_zero();
          const int w = threadIdx.x >> 5, lane0 = (threadIdx.x & 31) == 0;
          if (lane0 && w < 6) {
            const Sc a0 = xs[0], a1 = xs[1], a2 = xs[2], a3 = xs[3],
                     a4 = xs[4], a5 = xs[5];
            switch (w) {
              case 0: pr = s_mul<K, CX>(a0, a1); break;  // yy*btbt
              case 1: pr = s_mul<K, CX>(a2, a3); break;  // ybt*bty
              case 2: pr = s_mul<K, CX>(a1, a4); break;  // btbt*yt
              case 3: pr = s_mul<K, CX>(a2, a5); break;  // ybt*btt
              case 4: pr = s_mul<K, CX>(a0, a5); break;  // yy*btt
              default: pr = s_mul<K, CX>(a3, a4); break; // bty*yt
            }
          }
          __syncthreads();
          if (lane0 && w < 6) xs[w] = pr;
          __syncthreads();
          Sc df = sc_zero();
          if (lane0 && w < 3) df = s_sub<K, CX>(xs[2 * w], xs[2 * w + 1]);
          __syncthreads();
          if (lane0 && w < 3) xs[w] = df;  // delta, eta_num, zeta_num
          __syncthreads();
          const bool sing = s_is_zero<K, CX>(xs[0]);
          if (sing) {
            if (threadIdx.x == 0) finish_state(S_, S_->it, 0, kBdLs);
            return;
          }
          if (threadIdx.x == 0) S_->eta = s_div<K, CX>(xs[1], xs[0]);
          if (threadIdx.x == 32) S_->zeta = s_div<K, CX>(xs[2], xs[0]);
        });
    // K8: u, z, yhat, r updates ; norm2(r) [slot 1], rho_new [slot 0]
    rows<K, CX, 1, 1>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 1> &red) {
                        const Sc ze = Sd->zeta, et = Sd->eta, al = Sd->alpha;
                        double br[K], bi[K], ur[K], ui[K];
                        BP.load(i, br, bi);
                        if (Sd->it > 1) {
                          double dr[K], di[K], tr[K], ti[K], sr[K], si[K];
                          TPR.load(i, dr, di);
                          U.load(i, ur, ui);
                          e_axpy<K, CX>(Sd->beta, ur, ui, dr, di, tr, ti);
                          e_scale<K, CX>(et, tr, ti, sr, si);
                          e_axpy<K, CX>(ze, br, bi, sr, si, ur, ui);
                        } else {
                          e_scale<K, CX>(ze, br, bi, ur, ui);
                        }
                        U.store(i, ur, ui);
                        double zr[K], zi[K], z1r[K], z1i[K], rr[K], ri[K];
                        Z.load(i, zr, zi);
                        Rr.load(i, rr, ri);
                        e_scale<K, CX>(et, zr, zi, z1r, z1i);
                        e_axpy<K, CX>(ze, rr, ri, z1r, z1i, zr, zi);
                        const Sc ma = s_neg<K>(al);
                        e_axpy<K, CX>(ma, ur, ui, zr, zi, z1r, z1i);
                        Z.store(i, z1r, z1i);
                        double pr[K], pi[K], hr[K], hi[K], gr[K], gi[K];
                        P.load(i, pr, pi);
                        e_axpy<K, CX>(al, pr, pi, z1r, z1i, gr, gi);
                        YH.load(i, hr, hi);
                        e_add<K, CX>(hr, hi, gr, gi, pr, pi);
                        YH.store(i, pr, pi);
                        double tr[K], ti[K], bt_r[K], bt_i[K], yr[K], yi[K];
                        T.load(i, tr, ti);
                        BT.load(i, bt_r, bt_i);
                        YV.load(i, yr, yi);
                        e_axpy<K, CX>(s_neg<K>(ze), bt_r, bt_i, tr, ti, gr, gi);
                        e_axpy<K, CX>(s_neg<K>(et), yr, yi, gr, gi, rr, ri);
                        Rr.store(i, rr, ri);
                        double qr[K], qi[K];
                        RT.load(i, qr, qi);
                        acc_hdot<K, CX>(red.h[0], qr, qi, rr, ri);
                        acc_sumsq<K, CX>(red.nr[0], rr, ri);
                      });
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          Sc o[2];
          finalize_slots<K, CX, false>(pt_, G_, sm, o);
          const Sc rn = o[0], ss = o[1];
          // norm test (warp 0) and the two quotients of beta (warps 1, 2)
          // run concurrently; beta is only committed if the test continues
          Sc *xs = reinterpret_cast<Sc *>(sm);
          if (threadIdx.x == 0) xs[2] = rn;
          __syncthreads();
          const bool zz = s_is_zero<K, CX>(S_->zeta), zr = s_is_zero<K, CX>(S_->rho);
          if (threadIdx.x == 32 && !zz && !zr) xs[0] = s_div<K, CX>(S_->alpha, S_->zeta);
          if (threadIdx.x == 64 && !zz && !zr) xs[1] = s_div<K, CX>(xs[2], S_->rho);
          int *stop = reinterpret_cast<int *>(xs + 3);
          if (threadIdx.x == 0) {
            *stop = 1;
            if (check_nrm<K>(S_, H, ss)) {
            } else if (zz) {
              finish_state(S_, S_->it, 0, kBdZetaZero);
            } else if (zr) {
              finish_state(S_, S_->it, 0, kBdRhoZero);
            } else {
              *stop = 0;
            }
          }
          __syncthreads();
          if (threadIdx.x == 0 && !*stop) {
            S_->beta = s_mul<K, CX>(xs[0], xs[1]);
            S_->rho = rn;
            next_iter(S_);
          }
        });
  }

  // ---------------- BiCG (solvers.py:183-226) ----------------
  void bicg_alloc() {
    x = mc(); r = mc(); rt = mc(); pp = mc(); pt = mc(); qv = mc(); qt = mc();
    zf = fv(); ztf = fv();
  }
  void bicg_setup() {
    zero_mc(x);
    setup_residual(r, rt, false);
    const FVt Z = fvv(zf), ZT = fvv(ztf), Y = fvv(A.sw_y), Y2 = fvv(A.sw_y2);
    rows<K, CX, 0, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        Y.set_sent(i);
                        Z.set_sent(i);
                        Y2.set_sent(i);
                        ZT.set_sent(i);
                      });
    sweep(head_re(r), head_im(r), A.sw_y, zf, false, 0);
    sweep(head_re(rt), head_im(rt), A.sw_y2, ztf, true, 1);
    const MVt P = mv(pp), PT = mv(pt), Rr = mv(r);
    rows<K, CX, 1, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 1, 0> &red) {
                        double zr[K], zi[K], wr[K], wi[K], rr[K], ri[K];
                        Z.template load_mc<K>(i, zr, zi);
                        ZT.template load_mc<K>(i, wr, wi);
                        P.store(i, zr, zi);
                        PT.store(i, wr, wi);
                        Rr.load(i, rr, ri);
                        acc_hdot<K, CX>(red.h[0], wr, wi, rr, ri);
                      });
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc rho = finalize_slot<K, CX>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) S_->rho = rho;
        });
  }

  void bicg_iter() {
    const MVt X = mv(x), Rr = mv(r), RTv = mv(rt), P = mv(pp), PT = mv(pt),
              Q = mv(qv), QT = mv(qt);
    const FVt Z = fvv(zf), ZT = fvv(ztf), Y = fvv(A.sw_y), Y2 = fvv(A.sw_y2);
    State *Sd = S;
    double *H = hist;
    const DA a = da;
    const long long L = ld;
    const int np_ = nopre;
    const double *pc = pp, *ptc = pt;
    // q = A p ; sigma = hdot(pt, q) (role 0) || qt = A^H pt (role 1): the
    // two SpMV chains run on separate threads
    const long long nn = n;
    pre_spmv(pp, false);
    pre_spmv(pt, false, true);
    rows<K, CX, 1, 0>(
        n, done, part, st,
        [=] __device__(long long i, Red<K, CX, 1, 0> &red) {
          if (i < nn) {
            double qr[K], qi[K], pr[K], pi[K];
            spmv_mc<K, CX, false>(a, (int)i, pc, L, qr, qi);
            Q.store(i, qr, qi);
            PT.load(i, pr, pi);
            acc_hdot<K, CX>(red.h[0], pr, pi, qr, qi);
          } else {
            const long long j = i - nn;
            double wr[K], wi[K];
            spmv_mc<K, CX, true>(a, (int)j, ptc, L, wr, wi);
            QT.store(j, wr, wi);
          }
        },
        2);
    fin(S, err, part, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc sg = finalize_slot<K, CX>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) {
            if (s_is_zero<K, CX>(sg)) {
              finish_state(S_, S_->it, 0, kBdSigmaZero);
              return;
            }
            if (s_is_zero<K, CX>(S_->rho)) {
              finish_state(S_, S_->it, 0, kBdRhoZero);
              return;
            }
            S_->alpha = s_div<K, CX>(S_->rho, sg);
          }
        });
    rows<K, CX, 0, 1>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 1> &red) {
                        const Sc al = Sd->alpha;
                        double xr[K], xi[K], pr[K], pi[K], tr[K], ti[K];
                        X.load(i, xr, xi);
                        P.load(i, pr, pi);
                        e_axpy<K, CX>(al, pr, pi, xr, xi, tr, ti);
                        X.store(i, tr, ti);
                        double rr[K], ri[K], qr[K], qi[K];
                        Rr.load(i, rr, ri);
                        Q.load(i, qr, qi);
                        e_axpy<K, CX>(s_neg<K>(al), qr, qi, rr, ri, tr, ti);
                        Rr.store(i, tr, ti);
                        acc_sumsq<K, CX>(red.nr[0], tr, ti);
                        RTv.load(i, rr, ri);
                        QT.load(i, qr, qi);
                        e_axpy<K, CX>(s_neg<K>(s_conj<K, CX>(al)), qr, qi, rr,
                                      ri, xr, xi);
                        RTv.store(i, xr, xi);
                        Y.set_sent(i);
                        Z.set_sent(i);
                        Y2.set_sent(i);
                        ZT.set_sent(i);
                      });
    // the two preconditioner applies are independent: the adjoint one (and
    // hdot(zt, r), partials in part2) runs on the side branch, overlapped
    // with the norm test and the forward apply.  Work done after a stop is
    // dead (the next finalize exits on the done flag).
    fork(true);
    fin(S, err, part, G, st3,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc ss = finalize_slot<K, false>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) check_nrm<K>(S_, H, ss);
        });
    sweep(head_re(r), head_im(r), A.sw_y, zf, false, 0);
    sweep_on(st2, head_re(rt), head_im(rt), A.sw_y2, ztf, true, 1);
    rows<K, CX, 1, 0>(n, done, part2, st2,
                      [=] __device__(long long i, Red<K, CX, 1, 0> &red) {
                        double wr[K], wi[K], rr[K], ri[K];
                        ZT.template load_mc<K>(i, wr, wi);
                        Rr.load(i, rr, ri);
                        acc_hdot<K, CX>(red.h[0], wr, wi, rr, ri);
                      });
    join(true);
    fin(S, err, part2, G, st,
        [=] __device__(State * S_, const double *pt_, int G_, double *sm) {
          const Sc rn = finalize_slot<K, CX>(pt_, 0, G_, sm);
          if (threadIdx.x == 0) {
            S_->beta = s_div<K, CX>(rn, S_->rho);
            S_->rho = rn;
            next_iter(S_);
          }
        });
    // p = z + beta p ; pt = zt + conj(beta) pt (runs unless stopped above)
    rows<K, CX, 0, 0>(n, done, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        const Sc be = Sd->beta;
                        double pr[K], pi[K], zr[K], zi[K], tr[K], ti[K];
                        P.load(i, pr, pi);
                        Z.template load_mc<K>(i, zr, zi);
                        e_axpy<K, CX>(be, pr, pi, zr, zi, tr, ti);
                        P.store(i, tr, ti);
                        PT.load(i, pr, pi);
                        ZT.template load_mc<K>(i, zr, zi);
                        e_axpy<K, CX>(s_conj<K, CX>(be), pr, pi, zr, zi, tr, ti);
                        PT.store(i, tr, ti);
                      });
  }

  // ---------------- driver ----------------
  void setup() {
    switch (p.method) {
      case kBiCG: bicg_setup(); break;
      case kCGS: cgs_setup(); break;
      case kBiCGSTAB: bicgstab_setup(); break;
      default: gpbicg_setup(); break;
    }
  }
  void iter() {
    switch (p.method) {
      case kBiCG: bicg_iter(); break;
      case kCGS: cgs_iter(); break;
      case kBiCGSTAB: bicgstab_iter(); break;
      default: gpbicg_iter(); break;
    }
  }

  // x_out (planar MC) after the loop; returns false on error
  void finish(const State &hs, double *d_x) {
    const long long planes = K * (CX ? 2 : 1);
    if (p.method == kBiCGSTAB) bicgstab_finish(hs);
    if (p.method == kGPBiCG) {
      // x = M^-1 yhat (solvers.py:357-359), or yhat itself on the r0 exit
      if (hs.iterations == 0 && hs.converged) {
        cudaMemcpyAsync(d_x, yhat, sizeof(double) * planes * ld,
                        cudaMemcpyDeviceToDevice, st);
        return;
      }
      launch_sweep_reset(A.sw_y, x, n, CX, nullptr, st);
      sweep(head_re(yhat), head_im(yhat), A.sw_y, x, false, 0, true);
      promote(x, d_x);
      return;
    }
    gather_mc(x);
    cudaMemcpyAsync(d_x, x, sizeof(double) * planes * ld,
                    cudaMemcpyDeviceToDevice, st);
  }

  void promote(const double *f, double *d_x) {
    const FVt F = fvv(const_cast<double *>(f));
    const MVt X = mv(d_x);
    rows<K, CX, 0, 0>(n, nullptr, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 0> &) {
                        double xr[K], xi[K];
                        F.template load_mc<K>(i, xr, xi);
                        X.store(i, xr, xi);
                      });
  }

  // true residual ||b - A x|| / ||b|| (solvers.py:446-450); x planar MC
  void true_residual(const double *d_x) {
    const MVt B = mv(b);
    const DA a = da;
    const long long L = ld;
    const int np_ = nopre;
    pre_spmv(d_x, false, false, true);
    rows<K, CX, 0, 2>(n, nullptr, part, st,
                      [=] __device__(long long i, Red<K, CX, 0, 2> &red) {
                        double axr[K], axi[K], br[K], bi[K], rr[K], ri[K];
                        spmv_mc<K, CX, false>(a, (int)i, d_x, L, axr, axi);
                        B.load(i, br, bi);
                        e_sub<K, CX>(br, bi, axr, axi, rr, ri);
                        acc_sumsq<K, CX>(red.nr[0], rr, ri);
                        acc_sumsq<K, CX>(red.nr[1], br, bi);
                      });
    true_res_kernel_impl<K, CX><<<1, kBlock, 0, st>>>(S, part, G);
  }
};

// ---------------------------------------------------------------------
// graph execution
// ---------------------------------------------------------------------
#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      snprintf(errbuf, 256, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
               __FILE__, __LINE__);                                        \
      return 4;                                                            \
    }                                                                      \
  } while (0)

template <int K, bool CX>
int run_typed(DMat &A, const SolveParams &p, const double *d_b, double *d_x,
              double *d_hist, SolveOut *out, cudaStream_t st, char *errbuf) {
  if (p.method == kBiCG) ensure_adjoint(A, st);
  const char *nocond = getenv("MPK_NO_COND_GRAPH");
  const bool use_cond = !nocond || nocond[0] == '0';
  // plan cache: one workspace + graph per (method, K, field) on this matrix
  const int key = (p.precond_ilu == 1 ? 0 : (p.precond_ilu + 1) * 10000000) +
                  (p.ex ? 100000 * p.ex->world : 0) +
                  p.reduce_seq * 1000 + p.full_a * 5000 +
                  p.method * 100 + K * 10 + (CX ? 1 : 0);
  Solver<K, CX> *sv = nullptr;
  auto it = A.plans.find(key);
  if (it != A.plans.end()) {
    sv = static_cast<Solver<K, CX> *>(it->second.get());
    if (sv->hist_cap < p.hist_cap || sv->cond_graph != use_cond) {
      A.plans.erase(it);
      sv = nullptr;
    }
  }
  if (!sv) {
    SolveParams pp = p;
    pp.hist_cap = p.hist_cap > 0 ? p.hist_cap : 1;
    auto *fresh = new Solver<K, CX>(A, pp, st, errbuf);
    A.plans[key].reset(fresh);
    sv = fresh;
    if (!sv->ok) {
      A.plans.erase(key);
      return 4;
    }
    sv->cond_graph = use_cond;
  }
  sv->p = p;
  sv->errbuf = errbuf;
  struct SeqScope {  // every row kernel of this solve (eager or captured)
    explicit SeqScope(double *s) { tl_seq = s; }
    ~SeqScope() { tl_seq = nullptr; }
  } seq_scope(sv->seqbuf);
  struct ShardScope {  // row kernels of a sharded solve cover the own rows
    explicit ShardScope(const Solver<K, CX> *v) {
      if (v->p.ex) {
        tl_shard.ex = v->p.ex;
        tl_shard.r0 = v->r0;
        tl_shard.r1 = v->r1;
        tl_shard.gl = v->gl;
        tl_shard.boff = v->p.ex->rank * v->gl;
      }
    }
    ~ShardScope() { tl_shard = ShardCtx{}; }
  } shard_scope(sv);
  const bool sharded = p.ex != nullptr;
  const long long launches0 = tl_launches;
  State hs{};
  hs.max_iter = p.max_iter;
  hs.hist_cap = p.hist_cap;
  hs.eps_rel = p.eps_rel;
  hs.eps_abs = p.eps_abs;
  hs.relres = NAN;
  hs.true_relres = NAN;
  *sv->hp = hs;  // pinned staging: pageable copies serialise concurrent solves
  CK(cudaMemcpyAsync(sv->S, sv->hp, sizeof(State), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(A.err, 0, sizeof(int), st));
  sv->alloc_common(d_b);
  cudaEventRecord(sv->ev0, st);
  sv->setup();
  CK(cudaGetLastError());

  if (!sv->ge && !sharded) {
    if (use_cond) {
      // one iteration -> body of a device-side WHILE conditional node
      CK(cudaGraphCreate(&sv->g, 0));
      cudaGraphConditionalHandle h;
      CK(cudaGraphConditionalHandleCreate(&h, sv->g, 0, 0));
      cudaKernelNodeParams kp{};
      State *Sd = sv->S;
      int no_count = 0;
      void *args[] = {&h, &Sd, &no_count};
      kp.func = (void *)set_cond_kernel;
      kp.gridDim = dim3(1);
      kp.blockDim = dim3(1);
      kp.kernelParams = args;
      cudaGraphNode_t n1, n2;
      CK(cudaGraphAddKernelNode(&n1, sv->g, nullptr, 0, &kp));
      cudaGraphNodeParams cp{};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      CK(cudaGraphAddNode(&n2, sv->g, &n1, 1, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal));
      const long long c0 = tl_launches;
      sv->iter();
      set_cond_kernel<<<1, 1, 0, st>>>(h, sv->S, 1);
      sv->body_nodes = tl_launches - c0 + 1;
      tl_launches = c0;
      CK(cudaStreamEndCapture(st, &body));
    } else {
      // fallback: a plain one-iteration graph replayed in polled chunks
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      const long long c0 = tl_launches;
      sv->iter();
      sv->body_nodes = tl_launches - c0;
      tl_launches = c0;
      CK(cudaStreamEndCapture(st, &sv->g));
    }
    CK(cudaGraphInstantiate(&sv->ge, sv->g, 0));
  }
  tl_phase[2] = host_ms();  // setup enqueued, graph ready
  if (sharded) {
    // eager iterations (the exchanges are host-enqueued collectives); the
    // ranks compute identical stop decisions, so they leave together
    // (the device decides the stop, incl. max_iter, one body after the last
    // iteration: BiCGSTAB's norm test is deferred into the next body)
    long long launched = 0;
    const long long cap = p.max_iter + 8;
    int chunk = 4;
    State probe{};
    while (launched < cap) {
      for (int c = 0; c < chunk && launched < cap; ++c, ++launched) sv->iter();
      CK(cudaMemcpyAsync(sv->hp + 1, sv->S, sizeof(State), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      probe = sv->hp[1];
      if (probe.done) break;
      if (chunk < 16) chunk *= 2;
    }
  } else if (use_cond) {
    CK(cudaGraphLaunch(sv->ge, st));
    tl_launches += 1;  // the init node; body nodes counted per run below
  } else {
    long long launched = 0;
    int chunk = 4;
    State probe{};
    while (launched < p.max_iter) {
      for (int c = 0; c < chunk && launched < p.max_iter; ++c, ++launched) {
        CK(cudaGraphLaunch(sv->ge, st));
        tl_launches += sv->body_nodes;
      }
      CK(cudaMemcpyAsync(sv->hp + 1, sv->S, sizeof(State), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      probe = sv->hp[1];
      if (probe.done) break;
      if (chunk < 64) chunk *= 2;
    }
  }
  cudaEventRecord(sv->ev1, st);
  CK(cudaMemcpyAsync(sv->hp, sv->S, sizeof(State), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  hs = *sv->hp;
  tl_phase[3] = host_ms();  // loop done (synchronised)
  if (use_cond && !sharded) tl_launches += sv->body_nodes * hs.body_runs;
  const bool ran_out = !hs.done;
  if (ran_out) {
    // loop ran out without a device-side stop (max_iter reached; only the
    // plain-graph replay mode, MPK_NO_COND_GRAPH, can end this way)
    hs.iterations = p.max_iter;
    hs.converged = 0;
    hs.breakdown = kBdNone;
  }
  float loop_ms = 0;
  cudaEventElapsedTime(&loop_ms, sv->ev0, sv->ev1);
  out->loop_ms = loop_ms;
  out->hist_len = hs.hist_len;
  const long long hn = hs.hist_len < p.hist_cap ? hs.hist_len : p.hist_cap;
  if (d_hist && hn > 0)
    CK(cudaMemcpyAsync(d_hist, sv->hist, sizeof(double) * K * hn,
                       cudaMemcpyDeviceToDevice, st));
  auto sweep_fail = [&]() {
    out->iterations = 0;
    out->converged = 0;
    out->breakdown = kBdNumericSweep;
    out->half_exit = 0;
    out->relres = NAN;
    out->true_relres = NAN;
    out->launches = tl_launches - launches0;
    return 0;
  };
  if (hs.breakdown == kBdNumericSweep) return sweep_fail();
  sv->finish(hs, d_x);
  int e_after = 0;
  const bool chk_after = p.method == kGPBiCG && !(hs.iterations == 0 && hs.converged);
  if (chk_after)
    CK(cudaMemcpyAsync(sv->hpi, A.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  relres_kernel<K><<<1, 1, 0, st>>>(sv->S);
  tl_launches += 2;  // relres + true-residual finalize
  sv->true_residual(d_x);
  CK(cudaMemcpyAsync(sv->hp, sv->S, sizeof(State), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  hs = *sv->hp;
  if (ran_out) {  // the device State never recorded a stop
    hs.iterations = p.max_iter;
    hs.converged = 0;
    hs.breakdown = kBdNone;
  }
  tl_phase[4] = host_ms();  // finish + true residual done
  if (chk_after) e_after = *sv->hpi;
  CK(cudaGetLastError());
  if (e_after) return sweep_fail();
  out->iterations = hs.iterations;
  out->converged = hs.converged;
  out->breakdown = hs.breakdown;
  out->half_exit = hs.half_exit;
  out->relres = hs.relres;
  out->true_relres = hs.true_relres;
  out->launches = tl_launches - launches0;
  return 0;
}

}  // namespace mpk
