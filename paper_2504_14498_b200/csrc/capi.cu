// capi.cu -- C ABI (include/mpk_b200.h) over the device hot path.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mpk_b200.h"
#include "krylov.cuh"

namespace mpk {
int host_mc(int op, int k, const double *a_re, const double *a_im,
            const double *b_re, const double *b_im, double *o_re,
            double *o_im);
void launch_to_planar(long long n, int k, const double *re, const double *im,
                      double *dev, cudaStream_t st);
void launch_from_planar(long long n, int k, const double *dev, double *re,
                        double *im, cudaStream_t st);
}  // namespace mpk

using namespace mpk;

struct mpk_ctx {
  int device;
  cudaStream_t stream;
  int reduce_seq = 0;  // MPK_OPT_REDUCTION
  int precond = 1;     // MPK_OPT_PRECOND: 1 ILU(0)-mixed, 0 none (M = I)
};

// Per-k device I/O buffers of mpk_solve, kept across calls (no
// cudaMalloc/cudaFree -- which synchronise the device -- on the call path).
struct IoBufs {
  double *b = nullptr, *x = nullptr, *stage = nullptr, *hist = nullptr;
  long long hist_cap = 0;
};

struct mpk_matrix {
  mpk_ctx *ctx;
  DMat A;
  int *rowflag = nullptr;
  int *fscratch = nullptr;  // [0..1] ticket, [2] bad_row, [3] nonfinite
  float factor_ms = 0.f;
  IoBufs io[5];
  double *fpub = nullptr;      // factorization publish-by-value copy (FactorArgs::pub)
  int max_row = 0;             // longest row
  std::vector<double> h_vals;  // complex interleave staging
  int *hres = nullptr;         // pinned factor init/result words
};

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CKR(x)                                                            \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess)                                                \
      return fail(MPK_CUDA_ERROR, std::string(#x) + ": " +                \
                                      cudaGetErrorString(e_));            \
  } while (0)

namespace {

__global__ void gather_kernel(const double *src, const int *perm, double *dst,
                              long long m, int cx) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= m) return;
  if (cx)
    reinterpret_cast<double2 *>(dst)[q] =
        reinterpret_cast<const double2 *>(src)[perm[q]];
  else
    dst[q] = src[perm[q]];
}

template <class T>
int upload(T **dst, const std::vector<T> &v, cudaStream_t st) {
  if (cudaMalloc(dst, sizeof(T) * (v.size() ? v.size() : 1)) != cudaSuccess)
    return 4;
  if (!v.empty())
    cudaMemcpyAsync(*dst, v.data(), sizeof(T) * v.size(),
                    cudaMemcpyHostToDevice, st);
  return 0;
}

void gather(const double *src, const int *perm, double *dst, long long m,
            bool cx, cudaStream_t st) {
  if (m <= 0) return;
  gather_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(src, perm, dst,
                                                              m, cx ? 1 : 0);
}

// Level order of a triangular dependency DAG: rows are visited in `visit`
// order (every dependency visited first), level(i) = 1 + max level of its
// dependencies deps[dlo(i) .. dhi(i)); returns the rows sorted by level
// (stable), i.e. a topological order whose warps hold independent rows.
template <class Lo, class Hi>
static int level_order(int n, bool descending, const int *deps, Lo dlo, Hi dhi,
                       std::vector<int> &ord, std::vector<int> &ptr) {
  std::vector<int> lev(n, 0);
  int nlev = 0;
  for (int s = 0; s < n; ++s) {
    const int i = descending ? n - 1 - s : s;
    int l = 0;
    for (int p = dlo(i); p < dhi(i); ++p) {
      const int d = lev[deps[p]] + 1;
      if (d > l) l = d;
    }
    lev[i] = l;
    if (l + 1 > nlev) nlev = l + 1;
  }
  std::vector<int> cnt(nlev + 1, 0);
  for (int i = 0; i < n; ++i) cnt[lev[i] + 1]++;
  for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
  ptr = cnt;
  ord.assign(n, 0);
  for (int s = 0; s < n; ++s) {
    const int i = descending ? n - 1 - s : s;
    ord[cnt[lev[i]]++] = i;
  }
  return nlev;
}

__global__ void gather_phase_kernel(const double *lu, SweepPhase ph, int n,
                                    int cx) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < ph.nent) {
    const int s = ph.src[t];
    if (cx)
      reinterpret_cast<double2 *>(ph.val)[t] =
          s >= 0 ? reinterpret_cast<const double2 *>(lu)[s] : make_double2(0.0, 0.0);
    else
      ph.val[t] = s >= 0 ? lu[s] : 0.0;
  }
  if (t < n) {
    const int s = ph.dsrc[t];
    if (cx)
      reinterpret_cast<double2 *>(ph.dval)[t] =
          s >= 0 ? reinterpret_cast<const double2 *>(lu)[s] : make_double2(1.0, 0.0);
    else
      ph.dval[t] = s >= 0 ? lu[s] : 1.0;
  }
}

// Host copy of one phase: rows in level order `ord` (level pointers `lev`),
// row i's entries (col, src) produced by `ent(i, cb)` in the reference's
// order and its divisor source `div(i)` (-1 if none).
struct HPhase {
  int nlev = 0, maxw = 0;
  std::vector<int> lev;
  std::vector<int4> desc;  // per position {row, first entry, count, 0}
  std::vector<int> col, src, dsrc;
};

template <class Ent, class Div>
static HPhase make_hphase(int n, const std::vector<int> &ord,
                          const std::vector<int> &lev, int nlev, Ent ent,
                          Div div) {
  HPhase h;
  h.nlev = nlev;
  h.lev = lev;
  h.desc.resize(n);
  h.dsrc.resize(n);
  for (int r = 0; r < n; ++r) {
    const int i = ord[r];
    const int e0 = (int)h.col.size();
    ent(i, [&](int c, int s) {
      h.col.push_back(c);
      h.src.push_back(s);
    });
    h.desc[r] = make_int4(i, e0, (int)h.col.size() - e0, 0);
    h.dsrc[r] = div(i);
  }
  for (int L = 0; L < nlev; ++L) h.maxw = std::max(h.maxw, lev[L + 1] - lev[L]);
  return h;
}

static void build_phase(SweepPhase &ph, int n, bool cx, const HPhase &h,
                        cudaStream_t st) {
  ph.nlev = h.nlev;
  ph.maxw = h.maxw;
  ph.nent = (long long)h.col.size();
  upload(&ph.lev, h.lev, st);
  upload(&ph.desc, h.desc, st);
  upload(&ph.col, h.col, st);
  upload(&ph.src, h.src, st);
  upload(&ph.dsrc, h.dsrc, st);
  const size_t w = cx ? 2 : 1;
  cudaMalloc(&ph.val, sizeof(double) * w * (h.col.size() + 1));
  cudaMalloc(&ph.dval, sizeof(double) * w * (n + 1));
}

static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Cluster sweep plan (ilu.cuh CSweep) for the phase pair (f, b).  Rows of a
// level are split over the C CTAs in contiguous chunks of about equal work.
// Replicated vector when it fits next to the staging buffers (smallest such
// C from 2 up, or MPK_CSWEEP_C), else the distributed layout.  Returns false
// if no layout fits in shared memory.
static bool build_cplan_c(CSweep &p, int n, bool cx, const HPhase &f,
                          const HPhase &b, int C, bool repl, bool dflow,
                          bool commit, cudaStream_t st) {
  if (dflow && !repl) return false;
  const int nl = f.nlev + b.nlev;
  if (nl > 8192) return false;
  const size_t esz = cx ? 16 : 8;
  auto split = [&](const HPhase &h, std::vector<int> &cta) {
    cta.assign(n, 0);
    for (int L = 0; L < h.nlev; ++L) {
      const int lo = h.lev[L], hi = h.lev[L + 1];
      long long W = 0;
      for (int r = lo; r < hi; ++r) W += h.desc[r].z + 4;
      long long acc = 0;
      for (int r = lo; r < hi; ++r) {
        cta[r] = (int)std::min<long long>(C - 1, acc * C / W);
        acc += h.desc[r].z + 4;
      }
    }
  };
  std::vector<int> cf, cb;
  split(f, cf);
  split(b, cb);
  std::vector<int> pk(n), nslot(C, 0), kf(n), kb(n);
  std::vector<std::vector<int>> srow(C), brow(C);
  for (int r = 0; r < n; ++r) {  // level order -> slots in compute order
    const int i = f.desc[r].x, c = cf[r];
    kf[i] = (int)srow[c].size();
    pk[i] = repl ? i : ((c << 24) | nslot[c]++);
    srow[c].push_back(i);
  }
  for (int r = 0; r < n; ++r) {
    const int i = b.desc[r].x, c = cb[r];
    kb[i] = (int)brow[c].size();
    brow[c].push_back(i);
  }
  int ninit = 0;
  for (int c = 0; c < C; ++c)
    ninit = std::max(ninit, (int)std::max(srow[c].size(), brow[c].size()));
  auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
  // sizes first (cheap), then the stream only when committing
  std::vector<int4> seg((size_t)nl * C);
  size_t total = 0, maxseg = 0;
  int maxnd = 0;
  std::vector<std::vector<int>> rows_of(C);
  for (int g = 0; g < nl; ++g) {
    const bool fw = g < f.nlev;
    const HPhase &h = fw ? f : b;
    const std::vector<int> &cta = fw ? cf : cb;
    const int L = fw ? g : g - f.nlev;
    for (int c = 0; c < C; ++c) rows_of[c].clear();
    for (int r = h.lev[L]; r < h.lev[L + 1]; ++r) rows_of[cta[r]].push_back(r);
    for (int c = 0; c < C; ++c) {
      int nd = (int)rows_of[c].size(), ne = 0;
      for (int r : rows_of[c]) ne += h.desc[r].z + (h.dsrc[r] >= 0 ? 1 : 0);
      const size_t bytes = nd ? a16(16 * (size_t)nd + a16(4 * (size_t)ne) + esz * ne) : 0;
      seg[(size_t)g * C + c] = make_int4((int)(total >> 4), (int)bytes, nd, ne);
      total += bytes;
      maxseg = std::max(maxseg, bytes);
      maxnd = std::max(maxnd, nd);
    }
  }
  int maxslots = 0;
  for (int c = 0; c < C; ++c) maxslots = std::max(maxslots, nslot[c]);
  if (repl) maxslots = n;
  if ((total >> 4) > (size_t)INT_MAX) return false;
  auto smem_for = [&](int nb) {
    if (dflow)
      return 144 + (size_t)nl * 16 + a16((size_t)n * esz) + a16((size_t)ninit * esz) +
             nb * maxseg;
    return 80 + (size_t)nl * 16 + a16((size_t)maxslots * esz) + nb * maxseg;
  };
  int nb = std::min(8, std::max(3, env_int("MPK_CSWEEP_NBUF", 4)));
  while (nb > 3 && smem_for(nb) > csweep_smem_limit()) --nb;
  if (smem_for(nb) > csweep_smem_limit()) return false;
  if (!commit) return true;
  std::vector<unsigned char> stream(total, 0);
  std::vector<long long> eoff;
  std::vector<int> esrc;
  for (int g = 0; g < nl; ++g) {
    const bool fw = g < f.nlev;
    const HPhase &h = fw ? f : b;
    const std::vector<int> &cta = fw ? cf : cb;
    const int L = fw ? g : g - f.nlev;
    for (int c = 0; c < C; ++c) rows_of[c].clear();
    for (int r = h.lev[L]; r < h.lev[L + 1]; ++r) rows_of[cta[r]].push_back(r);
    for (int c = 0; c < C; ++c) {
      const int4 sg = seg[(size_t)g * C + c];
      if (!sg.z) continue;
      const size_t off = (size_t)sg.x << 4;
      unsigned char *q = stream.data() + off;
      const size_t refs_off = 16 * (size_t)sg.z;
      const size_t vals_off = refs_off + a16(4 * (size_t)sg.w);
      int e = 0, k = 0;
      for (int r : rows_of[c]) {
        const int4 hd = h.desc[r];
        const bool dv = h.dsrc[r] >= 0;
        const int kk = fw ? kf[hd.x] : kb[hd.x];
        CSDesc d{pk[hd.x], e, hd.z, (kk << 1) | (dv ? 1 : 0)};
        std::memcpy(q + 16 * (size_t)k++, &d, sizeof d);
        const double one = 1.0;  // placeholder until the first gather
        for (int t = hd.y; t < hd.y + hd.z; ++t, ++e) {
          const int ref = pk[h.col[t]];
          std::memcpy(q + refs_off + 4 * (size_t)e, &ref, 4);
          std::memcpy(q + vals_off + esz * (size_t)e, &one, 8);
          eoff.push_back((long long)((off + vals_off + esz * (size_t)e) / 8));
          esrc.push_back(h.src[t]);
        }
        if (dv) {
          std::memcpy(q + vals_off + esz * (size_t)e, &one, 8);
          eoff.push_back((long long)((off + vals_off + esz * (size_t)e) / 8));
          esrc.push_back(h.dsrc[r]);
          ++e;
        }
      }
    }
  }
  p.C = C;
  p.T = std::min(1024, std::max(64, (maxnd + 31) / 32 * 32));
  if (dflow) p.T = std::min(1024, p.T + 32);  // + the producer warp
  p.nl = nl;
  p.nf = f.nlev;
  p.repl = repl ? 1 : 0;
  p.dflow = dflow ? 1 : 0;
  p.ninit = ninit;
  p.nbuf = nb;
  p.nval = (long long)esrc.size();
  p.maxslots = maxslots;
  p.maxseg = (int)maxseg;
  p.smem = smem_for(nb);
  std::vector<int> slot_row, slot_off(C + 1, 0), brows, boff(C + 1, 0);
  for (int c = 0; c < C; ++c) {
    slot_off[c + 1] = slot_off[c] + (int)srow[c].size();
    slot_row.insert(slot_row.end(), srow[c].begin(), srow[c].end());
    boff[c + 1] = boff[c] + (int)brow[c].size();
    brows.insert(brows.end(), brow[c].begin(), brow[c].end());
  }
  upload(&p.brow, brows, st);
  upload(&p.boff, boff, st);
  upload(&p.seg, seg, st);
  upload(&p.stream, stream, st);
  upload(&p.eoff, eoff, st);
  upload(&p.esrc, esrc, st);
  upload(&p.slot_row, slot_row, st);
  upload(&p.slot_off, slot_off, st);
  cudaStreamSynchronize(st);  // host staging vectors die here
  return true;
}

static bool build_cplan(CSweep &p, int n, bool cx, const HPhase &f,
                        const HPhase &b, cudaStream_t st) {
  if (n == 0) return false;
  const int cenv = env_int("MPK_CSWEEP_C", 0);
  const int renv = env_int("MPK_CSWEEP_REPL", -1);
  const int denv = env_int("MPK_CSWEEP_DFLOW", 1);
  const int cs[] = {2, 4, 8, 16};
  if (renv != 0) {  // replicated: smallest C that fits (or the forced one)
    for (int dflow = denv ? 1 : 0; dflow >= 0; --dflow) {
      for (int C : cs) {
        if (cenv && C != cenv) continue;
        if (build_cplan_c(p, n, cx, f, b, C, true, dflow, false, st))
          return build_cplan_c(p, n, cx, f, b, C, true, dflow, true, st);
      }
    }
    if (cenv == 1 && build_cplan_c(p, n, cx, f, b, 1, true, false, false, st))
      return build_cplan_c(p, n, cx, f, b, 1, true, false, true, st);
  }
  if (renv == 1) return false;
  const int maxw = std::max(f.maxw, b.maxw);
  int C = cenv ? cenv : std::min(16, std::max(1, maxw / env_int("MPK_CSWEEP_ROWS", 24)));
  if (C > 16) C = 16;
  if (build_cplan_c(p, n, cx, f, b, C, false, false, false, st))
    return build_cplan_c(p, n, cx, f, b, C, false, false, true, st);
  return false;
}

// Ring sweep plan (ilu.cuh RSweep) for the phase pair (f, b): the stream of
// chunks (rows of one level, at most `slot` bytes each) in forward-then-
// backward level order.  Returns false when the vector plus a useful ring
// does not fit in one SM's shared memory.
static bool build_rplan(RSweep &p, int n, bool cx, const HPhase &f,
                        const HPhase &b, cudaStream_t st) {
  if (n == 0) return false;
  const size_t esz = cx ? 16 : 8, vsz = cx ? 16 : 8;
  const size_t vec = ((size_t)n * esz + 15) / 16 * 16;
  const size_t limit = csweep_smem_limit();
  const int S = 4;
  // chunk table <= 8 B per chunk; bound the count by rows + levels
  const size_t tab_max = 8 * (size_t)(2 * n + f.nlev + b.nlev + 64);
  const size_t fixed = ((16 * S + 16 + 15) / 16) * 16 + vec;
  if (fixed + 4 * 4096 > limit) return false;
  size_t slot = std::min<size_t>(48 * 1024, (limit - fixed - std::min(tab_max, (size_t)16384)) / S);
  slot = slot / 16 * 16;
  if (slot < 4096) return false;
  struct Row { int row, cnt, dsrc, e0; };
  std::vector<unsigned char> stream;
  std::vector<RChunk> chunks;
  std::vector<long long> eoff, doff;
  std::vector<int> esrc, dsrcv;
  int maxrows = 0;
  bool fits = true;
  auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
  auto emit = [&](const HPhase &h, bool fw, int lo, int hi, bool end) {
    // rows [lo, hi) of phase h (positions in its level order)
    int nent = 0;
    for (int r = lo; r < hi; ++r) nent += h.desc[r].z;
    const int nr = hi - lo;
    const size_t cols_off = 16 + 32 * (size_t)nr;
    const size_t vals_off = cols_off + a16((size_t)nent * 4);
    const size_t bytes = a16(vals_off + (size_t)nent * vsz);
    if (bytes > slot) fits = false;  // one row larger than a ring slot
    const size_t off = stream.size();
    stream.resize(off + bytes, 0);
    unsigned char *q = stream.data() + off;
    const int hdr[4] = {nr, nent, end ? 1 : 0, fw ? 1 : 0};
    std::memcpy(q, hdr, 16);
    int e = 0;
    for (int r = lo; r < hi; ++r) {
      const int4 hd = h.desc[r];
      RDesc d{};
      d.row = hd.x;
      d.e0 = e;
      d.cnt = hd.z;
      d.hasdiv = h.dsrc[r] >= 0 ? 1 : 0;
      d.dr = 1.0;
      d.di = 0.0;
      std::memcpy(q + 16 + 32 * (size_t)(r - lo), &d, sizeof d);
      doff.push_back((long long)((off + 16 + 32 * (size_t)(r - lo) + 16) / 8));
      dsrcv.push_back(h.dsrc[r]);
      for (int t = hd.y; t < hd.y + hd.z; ++t, ++e) {
        const int c = h.col[t];
        std::memcpy(q + cols_off + 4 * (size_t)e, &c, 4);
        const double one = 1.0;  // placeholder until the first gather
        std::memcpy(q + vals_off + vsz * (size_t)e, &one, 8);
        eoff.push_back((long long)((off + vals_off + vsz * (size_t)e) / 8));
        esrc.push_back(h.src[t]);
      }
    }
    RChunk ch{};
    ch.off = (long long)off;
    ch.bytes = (int)bytes;
    ch.nrows = nr;
    ch.nent = nent;
    ch.level_end = end ? 1 : 0;
    ch.fwd = fw ? 1 : 0;
    chunks.push_back(ch);
    maxrows = std::max(maxrows, nr);
    return true;
  };
  auto phase = [&](const HPhase &h, bool fw) -> bool {
    for (int L = 0; L < h.nlev; ++L) {
      int lo = h.lev[L];
      int ne = 0;
      for (int r = h.lev[L]; r < h.lev[L + 1]; ++r) {
        const int c = h.desc[r].z;
        const size_t nb = a16(16 + 32 * (size_t)(r - lo + 1)) + a16((size_t)(ne + c) * 4) +
                          a16((size_t)(ne + c) * vsz);
        if (nb > slot) {
          if (r == lo) return false;  // a single row exceeds the slot
          emit(h, fw, lo, r, false);
          lo = r;
          ne = 0;
        }
        ne += c;
      }
      emit(h, fw, lo, h.lev[L + 1], true);
    }
    return true;
  };
  if (!phase(f, true) || !phase(b, false) || !fits) return false;
  const size_t tab = ((8 * chunks.size() + 15) / 16) * 16;
  const size_t smem = fixed + tab + S * slot;
  if (smem > limit) return false;
  p.nchunks = (int)chunks.size();
  p.S = S;
  p.slot = (int)slot;
  const int nc = std::min(992, std::max(32, (maxrows + 31) / 32 * 32));
  p.T = nc + 32;
  p.nent = (long long)esrc.size();
  p.ndesc = (long long)dsrcv.size();
  p.smem = smem;
  upload(&p.stream, stream, st);
  upload(&p.chunks, chunks, st);
  upload(&p.eoff, eoff, st);
  upload(&p.esrc, esrc, st);
  upload(&p.doff, doff, st);
  upload(&p.dsrc, dsrcv, st);
  cudaStreamSynchronize(st);  // host staging vectors die here
  return true;
}

static void free_rplan(RSweep &p) {
  void *q[] = {p.stream, p.chunks, p.eoff, p.esrc, p.doff, p.dsrc};
  for (void *v : q)
    if (v) cudaFree(v);
  p = RSweep{};
}

static void free_cplan(CSweep &p) {
  void *q[] = {p.seg, p.stream, p.eoff, p.esrc, p.slot_row, p.slot_off, p.brow, p.boff};
  for (void *v : q)
    if (v) cudaFree(v);
  p = CSweep{};
}

// Sweep structures of one apply direction: the single-CTA sweep matrices
// when the vector fits one SM, and the cluster plan when it fits a cluster.
// Average device time of `reps` applies through one sweep plan (dummy input;
// the plans hold placeholder values before the first factorization).
static float time_plan(SweepMats &sm, int n, bool cx, bool adjoint, int which,
                       cudaStream_t st) {
  double *in = nullptr, *z = nullptr;
  int *err = nullptr;
  const size_t w = cx ? 2 : 1;
  cudaMalloc(&in, sizeof(double) * w * n + 16);
  cudaMalloc(&z, sizeof(double) * w * n + 16);
  cudaMalloc(&err, sizeof(int) * 4);
  cudaMemsetAsync(in, 0, sizeof(double) * w * n + 16, st);
  SweepArgs a{};
  a.n = n;
  a.in_re = in;
  a.in_im = cx ? in + n : nullptr;
  a.z = z;
  a.y = z;
  a.err = err;
  a.done = nullptr;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const long long l0 = tl_launches;
  auto go = [&]() {
    if (which == 0)
      launch_rsweep(a, sm.rs, cx, adjoint, st);
    else
      launch_csweep(a, sm.cs, cx, adjoint, st);
  };
  go();  // warm-up (attributes, code)
  cudaEventRecord(e0, st);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  tl_launches = l0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(in);
  cudaFree(z);
  cudaFree(err);
  if (cudaGetLastError() != cudaSuccess) return 1e30f;
  return ms / reps;
}

// Sweep structures of one apply direction: the single-CTA sweep matrices
// when the vector fits one SM, the ring plan (one SM, vector + streamed
// entries in shared memory) and the cluster plan; when both of the latter
// exist, the faster one on this device is kept (timed here, once per
// pattern; MPK_SWEEP_PICK=ring|cluster overrides).
static bool build_sweeps(SweepMats &sm, int n, bool cx, const HPhase &f,
                         const HPhase &b, bool adjoint, cudaStream_t st) {
  bool single = false;
  if (sweep_uses_smem(n, cx)) {
    build_phase(sm.fwd, n, cx, f, st);
    build_phase(sm.bwd, n, cx, b, st);
    single = true;
  }
  if (env_int("MPK_RSWEEP", 1)) build_rplan(sm.rs, n, cx, f, b, st);
  CSweep alt;  // the barrier-per-level variant when the dataflow plan exists
  if (env_int("MPK_CSWEEP", 1)) {
    build_cplan(sm.cs, n, cx, f, b, st);
    if (sm.cs.dflow && env_int("MPK_CSWEEP_C", 0) == 0) {
      const char *old = getenv("MPK_CSWEEP_DFLOW");
      const std::string keep_old = old ? old : "";
      setenv("MPK_CSWEEP_DFLOW", "0", 1);
      build_cplan(alt, n, cx, f, b, st);
      if (old)
        setenv("MPK_CSWEEP_DFLOW", keep_old.c_str(), 1);
      else
        unsetenv("MPK_CSWEEP_DFLOW");
    }
  }
  const char *pick = getenv("MPK_SWEEP_PICK");
  // candidates: 0 ring, 1 cluster plan, 2 alternative cluster plan
  float t[3] = {1e30f, 1e30f, 1e30f};
  if (pick && !strcmp(pick, "ring")) {
    t[0] = 0.f;
  } else if (pick && !strcmp(pick, "cluster")) {
    t[1] = 0.f;
  } else {
    if (sm.rs.nchunks > 0) t[0] = time_plan(sm, n, cx, adjoint, 0, st);
    if (sm.cs.C > 0) t[1] = time_plan(sm, n, cx, adjoint, 1, st);
    if (alt.C > 0) {
      std::swap(sm.cs, alt);
      t[2] = time_plan(sm, n, cx, adjoint, 1, st);
      std::swap(sm.cs, alt);
    }
  }
  int best = 0;
  for (int i = 1; i < 3; ++i)
    if (t[i] < t[best]) best = i;
  if (best == 2) std::swap(sm.cs, alt);
  free_cplan(alt);
  if (best == 0 && sm.rs.nchunks > 0) {
    free_cplan(sm.cs);
  } else if (sm.cs.C > 0) {
    free_rplan(sm.rs);
  }
  return single;
}

static bool csweep_candidate(int n, bool cx) {
  // vector spread over at most 16 SMs with room for staging
  return env_int("MPK_CSWEEP", 1) &&
         (size_t)n * (cx ? 16 : 8) <= 16 * (size_t)160 * 1024;
}

static void gather_phase(const double *lu, const SweepPhase &ph, int n, bool cx,
                         cudaStream_t st) {
  const long long m = ph.nent > n ? ph.nent : n;
  if (m <= 0) return;
  ++tl_launches;
  gather_phase_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(lu, ph, n,
                                                                   cx ? 1 : 0);
}

static void free_phase(SweepPhase &ph) {
  void *p[] = {ph.lev, ph.desc, ph.col, ph.src, ph.val, ph.dsrc, ph.dval};
  for (void *q : p)
    if (q) cudaFree(q);
}

static void free_sweeps(SweepMats &sm) {
  free_phase(sm.fwd);
  free_phase(sm.bwd);
  free_cplan(sm.cs);
  free_rplan(sm.rs);
  free_wsweep(sm.wf);
  free_ssweep(sm.ss);
}

// Average device time of one plain ILU(0) apply (sentinel reset + sweep)
// through the current plan dispatch (do_sweep); placeholder values.
static float time_apply_plan(DMat &A, cudaStream_t st) {
  const int n = A.n;
  const size_t w = A.cx ? 2 : 1;
  double *in = nullptr, *y = nullptr, *z = nullptr;
  int *err = nullptr, *tick = nullptr;
  cudaMalloc(&in, sizeof(double) * w * n + 16);
  cudaMalloc(&y, sizeof(double) * w * n + 16);
  cudaMalloc(&z, sizeof(double) * w * n + 16);
  cudaMalloc(&err, sizeof(int) * 4);
  cudaMalloc(&tick, sizeof(int) * 4);
  cudaMemsetAsync(in, 0, sizeof(double) * w * n + 16, st);
  cudaMemsetAsync(tick, 0, sizeof(int) * 4, st);
  SweepArgs a{};
  a.n = n;
  a.rp = A.rp;
  a.ci = A.ci;
  a.dp = A.dp;
  a.lu = A.lu ? A.lu : A.val;
  a.ord_f = A.ord_f;
  a.ord_b = A.ord_b;
  a.lev_f = A.lev_f;
  a.lev_b = A.lev_b;
  a.nlev_f = A.levels_f;
  a.nlev_b = A.levels_b;
  a.in_re = in;
  a.in_im = A.cx ? in + n : nullptr;
  a.y = y;
  a.z = z;
  a.tick = tick;
  a.err = err;
  a.done = nullptr;
  const long long l0 = tl_launches;
  auto go = [&]() {
    launch_sweep_reset(y, z, n, A.cx, nullptr, st);
    do_sweep(A, a, false, st);
  };
  go();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  tl_launches = l0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  void *q[] = {in, y, z, err, tick};
  for (void *v : q) cudaFree(v);
  if (cudaGetLastError() != cudaSuccess) return 1e30f;
  return ms / reps;
}

}  // namespace

namespace mpk {

// Transposed gather structures for spmv_adjoint (ascending source row,
// _kernels.py:281-297) and the adjoint sweeps (U^T ascending rows,
// L^T descending rows; ilu.py:346-371).
void ensure_adjoint(DMat &A, cudaStream_t st) {
  const int n = A.n;
  const bool cx = A.cx;
  if (!A.at_rp) {
    const auto &rp = A.h_rp, &ci = A.h_ci, &dp = A.h_dp;
    std::vector<int> cnt(n + 1, 0), ucnt(n + 1, 0), lcnt(n + 1, 0);
    for (int i = 0; i < n; ++i)
      for (int p = rp[i]; p < rp[i + 1]; ++p) {
        cnt[ci[p] + 1]++;
        if (p > dp[i]) ucnt[ci[p] + 1]++;
        if (p < dp[i]) lcnt[ci[p] + 1]++;
      }
    for (int i = 0; i < n; ++i) {
      cnt[i + 1] += cnt[i];
      ucnt[i + 1] += ucnt[i];
      lcnt[i + 1] += lcnt[i];
    }
    std::vector<int> at_ci(cnt[n]), at_perm(cnt[n]), ut_ci(ucnt[n]),
        ut_perm(ucnt[n]), lt_ci(lcnt[n]), lt_perm(lcnt[n]);
    std::vector<int> f(cnt.begin(), cnt.end() - 1), uf(ucnt.begin(), ucnt.end() - 1),
        lf(lcnt.begin(), lcnt.end() - 1);
    for (int i = 0; i < n; ++i)
      for (int p = rp[i]; p < rp[i + 1]; ++p) {
        const int c = ci[p];
        at_ci[f[c]] = i;
        at_perm[f[c]++] = p;
        if (p > dp[i]) {
          ut_ci[uf[c]] = i;
          ut_perm[uf[c]++] = p;
        }
      }
    for (int j = n - 1; j >= 0; --j)
      for (int p = rp[j]; p < dp[j]; ++p) {
        const int c = ci[p];
        lt_ci[lf[c]] = j;
        lt_perm[lf[c]++] = p;
      }
    upload(&A.at_rp, cnt, st);
    upload(&A.at_ci, at_ci, st);
    upload(&A.at_perm, at_perm, st);
    upload(&A.ut_rp, ucnt, st);
    upload(&A.ut_ci, ut_ci, st);
    upload(&A.ut_perm, ut_perm, st);
    upload(&A.lt_rp, lcnt, st);
    upload(&A.lt_ci, lt_ci, st);
    upload(&A.lt_perm, lt_perm, st);
    std::vector<int> of, ob, pf, pb;
    A.levels_fa = level_order(
        n, false, ut_ci.data(), [&](int c) { return ucnt[c]; },
        [&](int c) { return ucnt[c + 1]; }, of, pf);
    A.levels_ba = level_order(
        n, true, lt_ci.data(), [&](int c) { return lcnt[c]; },
        [&](int c) { return lcnt[c + 1]; }, ob, pb);
    upload(&A.ord_fa, of, st);
    upload(&A.ord_ba, ob, st);
    upload(&A.lev_fa, pf, st);
    upload(&A.lev_ba, pb, st);
    if (sweep_uses_smem(n, cx) || csweep_candidate(n, cx)) {
      // U^H forward: column c of U in ascending source rows, / conj(U_cc);
      // L^H backward: column c of L in descending source rows
      const HPhase hf = make_hphase(
          n, of, pf, A.levels_fa,
          [&](int c, auto cb) {
            for (int q = ucnt[c]; q < ucnt[c + 1]; ++q) cb(ut_ci[q], ut_perm[q]);
          },
          [&](int c) { return dp[c]; });
      const HPhase hb = make_hphase(
          n, ob, pb, A.levels_ba,
          [&](int c, auto cb) {
            for (int q = lcnt[c]; q < lcnt[c + 1]; ++q) cb(lt_ci[q], lt_perm[q]);
          },
          [&](int) { return -1; });
      A.smat_adj_built = build_sweeps(A.smat_adj, n, cx, hf, hb, true, st);
      A.smat_adj.conj = true;
    }
    const size_t w = cx ? 2 : 1;
    cudaMalloc(&A.at_val, sizeof(double) * w * (A.nnz ? A.nnz : 1));
    cudaMalloc(&A.ut_val, sizeof(double) * w * (ut_ci.size() + 1));
    cudaMalloc(&A.lt_val, sizeof(double) * w * (lt_ci.size() + 1));
    gather(A.val, A.at_perm, A.at_val, (long long)at_ci.size(), cx, st);
    A.h_adj_sizes[0] = (long long)ut_ci.size();
    A.h_adj_sizes[1] = (long long)lt_ci.size();
  }
  if (A.factored && !A.adj_ready) {
    gather(A.lu, A.ut_perm, A.ut_val, A.h_adj_sizes[0], cx, st);
    gather(A.lu, A.lt_perm, A.lt_val, A.h_adj_sizes[1], cx, st);
    if (A.smat_adj_built) {
      gather_phase(A.lu, A.smat_adj.fwd, n, cx, st);
      gather_phase(A.lu, A.smat_adj.bwd, n, cx, st);
    }
    gather_csweep(A.lu, A.smat_adj.cs, cx, st);
    gather_rsweep(A.lu, A.smat_adj.rs, cx, st);
    A.adj_ready = true;
  }
}

}  // namespace mpk

extern "C" {

const char *mpk_last_error(void) { return g_err.c_str(); }
int mpk_version(void) { return 1; }

int mpk_ctx_create(int device, mpk_ctx **out) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(MPK_CUDA_ERROR, "no CUDA device available");
  if (device < 0 || device >= ndev)
    return fail(MPK_INVALID, "device index out of range");
  CKR(cudaSetDevice(device));
  mpk_ctx *c = new mpk_ctx;
  c->device = device;
  CKR(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  *out = c;
  return MPK_OK;
}

void mpk_ctx_destroy(mpk_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int mpk_ctx_synchronize(mpk_ctx *ctx) {
  CKR(cudaStreamSynchronize(ctx->stream));
  return MPK_OK;
}

void *mpk_ctx_stream(mpk_ctx *ctx) { return (void *)ctx->stream; }

int mpk_ctx_set_option(mpk_ctx *ctx, int option, int64_t value) {
  if (!ctx) return fail(MPK_INVALID, "null context");
  switch (option) {
    case MPK_OPT_REDUCTION:
      if (value != MPK_REDUCE_TREE && value != MPK_REDUCE_SEQUENTIAL)
        return fail(MPK_INVALID, "reduction mode must be 0 (tree) or 1 (sequential)");
      ctx->reduce_seq = (int)value;
      return MPK_OK;
    case MPK_OPT_PRECOND:
      if (value != MPK_PRECOND_NONE && value != MPK_PRECOND_ILU0_MIXED &&
          value != MPK_PRECOND_ILU0_FULL)
        return fail(MPK_INVALID, "precond must be 0 (none), 1 (ilu0-mixed) or 2 (ilu0)");
      ctx->precond = (int)value;
      return MPK_OK;
    default:
      return fail(MPK_INVALID, "unknown option");
  }
}

static thread_local int tl_precond = -1;   // mpk_thread_set_option overrides
static thread_local int tl_spmv_full = 0;

int mpk_thread_set_option(int option, int64_t value) {
  if (option == MPK_OPT_SPMV) {
    if (value > MPK_SPMV_FULL) return fail(MPK_INVALID, "spmv mode must be 0 (mixed) or 1 (full)");
    tl_spmv_full = value == MPK_SPMV_FULL ? 1 : 0;
    return MPK_OK;
  }
  if (option != MPK_OPT_PRECOND)
    return fail(MPK_INVALID, "per-thread options: MPK_OPT_PRECOND, MPK_OPT_SPMV");
  if (value > MPK_PRECOND_ILU0_FULL)
    return fail(MPK_INVALID, "precond must be 0 (none), 1 (ilu0-mixed) or 2 (ilu0)");
  tl_precond = value < 0 ? -1 : (int)value;
  return MPK_OK;
}

int64_t mpk_plane_ld(int64_t n) { return plane_ld(n); }

int mpk_csr_upload(mpk_ctx *ctx, int64_t n, int64_t nnz,
                   const int64_t *row_ptr, const int64_t *col_idx,
                   const double *val_re, const double *val_im,
                   mpk_matrix **out) {
  // CsrMatrix._validate sparse.py:217-233
  const double t_up0 = host_ms();
  if (n < 0 || nnz < 0) return fail(MPK_INVALID, "negative size");
  if (n > INT_MAX - 1 || nnz > INT_MAX)
    return fail(MPK_INVALID, "matrix too large for int32 indices");
  if (row_ptr[0] != 0 || row_ptr[n] != nnz)
    return fail(MPK_INVALID, "inconsistent CSR row_ptr");
  CKR(cudaSetDevice(ctx->device));
  mpk_matrix *m = new mpk_matrix;
  m->ctx = ctx;
  DMat &A = m->A;
  A.n = (int)n;
  A.nnz = nnz;
  A.cx = val_im != nullptr;
  A.h_rp.resize(n + 1);
  A.h_ci.resize(nnz);
  A.h_dp.assign(n, -1);
  A.h_rp[n] = (int)nnz;
  // validation (CsrMatrix._validate sparse.py:217-233), int32 copies and the
  // diagonal positions (_find_diagonals :235-243) in one pass over the
  // rows, on a few host threads for large matrices; the first offending row
  // (lowest index) is the one reported
  {
    const int T = n >= (1 << 16) ? (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency())) : 1;
    std::vector<int64_t> bad(T, -1), badkind(T, 0);
    std::vector<int> mrow(T, 0);
    auto work = [&](int t) {
      const int64_t per = (n + T - 1) / T, lo = std::min<int64_t>(n, per * t),
                    hi = std::min<int64_t>(n, per * (t + 1));
      for (int64_t i = lo; i < hi; ++i) {
        A.h_rp[i] = (int)row_ptr[i];
        if (row_ptr[i + 1] < row_ptr[i] || row_ptr[i] < 0 || row_ptr[i + 1] > nnz) {
          bad[t] = i;
          badkind[t] = 1;
          return;
        }
        mrow[t] = std::max<int>(mrow[t], (int)(row_ptr[i + 1] - row_ptr[i]));
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
          const int64_t c = col_idx[p];
          if (c < 0 || c >= n || (p > row_ptr[i] && c <= col_idx[p - 1])) {
            bad[t] = i;
            badkind[t] = 2;
            return;
          }
          A.h_ci[p] = (int)c;
          if (c == i) A.h_dp[i] = (int)p;
        }
      }
    };
    if (T == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t) th.emplace_back(work, t);
      for (auto &x : th) x.join();
    }
    for (int t = 0; t < T; ++t) {
      if (bad[t] < 0) continue;
      const int64_t i = bad[t];
      const bool rp_bad = badkind[t] == 1;
      delete m;
      if (rp_bad) return fail(MPK_INVALID, "row_ptr must be non-decreasing");
      return fail(MPK_INVALID, "row " + std::to_string(i) +
                                   ": columns must be strictly increasing and in range");
    }
    for (int t = 0; t < T; ++t) m->max_row = std::max(m->max_row, mrow[t]);
  }
  cudaStream_t st = ctx->stream;
  const double t_up1 = host_ms();
  // level orders of the L (forward) and U (backward) DAGs; a missing
  // diagonal (dp = -1) only matters for the structural check at factor time
  std::vector<int> of, ob, pf, pb;
  {
    const int *rp = A.h_rp.data(), *dp = A.h_dp.data();
    std::thread tb([&] {  // the two DAGs are independent
      A.levels_b = level_order(
          (int)n, true, A.h_ci.data(),
          [&](int i) { return dp[i] < 0 ? rp[i + 1] : dp[i] + 1; },
          [&](int i) { return rp[i + 1]; }, ob, pb);
    });
    A.levels_f = level_order(
        (int)n, false, A.h_ci.data(), [&](int i) { return rp[i]; },
        [&](int i) { return dp[i] < 0 ? rp[i] : dp[i]; }, of, pf);
    tb.join();
  }
  const double t_up2 = host_ms();
  // deep L DAG (grid stencils: thousands of levels): factorization tickets
  // in level order, each level padded to whole warps (ilu.cu launch_factor)
  if (A.levels_f >= 1024) {
    std::vector<int> op;
    op.reserve(of.size() + 32 * (size_t)A.levels_f);
    for (int l = 0; l < A.levels_f; ++l) {
      for (int q = pf[l]; q < pf[l + 1]; ++q) op.push_back(of[q]);
      while (op.size() % 32) op.push_back(-1);
    }
    A.nt_fp = (int)op.size();
    if (upload(&A.ord_fp, op, st)) {
      delete m;
      return fail(MPK_CUDA_ERROR, "allocation failed");
    }
  }
  if (upload(&A.rp, A.h_rp, st) || upload(&A.ci, A.h_ci, st) ||
      upload(&A.dp, A.h_dp, st) || upload(&A.ord_f, of, st) ||
      upload(&A.ord_b, ob, st) || upload(&A.lev_f, pf, st) ||
      upload(&A.lev_b, pb, st)) {
    delete m;
    return fail(MPK_CUDA_ERROR, "allocation failed");
  }
  if (sweep_uses_smem((int)n, A.cx) || csweep_candidate((int)n, A.cx)) {
    const int *rp = A.h_rp.data(), *dp = A.h_dp.data(), *ci = A.h_ci.data();
    const HPhase hf = make_hphase(
        (int)n, of, pf, A.levels_f,
        [&](int i, auto cb) {
          const int hi = dp[i] < 0 ? rp[i] : dp[i];
          for (int p = rp[i]; p < hi; ++p) cb(ci[p], p);
        },
        [&](int) { return -1; });
    const HPhase hb = make_hphase(
        (int)n, ob, pb, A.levels_b,
        [&](int i, auto cb) {
          const int lo = dp[i] < 0 ? rp[i + 1] : dp[i] + 1;
          for (int p = lo; p < rp[i + 1]; ++p) cb(ci[p], p);
        },
        [&](int i) { return dp[i]; });
    A.smat_built = build_sweeps(A.smat, (int)n, A.cx, hf, hb, false, st);
  }
  const size_t w = A.cx ? 2 : 1;
  std::vector<double> vals(w * nnz);
  for (int64_t p = 0; p < nnz; ++p) {
    if (A.cx) {
      vals[2 * p] = val_re[p];
      vals[2 * p + 1] = val_im[p];
    } else {
      vals[p] = val_re[p];
    }
  }
  if (upload(&A.val, vals, st)) {
    delete m;
    return fail(MPK_CUDA_ERROR, "allocation failed");
  }
  const long long L = plane_ld(n);
  CKR(cudaMalloc(&A.sw_y, sizeof(double) * w * L));
  CKR(cudaMalloc(&A.sw_y2, sizeof(double) * w * L));
  CKR(cudaMalloc(&A.tick, sizeof(int) * 8));
  CKR(cudaMemsetAsync(A.tick, 0, sizeof(int) * 8, st));
  CKR(cudaMalloc(&A.err, sizeof(int) * 2));
  CKR(cudaMemsetAsync(A.err, 0, sizeof(int) * 2, st));
  CKR(cudaMalloc(&m->rowflag, sizeof(int) * (n + 1)));
  CKR(cudaMalloc(&m->fscratch, sizeof(int) * 4));
  CKR(cudaStreamSynchronize(st));
  // shuffle-wavefront plan (swf.cu) for stencil-structured real sweeps.
  // On a large pattern (the vector does not fit one SM's shared memory, so
  // the alternative is the sync-free ticket sweep at >= 10 us per DAG level)
  // the plan is kept as soon as its analysis succeeds: timing the
  // alternatives would cost more than the solves the plan serves (cfg4:
  // 8 x 64 ms ticket applies).  Small patterns are timed against the plan
  // chosen above (MPK_SWEEP_PICK=swf forces it).
  const double t_plan0 = host_ms();
  if (getenv("MPK_VERBOSE"))
    fprintf(stderr,
            "[mpk] upload n=%lld: validate+copy %.1f ms, level orders %.1f ms, uploads + "
            "SMEM plans %.1f ms\n",
            (long long)n, t_up1 - t_up0, t_up2 - t_up1, t_plan0 - t_up2);
  bool swf_kept_untimed = false;
  {
    SSweep ss;
    if (build_ssweep(ss, (int)n, A.cx, A.h_rp.data(), A.h_ci.data(), A.h_dp.data(), st)) {
      const char *pick = getenv("MPK_SWEEP_PICK");
      const bool force = pick && !strcmp(pick, "swf");
      const bool other = pick && !force;
      const bool large = n >= (1 << 18) && !getenv("MPK_SWEEP_TIME_ALL");
      float tb = 1e30f, ts = 0.f;
      if (!force && !other && !large) tb = time_apply_plan(A, st);
      gather_ssweep(A.val, ss, st);  // timing values (regathered after factorization)
      A.smat.ss = ss;
      if (!force && !other && !large) ts = time_apply_plan(A, st);
      if (other || !(ts < tb)) free_ssweep(A.smat.ss);
      swf_kept_untimed = A.smat.ss.on && large;
      if (getenv("MPK_VERBOSE"))
        fprintf(stderr,
                "[mpk] shuffle-wavefront plan n=%lld: fwd Lc=%d lag=%d groups=%d S=%d pat=%d, "
                "bwd Lc=%d lag=%d groups=%d S=%d pat=%d, cluster=%d smem=%zu; apply %.4f ms vs "
                "%.4f ms (other plan) -> %s%s\n",
                (long long)n, ss.f.Lc, ss.f.lag, ss.f.ngroups, ss.f.S, ss.f.pat, ss.b.Lc,
                ss.b.lag, ss.b.ngroups, ss.b.S, ss.b.pat, ss.f.cl, ss.smem, ts, tb,
                A.smat.ss.on ? "shuffle-wavefront" : "other", large ? " (untimed: large n)" : "");
    }
    CKR(cudaGetLastError());
  }
  // lane-chunk wavefront plan (wf.cu) for banded sweep DAGs: kept when it
  // beats the plan chosen above on this device (MPK_SWEEP_PICK=wf forces it)
  if (!swf_kept_untimed && !A.smat.ss.on) {
    WSweep wf;
    if (build_wsweep(wf, (int)n, A.cx, A.h_rp.data(), A.h_ci.data(),
                     A.h_dp.data(), A.levels_f, A.levels_b, st)) {
      const char *pick = getenv("MPK_SWEEP_PICK");
      const bool force = pick && !strcmp(pick, "wf");
      const bool other = pick && !force;
      float tb = 1e30f, tw = 0.f;
      if (!force && !other) tb = time_apply_plan(A, st);
      A.smat.wf = wf;
      if (!force && !other) tw = time_apply_plan(A, st);
      if (other || !(tw < tb)) free_wsweep(A.smat.wf);
      if (getenv("MPK_VERBOSE"))
        fprintf(stderr,
                "[mpk] wavefront plan n=%lld: fwd Lc=%d lag=%d groups=%d S=%d, "
                "bwd Lc=%d lag=%d groups=%d S=%d; apply %.4f ms vs %.4f ms "
                "(other plan) -> %s\n",
                (long long)n, wf.f.Lc, wf.f.lag, wf.f.ngroups, wf.f.S, wf.b.Lc,
                wf.b.lag, wf.b.ngroups, wf.b.S, tw, tb,
                A.smat.wf.on ? "wavefront" : "other");
    }
    CKR(cudaGetLastError());
  }
  if (getenv("MPK_VERBOSE"))
    fprintf(stderr, "[mpk] upload n=%lld: sweep plans %.1f ms\n", (long long)n,
            host_ms() - t_plan0);
  // Sweep-pipelined SpMV plan (units.cu pspmv_kernel): for a large real
  // stencil pattern on the shuffle-wavefront plan, the 32-row chunks of A
  // sorted by the backward-DAG level at which all their columns' z values
  // exist (counting sort over the levels).
  if (A.smat.ss.on && !A.cx && n >= env_int("MPK_PIPE_MIN_N", 1 << 18) &&
      ssweep_bwd_ctas(A.smat.ss) > 0 &&
      env_int("MPK_PIPE", 1) != 0) {
    const double t_p0 = host_ms();
    const int *rp = A.h_rp.data(), *ci = A.h_ci.data();
    int maxlen = 0;
    for (int64_t i = 0; i < n; ++i) maxlen = std::max(maxlen, rp[i + 1] - rp[i]);
    if (maxlen <= kPipeRow) {
      std::vector<int> levb(n);
      for (int l = 0; l < A.levels_b; ++l)
        for (int q = pb[l]; q < pb[l + 1]; ++q) levb[ob[q]] = l;
      const int nch = (int)((n + 31) / 32);
      std::vector<int> ready(nch, 0), cnt(A.levels_b + 1, 0), order(nch), last(nch, 0);
      for (int c = 0; c < nch; ++c) {
        const int64_t i1 = std::min<int64_t>(n, (int64_t)c * 32 + 32);
        int r = -1, lc = 0;
        for (int q = rp[(int64_t)c * 32]; q < rp[i1]; ++q)
          if (levb[ci[q]] > r) {
            r = levb[ci[q]];
            lc = ci[q];
          }
        if (r < 0) r = 0;
        ready[c] = r;
        last[c] = lc;
        ++cnt[r + 1];
      }
      for (int l = 0; l < A.levels_b; ++l) cnt[l + 1] += cnt[l];
      for (int c = 0; c < nch; ++c) order[cnt[ready[c]]++] = c;
      A.pipe_nchunks = nch;
      if (upload(&A.pipe_order, order, st) || upload(&A.pipe_last, last, st) ||
          cudaMalloc(&A.pipe_state, sizeof(int) * 4) != cudaSuccess ||
          cudaMalloc(&A.pipe_flag, sizeof(int) * nch) != cudaSuccess) {
        delete m;
        return fail(MPK_CUDA_ERROR, "allocation failed");
      }
      CKR(cudaMemsetAsync(A.pipe_state, 0, sizeof(int) * 4, st));
      CKR(cudaMemsetAsync(A.pipe_flag, 0, sizeof(int) * nch, st));
      CKR(cudaStreamSynchronize(st));
    }
    if (getenv("MPK_VERBOSE"))
      fprintf(stderr, "[mpk] upload n=%lld: pipelined-SpMV plan %.1f ms (%d chunks)\n",
              (long long)n, host_ms() - t_p0, A.pipe_nchunks);
  }
  *out = m;
  return MPK_OK;
}

void mpk_csr_free(mpk_matrix *m) {
  if (!m) return;
  cudaSetDevice(m->ctx->device);
  cudaStreamSynchronize(m->ctx->stream);
  DMat &A = m->A;
  void *ptrs[] = {A.rp,     A.ci,     A.dp,      A.val,    A.lu,
                  A.at_rp,  A.at_ci,  A.at_perm, A.at_val, A.ut_rp,
                  A.ut_ci,  A.ut_perm, A.lt_rp,  A.lt_ci,  A.lt_perm,
                  A.ut_val, A.lt_val, A.sw_y,    A.sw_y2,  A.tick,
                  A.ord_f,  A.ord_b,  A.ord_fa,  A.ord_ba,
                  A.lev_f,  A.lev_b,  A.lev_fa,  A.lev_ba,
                  A.err,    m->rowflag, m->fscratch, A.ord_fp,
                  A.pipe_order, A.pipe_last, A.pipe_state, A.pipe_flag};
  if (m->hres) cudaFreeHost(m->hres);
  if (m->fpub) cudaFree(m->fpub);
  for (auto &B : m->io) {
    void *q[] = {B.b, B.x, B.stage, B.hist};
    for (void *v : q)
      if (v) cudaFree(v);
  }
  free_sweeps(A.smat);
  free_sweeps(A.smat_adj);
  if (A.lu_mc) cudaFree(A.lu_mc);
  if (A.mcv) cudaFree(A.mcv);
  if (A.rcp_mc) cudaFree(A.rcp_mc);
  if (A.sw_mc) cudaFree(A.sw_mc);
  if (A.sw_mc2) cudaFree(A.sw_mc2);
  for (void *p : ptrs)
    if (p) cudaFree(p);
  delete m;
}

int mpk_ilu0_factor(mpk_matrix *m, int64_t *bad_row, int32_t *structural) {
  DMat &A = m->A;
  cudaStream_t st = m->ctx->stream;
  CKR(cudaSetDevice(m->ctx->device));
  // _structural_check ilu.py:172-175
  for (int i = 0; i < A.n; ++i) {
    if (A.h_dp[i] < 0) {
      if (bad_row) *bad_row = i;
      if (structural) *structural = 1;
      return fail(MPK_SINGULAR_PIVOT,
                  "ILU(0): structurally missing pivot U[" + std::to_string(i) +
                      "," + std::to_string(i) + "]");
    }
  }
  const size_t w = A.cx ? 2 : 1;
  if (!A.lu) CKR(cudaMalloc(&A.lu, sizeof(double) * w * (A.nnz ? A.nnz : 1)));
  CKR(cudaMemcpyAsync(A.lu, A.val, sizeof(double) * w * A.nnz,
                      cudaMemcpyDeviceToDevice, st));
  CKR(cudaMemsetAsync(m->rowflag, 0, sizeof(int) * (A.n + 1), st));
  if (!m->hres) CKR(cudaMallocHost(&m->hres, sizeof(int) * 8));
  int *init = m->hres;  // pinned (pageable copies serialise concurrent solves)
  init[0] = 0;
  init[1] = 0;
  init[2] = INT_MAX;
  init[3] = 0;
  CKR(cudaMemcpyAsync(m->fscratch, init, sizeof(int) * 4, cudaMemcpyHostToDevice,
                      st));
  FactorArgs fa{};
  fa.n = A.n;
  fa.rp = A.rp;
  fa.ci = A.ci;
  fa.dp = A.dp;
  fa.lu = A.lu;
  fa.rowflag = m->rowflag;
  fa.ord = A.ord_f;
  fa.lev = A.lev_f;
  fa.nlev = A.levels_f;
  fa.ordp = A.ord_fp;
  fa.nt = A.nt_fp;
  // real rows that all fit the register-resident row routine, shallow DAG:
  // results are published by value (ilu.cuh FactorArgs::pub).  Measured:
  // cfg1 0.46 -> 0.34 ms, cfg2 0.27 -> 0.25 ms; on the deep level-ordered
  // cfg4 DAG the ~38 k waiting rows polling five values each swamp L2
  // (39 -> 96 ms), so deep DAGs keep the one-word flags.  MPK_FACTOR_PUB=0|1
  // forces either protocol.
  if (!A.cx && A.nnz > 0 && m->max_row <= 32 &&
      env_int("MPK_FACTOR_PUB", A.ord_fp ? 0 : 1)) {
    if (!m->fpub) CKR(cudaMalloc(&m->fpub, sizeof(double) * A.nnz));
    launch_fill_sentinel(m->fpub, A.nnz, st);
    fa.pub = m->fpub;
  }
  fa.tick = m->fscratch;
  fa.bad_row = m->fscratch + 2;
  fa.nonfinite = m->fscratch + 3;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  if (A.n > 0) launch_factor(fa, A.cx, st);
  cudaEventRecord(e1, st);
  int *res = m->hres + 4;
  CKR(cudaMemcpyAsync(res, m->fscratch, sizeof(int) * 4, cudaMemcpyDeviceToHost,
                      st));
  CKR(cudaStreamSynchronize(st));
  CKR(cudaGetLastError());
  cudaEventElapsedTime(&m->factor_ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  A.factored = false;
  A.adj_ready = false;
  if (res[2] != INT_MAX) {
    if (bad_row) *bad_row = res[2];
    if (structural) *structural = 0;
    return fail(MPK_SINGULAR_PIVOT, "ILU(0): zero pivot U[" +
                                        std::to_string(res[2]) + "," +
                                        std::to_string(res[2]) + "]");
  }
  if (res[3]) return fail(MPK_NUMERIC_BREAKDOWN, "non-finite value in ILU(0) factors");
  A.factored = true;
  if (A.smat_built) {
    gather_phase(A.lu, A.smat.fwd, A.n, A.cx, m->ctx->stream);
    gather_phase(A.lu, A.smat.bwd, A.n, A.cx, m->ctx->stream);
  }
  gather_csweep(A.lu, A.smat.cs, A.cx, m->ctx->stream);
  gather_rsweep(A.lu, A.smat.rs, A.cx, m->ctx->stream);
  gather_wsweep(A.lu, A.smat.wf, A.cx, m->ctx->stream);
  gather_ssweep(A.lu, A.smat.ss, m->ctx->stream);
  return MPK_OK;
}

// binary64 values (complex: interleaved re, im) -> flat K-component
// entries (complex: re[K], im[K]) with zero tails
__global__ void promote_vals_kernel(long long nnz, int k, int cx, const double *v, double *o) {
  const int w = cx ? 2 * k : k;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < nnz;
       p += (long long)gridDim.x * blockDim.x)
    for (int c = 0; c < w; ++c) {
      const bool head = (c % k) == 0;
      o[p * w + c] = !head ? 0.0 : (cx ? v[2 * p + c / k] : v[p]);
    }
}

// planar MC matrix values (DMat::mcv) -> flat K-component entries
__global__ void mc_vals_kernel(long long nnz, int w, const double *v, long long vld, double *o) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < nnz;
       p += (long long)gridDim.x * blockDim.x)
    for (int c = 0; c < w; ++c) o[p * w + c] = v[c * vld + p];
}

// ilu0_factorize (ilu.py:279-281 -> _factorize_tuples at precision k > 1) of
// the uploaded binary64 matrix promoted to k components; real field.
int mpk_ilu0_factor_full(mpk_matrix *m, int k, int64_t *bad_row, int32_t *structural) {
  DMat &A = m->A;
  cudaStream_t st = m->ctx->stream;
  if (k < 2 || k > 4) return fail(MPK_INVALID, "working-precision ILU(0): k = 2..4");
  const int W = A.cx ? 2 * k : k;
  CKR(cudaSetDevice(m->ctx->device));
  for (int i = 0; i < A.n; ++i) {  // _structural_check ilu.py:172-175
    if (A.h_dp[i] < 0) {
      if (bad_row) *bad_row = i;
      if (structural) *structural = 1;
      return fail(MPK_SINGULAR_PIVOT, "ILU(0): structurally missing pivot U[" +
                                          std::to_string(i) + "," + std::to_string(i) + "]");
    }
  }
  const long long L = plane_ld(A.n);
  if (A.lu_mc_k != k) {
    if (A.lu_mc) cudaFree(A.lu_mc);
    if (A.rcp_mc) cudaFree(A.rcp_mc);
    if (A.sw_mc) cudaFree(A.sw_mc);
    if (A.sw_mc2) cudaFree(A.sw_mc2);
    A.lu_mc = A.rcp_mc = A.sw_mc = A.sw_mc2 = nullptr;
    CKR(cudaMalloc(&A.lu_mc, sizeof(double) * W * (A.nnz ? A.nnz : 1)));
    CKR(cudaMalloc(&A.rcp_mc, sizeof(double) * (A.cx ? 2 * (2 * k + 1) : k) * (A.n ? A.n : 1)));
    CKR(cudaMalloc(&A.sw_mc, sizeof(double) * W * L + 16));
    CKR(cudaMalloc(&A.sw_mc2, sizeof(double) * W * L + 16));
    A.lu_mc_k = k;
  }
  A.mc_factored = false;
  if (A.nnz > 0) {
    ++tl_launches;
    if (A.mcv && A.mcv_k == k)  // MC-valued matrix: ilu0_factorize(A) factors A itself
      mc_vals_kernel<<<sm_count() * 4, 256, 0, st>>>(A.nnz, W, A.mcv, A.mcv_ld, A.lu_mc);
    else
      promote_vals_kernel<<<sm_count() * 4, 256, 0, st>>>(A.nnz, k, A.cx ? 1 : 0, A.val, A.lu_mc);
  }
  CKR(cudaMemsetAsync(m->rowflag, 0, sizeof(int) * (A.n + 1), st));
  if (!m->hres) CKR(cudaMallocHost(&m->hres, sizeof(int) * 8));
  int *init = m->hres;
  init[0] = 0;
  init[1] = 0;
  init[2] = INT_MAX;
  init[3] = 0;
  CKR(cudaMemcpyAsync(m->fscratch, init, sizeof(int) * 4, cudaMemcpyHostToDevice, st));
  FactorMcArgs fa{};
  fa.n = A.n;
  fa.cx = A.cx ? 1 : 0;
  fa.rp = A.rp;
  fa.ci = A.ci;
  fa.dp = A.dp;
  fa.lu = A.lu_mc;
  fa.rowflag = m->rowflag;
  fa.tick = m->fscratch;
  fa.bad_row = m->fscratch + 2;
  fa.nonfinite = m->fscratch + 3;
  fa.ord = A.ord_f;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  if (A.n > 0) launch_factor_mc(fa, k, st);
  CKR(cudaGetLastError());
  cudaEventRecord(e1, st);
  int *res = m->hres + 4;
  CKR(cudaMemcpyAsync(res, m->fscratch, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  cudaEventElapsedTime(&m->factor_ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (res[2] != INT_MAX) {
    if (bad_row) *bad_row = res[2];
    if (structural) *structural = 0;
    return fail(MPK_SINGULAR_PIVOT, "ILU(0): zero pivot U[" + std::to_string(res[2]) + "," +
                                        std::to_string(res[2]) + "]");
  }
  if (res[3]) return fail(MPK_NUMERIC_BREAKDOWN, "non-finite value in ILU(0) factors");
  launch_recip_mc(A.n, A.dp, A.lu_mc, A.rcp_mc, k, A.cx, st);
  CKR(cudaGetLastError());
  A.mc_factored = true;
  return MPK_OK;
}

int mpk_ilu0_download_full(mpk_matrix *m, int k, double *lu) {
  DMat &A = m->A;
  if (!A.mc_factored || A.lu_mc_k != k) return fail(MPK_INVALID, "no working-precision factors");
  CKR(cudaSetDevice(m->ctx->device));
  CKR(cudaMemcpy(lu, A.lu_mc, sizeof(double) * (A.cx ? 2 * k : k) * A.nnz,
                 cudaMemcpyDeviceToHost));
  return MPK_OK;
}

// ilu0_apply / ilu0_apply_adjoint (ilu.py:410-433) at working precision,
// (n,k) host arrays
int mpk_ilu0_apply_full(mpk_matrix *m, int k, const double *r, double *z) {
  return mpk_ilu0_apply_full_ex(m, k, r, z, 0);
}
int mpk_ilu0_apply_full_ex(mpk_matrix *m, int k, const double *r, double *z, int adjoint) {
  DMat &A = m->A;
  if (adjoint) ensure_adjoint(A, m->ctx->stream);
  if (!A.mc_factored || A.lu_mc_k != k) return fail(MPK_INVALID, "no working-precision factors");
  CKR(cudaSetDevice(m->ctx->device));
  cudaStream_t st = m->ctx->stream;
  const long long n = A.n, L = plane_ld(A.n);
  double *din = nullptr, *dz = nullptr, *stage = nullptr;
  const int c2 = A.cx ? 2 : 1;
  CKR(cudaMalloc(&din, sizeof(double) * c2 * k * L + 16));
  CKR(cudaMalloc(&dz, sizeof(double) * c2 * k * L + 16));
  CKR(cudaMalloc(&stage, sizeof(double) * c2 * k * (n ? n : 1)));
  CKR(cudaMemcpyAsync(stage, r, sizeof(double) * n * k * c2, cudaMemcpyHostToDevice, st));
  launch_to_planar(n, k, stage, A.cx ? stage + n * k : nullptr, din, st);
  CKR(cudaMemsetAsync(A.err, 0, sizeof(int), st));
  SweepMcArgs a{};
  a.n = A.n;
  a.ld = L;
  a.rp = A.rp;
  a.ci = A.ci;
  a.dp = A.dp;
  a.lu = A.lu_mc;
  a.rcp = A.rcp_mc;
  a.in = din;
  a.y = A.sw_mc;
  a.z = dz;
  a.tick = A.tick;
  a.err = A.err;
  a.done = nullptr;
  a.adjoint = adjoint;
  a.cx = A.cx ? 1 : 0;
  a.ut_rp = A.ut_rp;
  a.ut_ci = A.ut_ci;
  a.ut_perm = A.ut_perm;
  a.lt_rp = A.lt_rp;
  a.lt_ci = A.lt_ci;
  a.lt_perm = A.lt_perm;
  a.ord_f = adjoint ? A.ord_fa : A.ord_f;
  a.ord_b = adjoint ? A.ord_ba : A.ord_b;
  launch_sweep_mc(a, k, st);
  launch_from_planar(n, k, dz, stage, A.cx ? stage + n * k : nullptr, st);
  CKR(cudaMemcpyAsync(z, stage, sizeof(double) * n * k * c2, cudaMemcpyDeviceToHost, st));
  int e = 0;
  CKR(cudaMemcpyAsync(&e, A.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  cudaFree(din);
  cudaFree(dz);
  cudaFree(stage);
  if (e) return fail(MPK_NUMERIC_BREAKDOWN, "non-finite value in triangular sweep");
  return MPK_OK;
}

int mpk_ilu0_download(mpk_matrix *m, double *lu_re, double *lu_im) {
  DMat &A = m->A;
  if (!A.factored) return fail(MPK_INVALID, "matrix is not factored");
  CKR(cudaSetDevice(m->ctx->device));
  const size_t w = A.cx ? 2 : 1;
  std::vector<double> h(w * A.nnz);
  CKR(cudaMemcpy(h.data(), A.lu, sizeof(double) * h.size(),
                 cudaMemcpyDeviceToHost));
  for (long long p = 0; p < A.nnz; ++p) {
    if (A.cx) {
      lu_re[p] = h[2 * p];
      lu_im[p] = h[2 * p + 1];
    } else {
      lu_re[p] = h[p];
    }
  }
  return MPK_OK;
}

// The sync-free sweeps signal "value ready" by overwriting a signalling-NaN
// sentinel (common.cuh kSentBits; the wavefront plans test its high word).
// No binary64 operation produces a signalling NaN, so inside a solve every
// sweep input (an MC arithmetic result) is safe; a caller-supplied vector
// could carry the pattern through a row without entries (a pure copy) and
// stall its consumers.  The apply entry points therefore quiet such values
// (-> the quiet NaN the hardware would make of them) before the sweep: the
// apply then ends with NumericBreakdownError like any non-finite input.
__global__ void quiet_sentinels_kernel(double *v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (__double2hiint(v[i]) == (int)(kSentBits >> 32))
      v[i] = __longlong_as_double((long long)kQNaNBits);
}

// apply on a device planar-MC input; output F vector in `fz`
static int apply_dev(mpk_matrix *m, int k, const double *in_mc, double *fz,
                     int adjoint) {
  DMat &A = m->A;
  cudaStream_t st = m->ctx->stream;
  if (adjoint) ensure_adjoint(A, st);
  const long long L = plane_ld(A.n);
  CKR(cudaMemsetAsync(A.err, 0, sizeof(int), st));
  launch_sweep_reset(A.sw_y, fz, A.n, A.cx, nullptr, st);
  if (A.n > 0) {  // head planes only: the sweeps read the demoted input
    double *head = const_cast<double *>(in_mc);
    quiet_sentinels_kernel<<<grid_for(A.n), kBlock, 0, st>>>(head, A.n);
    if (A.cx) quiet_sentinels_kernel<<<grid_for(A.n), kBlock, 0, st>>>(head + (long long)k * L, A.n);
  }
  SweepArgs a{};
  a.n = A.n;
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
  a.in_re = in_mc;
  a.in_im = A.cx ? in_mc + (long long)k * L : nullptr;
  a.y = A.sw_y;
  a.z = fz;
  a.tick = A.tick;
  a.err = A.err;
  a.done = nullptr;
  if (A.n > 0) do_sweep(A, a, adjoint != 0, st);
  int err = 0;
  CKR(cudaMemcpyAsync(&err, A.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  CKR(cudaGetLastError());
  if (err)
    return fail(MPK_NUMERIC_BREAKDOWN, "non-finite value in triangular sweep");
  return MPK_OK;
}

int mpk_ilu0_apply_f64(mpk_matrix *m, const double *r_re, const double *r_im,
                       double *z_re, double *z_im, int adjoint) {
  DMat &A = m->A;
  if (!A.factored) return fail(MPK_INVALID, "matrix is not factored");
  if (A.cx != (r_im != nullptr))
    return fail(MPK_INVALID, "field mismatch: factors/vector");
  CKR(cudaSetDevice(m->ctx->device));
  cudaStream_t st = m->ctx->stream;
  const long long L = plane_ld(A.n);
  double *din = nullptr, *dz = nullptr, *hin = nullptr;
  // binary64 input as a k=1 "MC" vector: planes re[, im]
  CKR(cudaMalloc(&din, sizeof(double) * 2 * L));
  CKR(cudaMalloc(&dz, sizeof(double) * 2 * L));
  CKR(cudaMemcpyAsync(din, r_re, sizeof(double) * A.n, cudaMemcpyHostToDevice, st));
  if (A.cx)
    CKR(cudaMemcpyAsync(din + L, r_im, sizeof(double) * A.n,
                        cudaMemcpyHostToDevice, st));
  (void)hin;
  // for a k=1 input the "demotion" of the complex value must be the
  // identity (complex(re, im) in ilu.py:301): the device applies the numpy
  // re + 1j*im rounding, which only normalises signed zeros.
  int rc = apply_dev(m, 1, din, dz, adjoint);
  if (rc == MPK_OK) {
    if (A.cx) {
      std::vector<double> h(2 * A.n);
      CKR(cudaMemcpy(h.data(), dz, sizeof(double) * 2 * A.n, cudaMemcpyDeviceToHost));
      for (int i = 0; i < A.n; ++i) {
        z_re[i] = h[2 * i];
        z_im[i] = h[2 * i + 1];
      }
    } else {
      CKR(cudaMemcpy(z_re, dz, sizeof(double) * A.n, cudaMemcpyDeviceToHost));
    }
  }
  cudaFree(din);
  cudaFree(dz);
  return rc;
}

static int to_dev_planar(mpk_ctx *ctx, int64_t n, int k, const double *re,
                         const double *im, double **dev) {
  cudaStream_t st = ctx->stream;
  const long long L = plane_ld(n);
  const int planes = k * (im ? 2 : 1);
  double *tmp = nullptr;
  CKR(cudaMalloc(dev, sizeof(double) * planes * L + 16));
  CKR(cudaMemsetAsync(*dev, 0, sizeof(double) * planes * L + 16, st));
  if (n == 0) return MPK_OK;
  CKR(cudaMalloc(&tmp, sizeof(double) * n * k * (im ? 2 : 1)));
  CKR(cudaMemcpyAsync(tmp, re, sizeof(double) * n * k, cudaMemcpyHostToDevice, st));
  if (im)
    CKR(cudaMemcpyAsync(tmp + n * k, im, sizeof(double) * n * k,
                        cudaMemcpyHostToDevice, st));
  launch_to_planar(n, k, tmp, im ? tmp + n * k : nullptr, *dev, st);
  CKR(cudaStreamSynchronize(st));
  cudaFree(tmp);
  return MPK_OK;
}

static int from_dev_planar(mpk_ctx *ctx, int64_t n, int k, const double *dev,
                           double *re, double *im) {
  cudaStream_t st = ctx->stream;
  if (n == 0) return MPK_OK;
  double *tmp = nullptr;
  CKR(cudaMalloc(&tmp, sizeof(double) * n * k * (im ? 2 : 1)));
  launch_from_planar(n, k, dev, tmp, im ? tmp + n * k : nullptr, st);
  CKR(cudaMemcpyAsync(re, tmp, sizeof(double) * n * k, cudaMemcpyDeviceToHost, st));
  if (im)
    CKR(cudaMemcpyAsync(im, tmp + n * k, sizeof(double) * n * k,
                        cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  cudaFree(tmp);
  return MPK_OK;
}

int mpk_to_planar(mpk_ctx *ctx, int64_t n, int k, const double *re,
                  const double *im, double *dev) {
  CKR(cudaSetDevice(ctx->device));
  double *d = nullptr;
  int rc = to_dev_planar(ctx, n, k, re, im, &d);
  if (rc) return rc;
  const long long L = plane_ld(n);
  CKR(cudaMemcpy(dev, d, sizeof(double) * k * (im ? 2 : 1) * L,
                 cudaMemcpyDeviceToDevice));
  cudaFree(d);
  return MPK_OK;
}

int mpk_from_planar(mpk_ctx *ctx, int64_t n, int k, const double *dev,
                    double *re, double *im, int cx) {
  CKR(cudaSetDevice(ctx->device));
  return from_dev_planar(ctx, n, k, dev, re, cx ? im : nullptr);
}

int mpk_ilu0_apply_mixed(mpk_matrix *m, int k, const double *r_re,
                         const double *r_im, double *z_re, double *z_im,
                         int adjoint) {
  DMat &A = m->A;
  if (!A.factored) return fail(MPK_INVALID, "matrix is not factored");
  if (k < 2) return fail(MPK_INVALID, "mixed apply expects a working precision above binary64");
  if (A.cx != (r_im != nullptr)) return fail(MPK_INVALID, "factors/vector mismatch");
  CKR(cudaSetDevice(m->ctx->device));
  double *din = nullptr, *dz = nullptr;
  int rc = to_dev_planar(m->ctx, A.n, k, r_re, r_im, &din);
  if (rc) return rc;
  const long long L = plane_ld(A.n);
  CKR(cudaMalloc(&dz, sizeof(double) * 2 * L));
  rc = apply_dev(m, k, din, dz, adjoint);
  if (rc == MPK_OK) {
    // _promote_exact ilu.py:436-445 after numpy demotion of z (sparse.py:392)
    const int w = A.cx ? 2 : 1;
    std::vector<double> h(w * A.n);
    CKR(cudaMemcpy(h.data(), dz, sizeof(double) * w * A.n, cudaMemcpyDeviceToHost));
    std::memset(z_re, 0, sizeof(double) * A.n * k);
    if (A.cx) std::memset(z_im, 0, sizeof(double) * A.n * k);
    for (int i = 0; i < A.n; ++i) {
      if (A.cx) {
        const double re0 = h[2 * i], im0 = h[2 * i + 1];
        z_re[(size_t)i * k] = mpk::dadd(re0, mpk::dsub(mpk::dmul(0.0, im0), 0.0));
        z_im[(size_t)i * k] = mpk::dadd(0.0, im0);
      } else {
        z_re[(size_t)i * k] = h[i];
      }
    }
  }
  cudaFree(din);
  cudaFree(dz);
  return rc;
}

int mpk_spmv_mixed(mpk_matrix *m, int k, const double *x_re,
                   const double *x_im, double *y_re, double *y_im,
                   int adjoint) {
  DMat &A = m->A;
  if (k < 2) return fail(MPK_INVALID, "mixed SpMV requires a working precision above binary64");
  if (A.cx != (x_im != nullptr))
    return fail(MPK_INVALID, std::string("field mismatch: matrix ") +
                                 (A.cx ? "complex" : "real") + ", vector " +
                                 (x_im ? "complex" : "real"));
  CKR(cudaSetDevice(m->ctx->device));
  cudaStream_t st = m->ctx->stream;
  double *dx = nullptr, *dy = nullptr;
  int rc = to_dev_planar(m->ctx, A.n, k, x_re, x_im, &dx);
  if (rc) return rc;
  const long long L = plane_ld(A.n);
  CKR(cudaMalloc(&dy, sizeof(double) * k * 2 * L + 16));
  rc = unit_spmv(A, k, adjoint != 0, false, dx, dy, st);
  if (rc) return fail(rc, "unsupported k");
  CKR(cudaGetLastError());
  rc = from_dev_planar(m->ctx, A.n, k, dy, y_re, A.cx ? y_im : nullptr);
  cudaFree(dx);
  cudaFree(dy);
  return rc;
}

int mpk_hdot(mpk_ctx *ctx, int64_t n, int k, const double *x_re,
             const double *x_im, const double *y_re, const double *y_im,
             double *out_re, double *out_im) {
  if (k < 2 || k > 4) return fail(MPK_INVALID, "k must be 2..4");
  CKR(cudaSetDevice(ctx->device));
  double *dx = nullptr, *dy = nullptr;
  int rc = to_dev_planar(ctx, n, k, x_re, x_im, &dx);
  if (rc) return rc;
  rc = to_dev_planar(ctx, n, k, y_re, y_im, &dy);
  if (rc) return rc;
  double out[8];
  rc = unit_reduce(k, x_im != nullptr, 0, n, dx, dy, out, ctx->stream, ctx->reduce_seq);
  for (int c = 0; c < k; ++c) {
    out_re[c] = out[c];
    if (out_im) out_im[c] = out[4 + c];
  }
  cudaFree(dx);
  cudaFree(dy);
  return rc ? fail(rc, "hdot failed") : MPK_OK;
}

int mpk_norm2(mpk_ctx *ctx, int64_t n, int k, const double *x_re,
              const double *x_im, double *out) {
  if (k < 2 || k > 4) return fail(MPK_INVALID, "k must be 2..4");
  CKR(cudaSetDevice(ctx->device));
  double *dx = nullptr;
  int rc = to_dev_planar(ctx, n, k, x_re, x_im, &dx);
  if (rc) return rc;
  double o[8];
  rc = unit_reduce(k, x_im != nullptr, 1, n, dx, dx, o, ctx->stream, ctx->reduce_seq);
  for (int c = 0; c < k; ++c) out[c] = o[c];
  cudaFree(dx);
  return rc ? fail(rc, "norm2 failed") : MPK_OK;
}

int mpk_axpy(mpk_ctx *ctx, int64_t n, int k, const double *alpha_re,
             const double *alpha_im, const double *x_re, const double *x_im,
             const double *y_re, const double *y_im, double *out_re,
             double *out_im) {
  if (k < 2 || k > 4) return fail(MPK_INVALID, "k must be 2..4");
  CKR(cudaSetDevice(ctx->device));
  double *dx = nullptr, *dy = nullptr, *dout = nullptr;
  int rc = to_dev_planar(ctx, n, k, x_re, x_im, &dx);
  if (rc) return rc;
  rc = to_dev_planar(ctx, n, k, y_re, y_im, &dy);
  if (rc) return rc;
  const long long L = plane_ld(n);
  CKR(cudaMalloc(&dout, sizeof(double) * k * 2 * L + 16));
  rc = unit_axpy(k, x_im != nullptr, n, alpha_re, alpha_im, dx, dy, dout,
                 ctx->stream);
  if (rc) return fail(rc, "axpy failed");
  rc = from_dev_planar(ctx, n, k, dout, out_re, x_im ? out_im : nullptr);
  cudaFree(dx);
  cudaFree(dy);
  cudaFree(dout);
  return rc;
}

int mpk_mc_elementwise(mpk_ctx *ctx, int op, int k, int64_t n,
                       const double *a_re, const double *a_im,
                       const double *b_re, const double *b_im, double *o_re,
                       double *o_im) {
  if (k < 2 || k > 4) return fail(MPK_INVALID, "k must be 2..4");
  CKR(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int sa = (op == 7) ? 7 : k;
  double *d[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  const double *src[4] = {a_re, a_im, b_re, b_im};
  const size_t sz[4] = {(size_t)sa, (size_t)k, (size_t)k, (size_t)k};
  for (int q = 0; q < 4; ++q) {
    if (!src[q]) continue;
    CKR(cudaMalloc(&d[q], sizeof(double) * n * sz[q] + 8));
    CKR(cudaMemcpyAsync(d[q], src[q], sizeof(double) * n * sz[q],
                        cudaMemcpyHostToDevice, st));
  }
  CKR(cudaMalloc(&d[4], sizeof(double) * n * k + 8));
  if (o_im) CKR(cudaMalloc(&d[5], sizeof(double) * n * k + 8));
  int rc = unit_mc(op, k, d[0], d[1], d[2], d[3], d[4], d[5], (int)n, st);
  if (rc) return fail(rc, "bad op");
  CKR(cudaGetLastError());
  CKR(cudaMemcpyAsync(o_re, d[4], sizeof(double) * n * k, cudaMemcpyDeviceToHost, st));
  if (o_im)
    CKR(cudaMemcpyAsync(o_im, d[5], sizeof(double) * n * k, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  for (int q = 0; q < 6; ++q)
    if (d[q]) cudaFree(d[q]);
  return MPK_OK;
}

int mpk_mc_host(int op, int k, const double *a_re, const double *a_im,
                const double *b_re, const double *b_im, double *o_re,
                double *o_im) {
  int rc = host_mc(op, k, a_re, a_im, b_re, b_im, o_re, o_im);
  return rc ? fail(rc, "unsupported op/k") : MPK_OK;
}

static void fill_report(mpk_report *rep, const SolveOut &o, float factor_ms) {
  rep->iterations = o.iterations;
  rep->converged = o.converged;
  rep->breakdown = o.breakdown;
  rep->has_x = o.breakdown != kBdNumericSweep;
  rep->final_recursive_relres = o.relres;
  rep->true_relres = o.true_relres;
  rep->hist_len = o.hist_len;
  rep->factor_ms = factor_ms;
  rep->solve_ms = o.loop_ms;
}

int mpk_bench_apply(mpk_matrix *m, int k, int reps, double *ms_avg) {
  DMat &A = m->A;
  if (!A.factored) return fail(MPK_INVALID, "matrix is not factored");
  if (k < 1 || k > 4 || reps < 1) return fail(MPK_INVALID, "bad k/reps");
  CKR(cudaSetDevice(m->ctx->device));
  cudaStream_t st = m->ctx->stream;
  const long long L = plane_ld(A.n);
  double *din = nullptr, *dz = nullptr;
  const size_t planes = (size_t)k * (A.cx ? 2 : 1);
  CKR(cudaMalloc(&din, sizeof(double) * planes * L));
  CKR(cudaMalloc(&dz, sizeof(double) * 2 * L));
  // input: the matrix values reused as a deterministic right-hand side head
  CKR(cudaMemsetAsync(din, 0, sizeof(double) * planes * L, st));
  CKR(cudaMemcpyAsync(din, A.val, sizeof(double) * (A.n < A.nnz ? A.n : A.nnz),
                      cudaMemcpyDeviceToDevice, st));
  SweepArgs a{};
  a.n = A.n;
  a.rp = A.rp;
  a.ci = A.ci;
  a.dp = A.dp;
  a.lu = A.lu;
  a.ord_f = A.ord_f;
  a.ord_b = A.ord_b;
  a.lev_f = A.lev_f;
  a.lev_b = A.lev_b;
  a.nlev_f = A.levels_f;
  a.nlev_b = A.levels_b;
  a.in_re = din;
  a.in_im = A.cx ? din + (long long)k * L : nullptr;
  a.y = A.sw_y;
  a.z = dz;
  a.tick = A.tick;
  a.err = A.err;
  a.done = nullptr;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double tot = 0.0;
  for (int r = 0; r < reps; ++r) {
    launch_sweep_reset(A.sw_y, dz, A.n, A.cx, nullptr, st);
    cudaEventRecord(e0, st);
    do_sweep(A, a, false, st);
    cudaEventRecord(e1, st);
    CKR(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    tot += ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(din);
  cudaFree(dz);
  CKR(cudaGetLastError());
  *ms_avg = tot / reps;
  return MPK_OK;
}

int mpk_sweep_info(mpk_matrix *m, int64_t *info, int ninfo) {
  if (!m || !info || ninfo < 1) return fail(MPK_INVALID, "bad arguments");
  const DMat &A = m->A;
  const SweepMats &S = A.smat;
  int64_t v[12] = {0};
  v[0] = A.levels_f;
  v[1] = A.levels_b;
  v[2] = S.ss.on ? 5 : S.wf.on ? 4 : S.rs.nchunks > 0 ? 3 : S.cs.C > 0 ? 2 : A.smat_built ? 1 : 0;
  if (S.ss.on) {
    v[3] = S.ss.f.Lc;
    v[4] = S.ss.f.lag;
    v[5] = S.ss.f.ngroups;
    v[6] = S.ss.f.S;
    v[7] = S.ss.b.lag;
    v[8] = S.ss.b.S;
    v[9] = S.ss.W;
    v[10] = S.ss.f.chunkb;
    v[11] = S.ss.f.cl;
  }
  for (int i = 0; i < ninfo && i < 12; ++i) info[i] = v[i];
  return MPK_OK;
}

int mpk_bench_spmv(mpk_matrix *m, int k, int reps, double *ms_avg) {
  DMat &A = m->A;
  if (k < 2 || k > 4 || reps < 1) return fail(MPK_INVALID, "bad k/reps");
  CKR(cudaSetDevice(m->ctx->device));
  cudaStream_t st = m->ctx->stream;
  const long long L = plane_ld(A.n);
  const size_t c = A.cx ? 2 : 1;
  double *dx = nullptr, *dy = nullptr;
  // x: an F vector (binary64 head, the output of an ILU(0)-mixed apply, as
  // in BiCGSTAB/CGS/GPBiCG); y: a k-component planar MC vector
  CKR(cudaMalloc(&dx, sizeof(double) * c * L));
  CKR(cudaMalloc(&dy, sizeof(double) * c * k * L));
  CKR(cudaMemsetAsync(dx, 0, sizeof(double) * c * L, st));
  CKR(cudaMemcpyAsync(dx, A.val, sizeof(double) * (A.n < A.nnz ? A.n : A.nnz),
                      cudaMemcpyDeviceToDevice, st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double tot = 0.0;
  int rc = 0;
  for (int r = 0; r < reps && rc == 0; ++r) {
    cudaEventRecord(e0, st);
    rc = unit_spmv(A, k, false, true, dx, dy, st);
    cudaEventRecord(e1, st);
    CKR(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    tot += ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(dx);
  cudaFree(dy);
  CKR(cudaGetLastError());
  if (rc) return fail(MPK_INVALID, "spmv dispatch");
  *ms_avg = tot / reps;
  return MPK_OK;
}

static int solve_core(mpk_matrix *m, int method, int k, double eps_rel,
                      double eps_abs, int64_t max_iter, const double *d_b,
                      double *d_x, double *d_hist, int64_t hist_cap,
                      mpk_report *rep, Exchange *ex = nullptr) {
  std::memset(rep, 0, sizeof(*rep));
  rep->final_recursive_relres = NAN;
  rep->true_relres = NAN;
  if (method < 0 || method > 3) return fail(MPK_INVALID, "unknown method");
  if (k < 2 || k > 4)
    return fail(MPK_INVALID, "mixed SpMV needs a working precision above binary64");
  if (!(eps_rel > 0) || !(eps_abs > 0))
    return fail(MPK_INVALID, "eps_rel and eps_abs must be positive");
  // build_preconditioner (ilu.py:514-522) inside the timed solve, as the
  // reference's total_seconds includes the factorization (solvers.py:426)
  int64_t bad = -1;
  int32_t structural = 0;
  tl_phase[0] = host_ms();
  const int pre = tl_precond >= 0 ? tl_precond : m->ctx->precond;
  const bool ilu = pre != MPK_PRECOND_NONE;
  if (pre != MPK_PRECOND_ILU0_MIXED && ex)
    return fail(MPK_INVALID, "sharded solve: ILU(0)-mixed only");
  int rc = MPK_OK;
  if (pre == MPK_PRECOND_ILU0_MIXED)
    rc = mpk_ilu0_factor(m, &bad, &structural);
  else if (pre == MPK_PRECOND_ILU0_FULL)
    rc = mpk_ilu0_factor_full(m, k, &bad, &structural);
  if (!ilu) m->factor_ms = 0.f;  // M = I: no factors
  tl_phase[1] = host_ms();
  if (rc == MPK_SINGULAR_PIVOT || rc == MPK_NUMERIC_BREAKDOWN) {
    rep->iterations = 0;
    rep->converged = 0;
    rep->breakdown = rc == MPK_SINGULAR_PIVOT ? MPK_BD_SINGULAR_PIVOT
                                              : MPK_BD_NUMERIC_FACTOR;
    rep->bad_row = bad;
    rep->structural = structural;
    rep->has_x = 0;
    rep->factor_ms = m->factor_ms;
    return MPK_OK;
  }
  if (rc) return rc;
  SolveParams p{};
  p.method = method;
  p.k = k;
  p.eps_rel = eps_rel;
  p.eps_abs = eps_abs;
  p.max_iter = max_iter < 0 ? 3LL * m->A.n : max_iter;
  p.precond_ilu = pre == MPK_PRECOND_ILU0_FULL ? 2 : (ilu ? 1 : 0);
  p.hist_cap = hist_cap;
  p.reduce_seq = m->ctx->reduce_seq;
  p.ex = ex;
  p.full_a = (tl_spmv_full && m->A.mcv) ? 1 : 0;
  if (p.full_a && m->A.mcv_k != k)
    return fail(MPK_INVALID, "matrix and vector precision must match for spmv");
  if (p.full_a && ex) return fail(MPK_INVALID, "sharded solve: binary64-valued matrices only");
  SolveOut o{};
  char eb[256] = {0};
  rc = run_solve(m->A, p, d_b, d_x, d_hist, &o, m->ctx->stream, eb);
  if (rc) return fail(rc, eb);
  fill_report(rep, o, m->factor_ms);
  return MPK_OK;
}

int mpk_solve_dev(mpk_matrix *m, int method, int k, double eps_rel,
                  double eps_abs, int64_t max_iter, const double *b_dev,
                  double *x_dev, double *hist_dev, int64_t hist_cap,
                  mpk_report *rep) {
  const auto t0 = std::chrono::steady_clock::now();
  const long long l0 = tl_launches;
  CKR(cudaSetDevice(m->ctx->device));
  int rc = solve_core(m, method, k, eps_rel, eps_abs, max_iter, b_dev, x_dev,
                      hist_dev, hist_cap, rep);
  rep->total_ms = std::chrono::duration<double, std::milli>(
                      std::chrono::steady_clock::now() - t0)
                      .count();
  rep->launches = tl_launches - l0;
  static const bool phases = getenv("MPK_PHASE_TIMES") != nullptr;
  if (phases)
    fprintf(stderr,
            "[mpk] factor %.3f | setup+capture %.3f | loop %.3f | finish %.3f | "
            "tail %.3f ms\n",
            tl_phase[1] - tl_phase[0], tl_phase[2] - tl_phase[1],
            tl_phase[3] - tl_phase[2], tl_phase[4] - tl_phase[3],
            host_ms() - tl_phase[4]);
  return rc;
}

// ---- row-block sharded solve (shard.cuh) ----
struct mpk_comm {
  Exchange *ex = nullptr;
};

int mpk_comm_unique_id(void *id128) {
  char eb[256] = {0};
  if (nccl_unique_id(id128, eb)) return fail(MPK_CUDA_ERROR, eb);
  return MPK_OK;
}

int mpk_comm_create(int device, int rank, int world, const void *id128,
                    mpk_comm **out) {
  if (world < 1 || rank < 0 || rank >= world || !out)
    return fail(MPK_INVALID, "bad rank / world");
  char eb[256] = {0};
  Exchange *ex = make_nccl_exchange(device, rank, world, id128, eb);
  if (!ex) return fail(MPK_CUDA_ERROR, eb);
  *out = new mpk_comm{ex};
  return MPK_OK;
}

int mpk_comm_create_local(int world, mpk_comm **out) {
  if (world < 1 || !out) return fail(MPK_INVALID, "bad world");
  std::vector<Exchange *> ex(world);
  if (make_local_exchanges(world, ex.data())) return fail(MPK_CUDA_ERROR, "events");
  for (int r = 0; r < world; ++r) out[r] = new mpk_comm{ex[r]};
  return MPK_OK;
}

void mpk_comm_destroy(mpk_comm *c) {
  if (!c) return;
  delete c->ex;
  delete c;
}

int mpk_comm_rank(const mpk_comm *c) { return c ? c->ex->rank : -1; }
int mpk_comm_world(const mpk_comm *c) { return c ? c->ex->world : -1; }

int mpk_solve_dev_sharded(mpk_matrix *m, mpk_comm *comm, int method, int k,
                          double eps_rel, double eps_abs, int64_t max_iter,
                          const double *b_dev, double *x_dev, double *hist_dev,
                          int64_t hist_cap, mpk_report *rep) {
  if (!comm) return fail(MPK_INVALID, "null communicator");
  if (method != MPK_BICGSTAB)
    return fail(MPK_INVALID, "sharded solve: BiCGSTAB only");
  if (m->ctx->reduce_seq)
    return fail(MPK_INVALID, "sharded solve: tree reductions only");
  const auto t0 = std::chrono::steady_clock::now();
  const long long l0 = tl_launches;
  CKR(cudaSetDevice(m->ctx->device));
  int rc = solve_core(m, method, k, eps_rel, eps_abs, max_iter, b_dev, x_dev,
                      hist_dev, hist_cap, rep, comm->ex);
  rep->total_ms = std::chrono::duration<double, std::milli>(
                      std::chrono::steady_clock::now() - t0)
                      .count();
  rep->launches = tl_launches - l0;
  return rc;
}

int mpk_solve(mpk_matrix *m, int method, int k, double eps_rel,
              double eps_abs, int64_t max_iter, const double *b_re,
              const double *b_im, double *x_re, double *x_im, double *hist,
              int64_t hist_cap, mpk_report *rep) {
  const auto t0 = std::chrono::steady_clock::now();
  const long long l0 = tl_launches;
  DMat &A = m->A;
  if (A.cx != (b_im != nullptr))
    return fail(MPK_INVALID, "matrix/vector field mismatch");
  if (k < 2 || k > 4)
    return fail(MPK_INVALID, "mixed SpMV needs a working precision above binary64");
  CKR(cudaSetDevice(m->ctx->device));
  cudaStream_t st = m->ctx->stream;
  const long long n = A.n, L = plane_ld(A.n);
  const int c = A.cx ? 2 : 1;
  IoBufs &B = m->io[k];
  if (!B.b) {
    CKR(cudaMalloc(&B.b, sizeof(double) * k * c * L + 16));
    CKR(cudaMalloc(&B.x, sizeof(double) * k * c * L + 16));
    CKR(cudaMalloc(&B.stage, sizeof(double) * k * c * (n ? n : 1)));
  }
  const int64_t hc = hist && hist_cap > 0 ? hist_cap : 0;
  if (hc > B.hist_cap) {
    if (B.hist) cudaFree(B.hist);
    CKR(cudaMalloc(&B.hist, sizeof(double) * k * hc));
    B.hist_cap = hc;
  }
  // H2D of b (the caller's buffer, pinned for full bandwidth) -> planar
  CKR(cudaMemsetAsync(B.b, 0, sizeof(double) * k * c * L, st));
  CKR(cudaMemsetAsync(B.x, 0, sizeof(double) * k * c * L, st));
  if (n > 0) {
    CKR(cudaMemcpyAsync(B.stage, b_re, sizeof(double) * n * k,
                        cudaMemcpyHostToDevice, st));
    if (A.cx)
      CKR(cudaMemcpyAsync(B.stage + n * k, b_im, sizeof(double) * n * k,
                          cudaMemcpyHostToDevice, st));
    launch_to_planar(n, k, B.stage, A.cx ? B.stage + n * k : nullptr, B.b, st);
  }
  int rc = solve_core(m, method, k, eps_rel, eps_abs, max_iter, B.b, B.x,
                      hc ? B.hist : nullptr, hc, rep);
  if (rc == MPK_OK && rep->has_x && n > 0) {
    launch_from_planar(n, k, B.x, B.stage, A.cx ? B.stage + n * k : nullptr, st);
    CKR(cudaMemcpyAsync(x_re, B.stage, sizeof(double) * n * k,
                        cudaMemcpyDeviceToHost, st));
    if (A.cx)
      CKR(cudaMemcpyAsync(x_im, B.stage + n * k, sizeof(double) * n * k,
                          cudaMemcpyDeviceToHost, st));
  }
  if (rc == MPK_OK && hc) {
    const int64_t cnt = rep->hist_len < hc ? rep->hist_len : hc;
    if (cnt > 0)
      CKR(cudaMemcpyAsync(hist, B.hist, sizeof(double) * k * cnt,
                          cudaMemcpyDeviceToHost, st));
  }
  CKR(cudaStreamSynchronize(st));
  rep->total_ms = std::chrono::duration<double, std::milli>(
                      std::chrono::steady_clock::now() - t0)
                      .count();
  rep->launches = tl_launches - l0;
  return rc;
}

int mpk_csr_set_values(mpk_matrix *m, const double *val_re,
                       const double *val_im) {
  DMat &A = m->A;
  if (A.cx != (val_im != nullptr))
    return fail(MPK_INVALID, "field mismatch: matrix/values");
  CKR(cudaSetDevice(m->ctx->device));
  cudaStream_t st = m->ctx->stream;
  if (A.nnz > 0) {
    if (!A.cx) {
      CKR(cudaMemcpyAsync(A.val, val_re, sizeof(double) * A.nnz,
                          cudaMemcpyHostToDevice, st));
    } else {
      m->h_vals.resize(2 * A.nnz);
      for (long long p = 0; p < A.nnz; ++p) {
        m->h_vals[2 * p] = val_re[p];
        m->h_vals[2 * p + 1] = val_im[p];
      }
      CKR(cudaMemcpyAsync(A.val, m->h_vals.data(), sizeof(double) * 2 * A.nnz,
                          cudaMemcpyHostToDevice, st));
    }
    if (A.at_rp) gather(A.val, A.at_perm, A.at_val, A.nnz, A.cx, st);
  }
  A.factored = false;
  A.adj_ready = false;
  CKR(cudaStreamSynchronize(st));
  return MPK_OK;
}

// CsrMatrix values at working precision (sparse.py:192-249 val_re / val_im,
// shape (nnz, k) row-major): attaches all k components of every entry for
// spmv_mode 'full' (mpk_spmv_full, MPK_OPT_SPMV) and for the
// working-precision ILU(0); k = 0 detaches them.  The binary64 heads
// uploaded by mpk_csr_upload / mpk_csr_set_values stay the demoted matrix.
int mpk_csr_set_mc_values(mpk_matrix *m, int k, const double *val_re,
                          const double *val_im) {
  DMat &A = m->A;
  CKR(cudaSetDevice(m->ctx->device));
  if (A.mcv) {
    CKR(cudaStreamSynchronize(m->ctx->stream));
    cudaFree(A.mcv);
    A.mcv = nullptr;
    A.mcv_k = 0;
    A.mc_factored = false;
  }
  if (k == 0) return MPK_OK;
  if (k < 2 || k > 4) return fail(MPK_INVALID, "MC matrix values: k = 2..4");
  if (!val_re || A.cx != (val_im != nullptr))
    return fail(MPK_INVALID, "field mismatch: matrix/values");
  int rc = to_dev_planar(m->ctx, A.nnz, k, val_re, val_im, &A.mcv);
  if (rc) return rc;
  A.mcv_k = k;
  A.mcv_ld = plane_ld(A.nnz);
  return MPK_OK;
}

// spmv / spmv_adjoint (sparse.py:414-451): y = A x or A^H x with the matrix
// at working precision; binary64-valued matrices (no MC values attached)
// take the mixed kernels, which compute the same thing bit for bit
int mpk_spmv_full(mpk_matrix *m, int k, const double *x_re, const double *x_im,
                  double *y_re, double *y_im, int adjoint) {
  DMat &A = m->A;
  if (!A.mcv) return mpk_spmv_mixed(m, k, x_re, x_im, y_re, y_im, adjoint);
  if (A.mcv_k != k)
    return fail(MPK_INVALID, "matrix and vector precision must match for spmv");
  if (A.cx != (x_im != nullptr))
    return fail(MPK_INVALID, std::string("field mismatch: matrix ") +
                                 (A.cx ? "complex" : "real") + ", vector " +
                                 (x_im ? "complex" : "real"));
  CKR(cudaSetDevice(m->ctx->device));
  cudaStream_t st = m->ctx->stream;
  double *dx = nullptr, *dy = nullptr;
  int rc = to_dev_planar(m->ctx, A.n, k, x_re, x_im, &dx);
  if (rc) return rc;
  const long long L = plane_ld(A.n);
  CKR(cudaMalloc(&dy, sizeof(double) * k * 2 * L + 16));
  rc = unit_spmv_full(A, k, adjoint != 0, false, dx, dy, nullptr, st);
  if (rc) return fail(MPK_INVALID, "unsupported k");
  CKR(cudaGetLastError());
  rc = from_dev_planar(m->ctx, A.n, k, dy, y_re, A.cx ? y_im : nullptr);
  cudaFree(dx);
  cudaFree(dy);
  return rc;
}

int mpk_solve_batch(int nsys, mpk_matrix **ms, int method, int k,
                    double eps_rel, double eps_abs, int64_t max_iter,
                    const double *const *b_re, double *const *x_re,
                    mpk_report *reps) {
  if (nsys <= 0) return MPK_OK;
  // one host thread + stream per lane; systems dealt round-robin
  const int lanes = nsys < 8 ? nsys : 8;
  std::vector<int> rcs(lanes, 0);
  std::vector<std::string> errs(lanes);
  std::vector<std::thread> th;
  for (int l = 0; l < lanes; ++l) {
    th.emplace_back([&, l]() {
      for (int s = l; s < nsys; s += lanes) {
        int rc = mpk_solve(ms[s], method, k, eps_rel, eps_abs, max_iter,
                           b_re[s], nullptr, x_re[s], nullptr, nullptr, 0,
                           &reps[s]);
        if (rc) {
          rcs[l] = rc;
          errs[l] = g_err;
        }
      }
    });
  }
  for (auto &t : th) t.join();
  for (int l = 0; l < lanes; ++l)
    if (rcs[l]) return fail(rcs[l], errs[l]);
  return MPK_OK;
}

}  // extern "C"

extern "C" int mpk_run_jobs(mpk_job *jobs, int njobs, int device_resident) {
  if (njobs <= 0) return MPK_OK;
  auto run = [&](int j) {
    mpk_job &J = jobs[j];
    int rc = MPK_OK;
    if (!device_resident && J.val_re)
      rc = mpk_csr_set_values(J.m, J.val_re, J.val_im);
    if (rc == MPK_OK) {
      if (device_resident)
        rc = mpk_solve_dev(J.m, J.method, J.k, J.eps_rel, J.eps_abs, J.max_iter,
                           J.b_re, J.x_re, J.hist, J.hist_cap, &J.rep);
      else
        rc = mpk_solve(J.m, J.method, J.k, J.eps_rel, J.eps_abs, J.max_iter,
                       J.b_re, J.b_im, J.x_re, J.x_im, J.hist, J.hist_cap,
                       &J.rep);
    }
    J.rc = rc;
  };
  if (njobs == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    th.reserve(njobs);
    for (int j = 0; j < njobs; ++j) th.emplace_back(run, j);
    for (auto &t : th) t.join();
  }
  for (int j = 0; j < njobs; ++j)
    if (jobs[j].rc) return jobs[j].rc;
  return MPK_OK;
}
