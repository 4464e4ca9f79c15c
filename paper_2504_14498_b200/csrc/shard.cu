// shard.cu -- exchanges of the row-block sharded solve (see shard.cuh).
#include <dlfcn.h>

#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include <nccl.h>

#include "shard.cuh"

namespace mpk {

namespace {

struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*get_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allgather)(const void *, void *, size_t, ncclDataType_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char *(*errstr)(ncclResult_t) = nullptr;
  bool load(char *eb) {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(eb, 256, "libnccl.so.2 not loadable: %s", dlerror());
      return false;
    }
    get_id = (decltype(get_id))dlsym(h, "ncclGetUniqueId");
    init_rank = (decltype(init_rank))dlsym(h, "ncclCommInitRank");
    allgather = (decltype(allgather))dlsym(h, "ncclAllGather");
    destroy = (decltype(destroy))dlsym(h, "ncclCommDestroy");
    errstr = (decltype(errstr))dlsym(h, "ncclGetErrorString");
    if (!get_id || !init_rank || !allgather || !destroy) {
      snprintf(eb, 256, "libnccl.so.2 lacks the collective entry points");
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

struct NcclExchange : Exchange {
  ncclComm_t comm = nullptr;
  ~NcclExchange() override {
    if (comm) g_nccl.destroy(comm);
  }
  int allgather_inplace(double *buf, size_t count, cudaStream_t st) override {
    if (world == 1) return 0;
    const ncclResult_t r = g_nccl.allgather(buf + (size_t)rank * count, buf, count,
                                            ncclFloat64, comm, st);
    return r == ncclSuccess ? 0 : 4;
  }
  const char *kind() const override { return "nccl"; }
};

// generation barrier of the virtual ranks' host threads
struct LocalGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int count = 0;
  long long gen = 0;
  std::vector<double *> ptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  explicit LocalGroup(int w) : world(w), ptr(w), ev_in(w), ev_out(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++count == world) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  int refs = 0;
};

struct LocalExchange : Exchange {
  LocalGroup *g = nullptr;
  cudaEvent_t e_in = nullptr, e_out = nullptr;
  ~LocalExchange() override {
    if (e_in) cudaEventDestroy(e_in);
    if (e_out) cudaEventDestroy(e_out);
    bool last = false;
    {
      std::lock_guard<std::mutex> lk(g->m);
      last = --g->refs == 0;
    }
    if (last) delete g;
  }
  int allgather_inplace(double *buf, size_t count, cudaStream_t st) override {
    if (world == 1) return 0;
    // 1: every rank's own range is ready (event), pointers published
    g->ptr[rank] = buf;
    cudaEventRecord(e_in, st);
    g->ev_in[rank] = e_in;
    g->barrier();
    // 2: pull the peers' ranges, after their producers
    for (int q = 0; q < world; ++q) {
      if (q == rank) continue;
      cudaStreamWaitEvent(st, g->ev_in[q], 0);
      cudaMemcpyAsync(buf + (size_t)q * count, g->ptr[q] + (size_t)q * count,
                      sizeof(double) * count, cudaMemcpyDeviceToDevice, st);
    }
    // 3: nobody overwrites its range before every peer has copied it
    cudaEventRecord(e_out, st);
    g->ev_out[rank] = e_out;
    g->barrier();
    for (int q = 0; q < world; ++q)
      if (q != rank) cudaStreamWaitEvent(st, g->ev_out[q], 0);
    g->barrier();  // events / pointers may be reused by the next call
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
  }
  const char *kind() const override { return "local"; }
};

}  // namespace

int nccl_unique_id(void *id128, char *errbuf) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (!g_nccl.load(errbuf)) return 4;
  ncclUniqueId id;
  if (g_nccl.get_id(&id) != ncclSuccess) {
    snprintf(errbuf, 256, "ncclGetUniqueId failed");
    return 4;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(id128, &id, 128);
  return 0;
}

Exchange *make_nccl_exchange(int device, int rank, int world, const void *id128,
                             char *errbuf) {
  {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl.load(errbuf)) return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    snprintf(errbuf, 256, "cudaSetDevice(%d) failed", device);
    return nullptr;
  }
  auto *ex = new NcclExchange;
  ex->rank = rank;
  ex->world = world;
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  const ncclResult_t r = g_nccl.init_rank(&ex->comm, world, id, rank);
  if (r != ncclSuccess) {
    snprintf(errbuf, 256, "ncclCommInitRank failed: %s",
             g_nccl.errstr ? g_nccl.errstr(r) : "?");
    ex->comm = nullptr;
    delete ex;
    return nullptr;
  }
  return ex;
}

int make_local_exchanges(int world, Exchange **out) {
  auto *g = new LocalGroup(world);
  g->refs = world;
  for (int r = 0; r < world; ++r) {
    auto *ex = new LocalExchange;
    ex->rank = r;
    ex->world = world;
    ex->g = g;
    cudaEventCreateWithFlags(&ex->e_in, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ex->e_out, cudaEventDisableTiming);
    out[r] = ex;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace mpk
