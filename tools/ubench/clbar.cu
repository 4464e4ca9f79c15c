// Cluster barrier / DSMEM latency on B200 (cycles per iteration).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 clbar.cu -o clbar
#include <cstdio>
#include <cstdint>

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
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(rank));
  return o;
}

// mode 0: barrier.cluster arrive+wait; 1: __syncthreads; 2: dependent DSMEM
// load chain to rank (r+1)%C; 3: dependent local ld.shared chain via mapa;
// 4: arrive/wait with a remote store before
__global__ void k(int mode, int iters, long long *out) {
  __shared__ uint32_t buf[256];
  const uint32_t r = cl_rank();
  uint32_t C;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(C));
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = (i + 1) % 256;
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const uint32_t remote = cl_map(smem_u32(buf), (r + 1) % C);
  const uint32_t local = cl_map(smem_u32(buf), r);
  long long t0 = clock64();
  uint32_t j = 0;
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 1) {
      __syncthreads();
    } else if (mode == 2) {
      uint32_t v;
      asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(remote + j * 4) : "memory");
      j = v;
    } else if (mode == 3) {
      uint32_t v;
      asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(local + j * 4) : "memory");
      j = v;
    } else if (mode == 4) {
      asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote + (threadIdx.x % 256) * 4), "r"(j) : "memory");
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 5) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0 && r == 0) out[0] = (t1 - t0) / iters + (j == 12345 ? 1 : 0);
}

int main() {
  long long *d;
  cudaMalloc(&d, 8);
  const char *names[] = {"cluster barrier", "__syncthreads", "DSMEM ld chain (remote)",
                         "DSMEM ld chain (own, mapa)", "remote st + barrier", "barrier relaxed"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int C : {1, 2, 4, 8, 16}) {
      for (int T : {128, 256, 1024}) {
        if (mode >= 2 && mode <= 3 && T != 128) continue;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(mode == 2 || mode == 3 ? 32 : T);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchKernelEx(&cfg, k, mode, 1000, d);
        long long h = -1;
        cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-28s C=%2d T=%4d : %lld cyc  %s\n", names[mode], C, (int)cfg.blockDim.x, h,
               e ? cudaGetErrorString(e) : "");
      }
    }
  }
  return 0;
}
