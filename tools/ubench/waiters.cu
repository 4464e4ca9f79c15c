// Does a warp waiting in an mbarrier try_wait loop (or a nanosleep/LDS
// poll loop) slow down a working warp of the same CTA?  Warp 0 runs a
// dependent FP64 + shuffle chain; warps 1..W-1 wait (mode 0: __syncthreads,
// 1: mbarrier try_wait loop, 2: nanosleep+LDS poll, 3: LDS spin) until warp
// 0 sets a flag.  Prints warp 0's cycles per iteration.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int mode, int iters, double *out, long long *cyc) {
  __shared__ uint64_t bar;
  __shared__ volatile int flag;
  const int w = threadIdx.x >> 5, j = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    flag = 0;
  }
  __syncthreads();
  if (w == 0) {
    double x = 1.0 + j * 1e-3, y = 0.5;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      x = __dsub_rn(x, __dmul_rn(y, x));
      x = __dadd_rn(x, 1.0);
      x = __shfl_sync(0xffffffffu, x, (j + 31) & 31);
    }
    long long t1 = clock64();
    if (j == 0) { cyc[0] = t1 - t0; flag = 1; asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory"); }
    out[threadIdx.x] = x;
  } else if (mode == 1) {
    asm volatile("{\n .reg .pred p;\nW%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W%=;\n}\n" ::"r"(su32(&bar)) : "memory");
  } else if (mode == 2) {
    while (!flag) __nanosleep(64);
  } else if (mode == 3) {
    while (!flag) {}
  }
  __syncthreads();
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
  const char *names[] = {"syncthreads", "mbarrier try_wait", "nanosleep poll", "LDS spin"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode)
      for (int W : {1, 2, 3, 4, 8}) {
        k<<<1, 32 * W>>>(mode, 20000, o, c);
        long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("%-18s W=%d: %.1f cycles/iter\n", names[mode], W, cy / 20000.0);
      }
  return 0;
}
