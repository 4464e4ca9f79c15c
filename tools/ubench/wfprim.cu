// Latencies of the primitives on the wavefront sweep's per-step critical
// path (B200): dependent DADD / DMUL / DDIV, dependent LDS, STS -> __syncwarp
// -> LDS hand-off between lanes, __syncwarp alone, cp.async 8 B + wait_group 0,
// ld.relaxed.gpu L2 hit.  nvcc -gencode arch=compute_100a,code=sm_100a wfprim.cu
#include <cstdio>
__global__ void k_all(double *o, const double *g, long long *cyc, int n) {
  __shared__ double sm[64 * 32];
  __shared__ int si[64];
  const int j = threadIdx.x;
  double x = 1.0000001 + j, a = 1.0000001;
  long long t0, t1;
  // DADD
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
  t1 = clock64(); if (j == 0) cyc[0] = t1 - t0;
  // DMUL
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, a);
  t1 = clock64(); if (j == 0) cyc[1] = t1 - t0;
  // DDIV
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __ddiv_rn(x, a);
  t1 = clock64(); if (j == 0) cyc[2] = t1 - t0;
  // dependent LDS chain
  if (j < 64) si[j] = (j + 1) & 63;
  __syncwarp();
  int q = j & 63;
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = si[q];
  t1 = clock64(); if (j == 0) cyc[3] = t1 - t0;
  // __syncwarp alone
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncwarp();
  t1 = clock64(); if (j == 0) cyc[4] = t1 - t0;
  // hand-off: lane j reads lane j-1's value of the previous step
  double v = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    sm[(i & 63) * 32 + j] = v;
    __syncwarp();
    v = __dadd_rn(sm[(i & 63) * 32 + ((j + 31) & 31)], a);
  }
  t1 = clock64(); if (j == 0) cyc[5] = t1 - t0;
  // shuffle hand-off
  t0 = clock64();
  for (int i = 0; i < n; ++i) v = __dadd_rn(__shfl_up_sync(0xffffffffu, v, 1), a);
  t1 = clock64(); if (j == 0) cyc[6] = t1 - t0;
  // cp.async 8 B + wait 0 (L2 / L1)
  t0 = clock64();
  for (int i = 0; i < n / 16; ++i) {
    unsigned d = (unsigned)__cvta_generic_to_shared(&sm[j]);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(g + ((i * 97) & 4095) * 32 + j) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    v += sm[j];
  }
  t1 = clock64(); if (j == 0) cyc[7] = (t1 - t0) * 16;
  // ld.relaxed.gpu dependent chain (L2 hit)
  const double *pp = g;
  t0 = clock64();
  for (int i = 0; i < n / 16; ++i) {
    double w;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(w) : "l"(pp));
    pp = g + (((long long)w) & 4095) * 32;
    v += w;
  }
  t1 = clock64(); if (j == 0) cyc[8] = (t1 - t0) * 16;
  o[j] = x + v;
}
int main() {
  double *o, *g; long long *c;
  cudaMalloc(&o, 8 * 32); cudaMalloc(&c, 8 * 16); cudaMalloc(&g, 8 * 4096 * 32);
  double *h = new double[4096 * 32];
  for (int i = 0; i < 4096 * 32; ++i) h[i] = (double)((i * 7 + 3) % 4096);
  cudaMemcpy(g, h, 8 * 4096 * 32, cudaMemcpyHostToDevice);
  const int n = 4096;
  long long cyc[16];
  const char *nm[] = {"DADD dep", "DMUL dep", "DDIV (__ddiv_rn) dep", "LDS dep chain",
                      "__syncwarp", "STS->syncwarp->LDS(lane-1)->DADD", "shfl_up->DADD",
                      "cp.async 8B + wait_group 0", "ld.relaxed.gpu dep (L2)"};
  for (int rep = 0; rep < 2; ++rep) {
    k_all<<<1, 32>>>(o, g, c, n);
    cudaMemcpy(cyc, c, 8 * 16, cudaMemcpyDeviceToHost);
  }
  for (int i = 0; i < 9; ++i) printf("%-36s %7.1f cycles\n", nm[i], (double)cyc[i] / n);
  return 0;
}
