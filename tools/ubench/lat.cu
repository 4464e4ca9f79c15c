// Micro-benchmarks of the latencies that bound the latency-bound kernels:
// dependent DADD / DMUL / DFMA chains, L2-hit global load chain,
// __syncthreads, volatile load round trip.  nvcc -arch=sm_100a lat.cu
#include <cstdio>
__global__ void k_dadd(double *o, double a, int n, long long *cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  o[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_dmul(double *o, double a, int n, long long *cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, a);
  long long t1 = clock64();
  o[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_chase(const int *p, int n, int *o, long long *cyc) {
  int j = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = __ldcg(p + j);
  long long t1 = clock64();
  o[0] = j; cyc[0] = t1 - t0;
}
__global__ void k_sync(int n, long long *cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *o; long long *c; int *p, *oi;
  cudaMalloc(&o, 8); cudaMalloc(&c, 8); cudaMalloc(&oi, 4);
  const int N = 1 << 20;  // 4 MB ring (L2 resident), stride 1024 ints
  int *h = new int[N];
  for (int i = 0; i < N; ++i) h[i] = (i + 4099) % N;
  cudaMalloc(&p, N * 4); cudaMemcpy(p, h, N * 4, cudaMemcpyHostToDevice);
  long long cyc; const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    k_dadd<<<1, 1>>>(o, 1.0000001, n, c); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("DADD dependent latency: %.1f cycles\n", (double)cyc / n);
    k_dmul<<<1, 1>>>(o, 1.0000001, n, c); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("DMUL dependent latency: %.1f cycles\n", (double)cyc / n);
    k_chase<<<1, 1>>>(p, 2000, oi, c); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("L2-hit dependent load (ld.cg): %.1f cycles\n", cyc / 2000.0);
    for (int th : {128, 512, 1024}) {
      k_sync<<<1, th>>>(1000, c); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("__syncthreads (%d thr): %.1f cycles\n", th, cyc / 1000.0);
    }
  }
  return 0;
}
