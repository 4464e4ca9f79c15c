// Single-thread latency of the MC scalar ops (cycles): first call (cold
// instruction cache) vs the average of the next 9 (warm).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17
//      -I../../paper_2504_14498_b200/csrc mclat.cu -o mclat
#include <cstdio>

#include "mc.cuh"

using namespace mpk;

template <int K, int OP>
__global__ void k_op(double *io, long long *cyc) {
  V<K> a, b;
  for (int i = 0; i < K; ++i) {
    a.c[i] = io[i];
    b.c[i] = io[8 + i];
  }
  long long t[11];
  for (int r = 0; r < 10; ++r) {
    t[r] = clock64();
    V<K> o;
    if (OP == 0) add<K>(a.c, b.c, o.c);
    if (OP == 1) mul<K>(a.c, b.c, o.c);
    if (OP == 2) o = div_v<K>(a, b);
    if (OP == 3) o = sqrt_v<K>(a);
    // feed back (keeps the chain dependent, values stay O(1))
    for (int i = 0; i < K; ++i) a.c[i] = (o.c[0] == 12345.0) ? o.c[i] : a.c[i];
    io[16 + r] = o.c[0];
  }
  t[10] = clock64();
  cyc[0] = t[1] - t[0];
  cyc[1] = (t[10] - t[1]) / 9;
}

template <int K, int OP>
void run(const char *name, double *io, long long *cyc) {
  k_op<K, OP><<<1, 1>>>(io, cyc);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  printf("k=%d %-5s cold %7lld cyc  warm %7lld cyc\n", K, name, h[0], h[1]);
}

template <int K>
void all(double *io, long long *cyc) {
  run<K, 0>("add", io, cyc);
  run<K, 1>("mul", io, cyc);
  run<K, 2>("div", io, cyc);
  run<K, 3>("sqrt", io, cyc);
}

int main() {
  double h[32] = {1.2345678901234567, 1e-17, 3e-34, -2e-50, 0, 0, 0, 0,
                  0.987654321, -3e-18, 1e-35, 7e-52};
  double *io;
  long long *cyc;
  cudaMalloc(&io, sizeof h);
  cudaMalloc(&cyc, 64);
  cudaMemcpy(io, h, sizeof h, cudaMemcpyHostToDevice);
  all<2>(io, cyc);
  all<3>(io, cyc);
  all<4>(io, cyc);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
