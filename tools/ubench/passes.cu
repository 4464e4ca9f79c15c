// Distribution of renorm pass counts for MC add / mul on random normalised
// operands (how often the reference's strictness loop needs > 1 pass).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17
//      -DMPK_COUNT_PASSES -I../../paper_2504_14498_b200/csrc passes.cu -o passes
#include <cstdio>

#include "mc.cuh"

using namespace mpk;

__device__ double rnd(unsigned long long &s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

template <int K>
__device__ void mk(unsigned long long &s, double (&x)[K]) {
  double t[K];
  double sc = ldexp(1.0, (int)(rnd(s) * 20));
  for (int i = 0; i < K; ++i) {
    t[i] = rnd(s) * sc;
    sc = ldexp(sc, -53);
  }
  renorm<K, K>(t, x);
}

template <int K, int OP>
__global__ void k(int n) {
  unsigned long long s = 1234567ull + blockIdx.x * 7919ull + threadIdx.x * 104729ull;
  double x[K], y[K], o[K];
  mk<K>(s, x);
  for (int it = 0; it < n; ++it) {
    mk<K>(s, y);
    if (OP == 0) add<K>(x, y, o);
    if (OP == 1) mul<K>(x, y, o);
    if (OP == 2) mul_lf<K>(y[0], x, o);
    for (int i = 0; i < K; ++i) x[i] = o[i];
    if (!(x[0] < 1e100 && x[0] > -1e100)) mk<K>(s, x);
  }
}

template <int K, int OP>
void run(const char *nm) {
  unsigned long long z[20][8] = {};
  cudaMemcpyToSymbol(g_pass_hist, z, sizeof z);
  k<K, OP><<<64, 128>>>(200);
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(z, g_pass_hist, sizeof z);
  for (int m = 0; m < 20; ++m) {
    if (!z[m][0]) continue;
    printf("k=%d %-6s M=%2d calls %llu:", K, nm, m, z[m][0]);
    for (int p = 0; p < 8; ++p) printf(" %.4f", (double)z[m][p] / z[m][0]);
    printf("\n");
  }
}

int main() {
  run<2, 0>("add");
  run<2, 1>("mul");
  run<3, 0>("add");
  run<3, 1>("mul");
  run<4, 0>("add");
  run<4, 1>("mul");
  run<4, 2>("mul_lf");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
