// Stage timing of one renorm inside mul<4> / add<4> (warm, single thread).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17
//      -DMPK_RENORM_TIMING -I../../paper_2504_14498_b200/csrc rtime.cu -o rtime
#include <cstdio>
#include "mc.cuh"
using namespace mpk;
template <int OP>
__global__ void k(double *io, long long *out) {
  double a[4], b[4], o[4];
  for (int i = 0; i < 4; ++i) { a[i] = io[i]; b[i] = io[8 + i]; }
  long long t0 = 0, t1 = 0;
  for (int r = 0; r < 6; ++r) {
    t0 = clock64();
    if (OP == 0) add<4>(a, b, o); else mul<4>(a, b, o);
    t1 = clock64();
    for (int i = 0; i < 4; ++i) a[i] = (o[0] == 12345.0) ? o[i] : a[i];
    io[16 + r] = o[0];
  }
  out[0] = t1 - t0;
  for (int i = 0; i < 7; ++i) out[1 + i] = g_rt[i] - t0;
}
int main() {
  double h[32] = {1.2345678901234567, 1e-17, 3e-34, -2e-50, 0, 0, 0, 0,
                  0.987654321, -3e-18, 1e-35, 7e-52};
  double *io; long long *d;
  cudaMalloc(&io, sizeof h); cudaMalloc(&d, 64 * 8);
  cudaMemcpy(io, h, sizeof h, cudaMemcpyHostToDevice);
  for (int op = 0; op < 2; ++op) {
    if (op == 0) k<0><<<1, 1>>>(io, d); else k<1><<<1, 1>>>(io, d);
    long long r[8];
    cudaMemcpy(r, d, sizeof r, cudaMemcpyDeviceToHost);
    printf("%s total %lld | renorm start %lld, passes start %lld, sweep1 done %lld, sweep2 done %lld, check done %lld, passes end %lld, compaction end %lld\n",
           op ? "mul<4>" : "add<4>", r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7]);
  }
  return 0;
}
