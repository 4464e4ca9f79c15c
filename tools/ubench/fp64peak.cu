// FP64 pipe peak on this GPU ("measure it first"): every SM
// fully occupied, 8 independent chains per thread of DFMA (2 flop), DADD or
// DMUL (1 flop); CUDA events around the kernel, best of 5.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64peak.cu -o fp64peak
#include <cstdio>
template <int OP>
__global__ void __launch_bounds__(256) k(double *o, double a, double b, int n) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) acc[i] = fma(acc[i], a, b);
      if (OP == 1) acc[i] = __dadd_rn(acc[i], b);
      if (OP == 2) acc[i] = __dmul_rn(acc[i], a);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1234.5) o[0] = s;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *o;
  cudaMalloc(&o, 8);
  const int n = 1 << 14, blocks = sms * 8, th = 256;
  const char *nm[] = {"DFMA", "DADD", "DMUL"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int op = 0; op < 3; ++op) {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      if (op == 0) k<0><<<blocks, th>>>(o, 0.999999, 1e-9, n);
      if (op == 1) k<1><<<blocks, th>>>(o, 0.999999, 1e-9, n);
      if (op == 2) k<2><<<blocks, th>>>(o, 0.999999, 1e-9, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    const double ops = (double)blocks * th * 8 * n;
    const double fl = ops * (op == 0 ? 2 : 1);
    printf("%s: %.1f G inst/s, %.2f TFLOP/s (%d SMs)\n", nm[op], ops / best / 1e6,
           fl / best / 1e9, sms);
  }
  return 0;
}
