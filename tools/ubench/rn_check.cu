// Bitwise check of the MC operations in csrc/mc.cuh against a frozen copy of
// the previous (golden-verified) implementation (mc_ref.cuh, namespace
// mpkref), over adversarial random operands.  Prints mismatch counts.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17
//      -I../../paper_2504_14498_b200/csrc rn_check.cu -o rn_check
#include <cstdio>

#include "mc.cuh"
#include "mc_ref.cuh"

__device__ unsigned long long rng(unsigned long long &s) {
  s ^= s << 13;
  s ^= s >> 7;
  s ^= s << 17;
  return s;
}
__device__ double urand(unsigned long long &s) {
  return (rng(s) >> 11) * (1.0 / 9007199254740992.0);
}

// operand generator: mode picks the distribution
template <int K>
__device__ void gen(unsigned long long &s, int mode, double (&x)[K]) {
  const int sh = (int)(rng(s) % 64) - 32;
  double sc = ldexp(1.0, sh);
  for (int i = 0; i < K; ++i) x[i] = 0.0;
  switch (mode) {
    case 0: {  // normalised expansion
      double t[K];
      for (int i = 0; i < K; ++i) {
        t[i] = (urand(s) * 2 - 1) * sc;
        sc = ldexp(sc, -53);
      }
      mpkref::renorm<K, K>(t, x);
      break;
    }
    case 1:  // arbitrary components (unsorted, overlapping)
      for (int i = 0; i < K; ++i) x[i] = (urand(s) * 2 - 1) * ldexp(1.0, (int)(rng(s) % 80) - 40);
      break;
    case 2: {  // zeros / negative zeros sprinkled
      for (int i = 0; i < K; ++i) {
        const int r = (int)(rng(s) % 4);
        x[i] = r == 0 ? 0.0 : r == 1 ? -0.0 : (urand(s) * 2 - 1) * ldexp(sc, -53 * i);
      }
      break;
    }
    case 3: {  // ties: components of equal magnitude, small integers
      for (int i = 0; i < K; ++i) x[i] = (double)((int)(rng(s) % 7) - 3) * ldexp(1.0, -(int)(rng(s) % 3));
      break;
    }
    case 4: {  // huge / tiny exponents (overflow and subnormal territory)
      for (int i = 0; i < K; ++i) {
        const int e = (rng(s) & 1) ? 990 + (int)(rng(s) % 33) : -1070 + (int)(rng(s) % 40);
        x[i] = (urand(s) * 2 - 1) * ldexp(1.0, e);
      }
      break;
    }
    default: {  // near-cancellation partner of a normalised value
      double t[K];
      for (int i = 0; i < K; ++i) {
        t[i] = (urand(s) * 2 - 1) * sc;
        sc = ldexp(sc, -52);
      }
      mpkref::renorm<K, K>(t, x);
    }
  }
}

__device__ bool same(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b) || (isnan(a) && isnan(b));
}

template <int K>
__global__ void check(unsigned long long seed, int iters, unsigned long long *bad) {
  unsigned long long s = seed + 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int it = 0; it < iters; ++it) {
    double x[K], y[K], o1[K], o2[K];
    const int mx = (int)(rng(s) % 6), my = (int)(rng(s) % 6);
    gen<K>(s, mx, x);
    gen<K>(s, my, y);
    if (my == 5 && mx != 1)
      for (int i = 0; i < K; ++i) y[i] = -x[i] * (1.0 + ldexp(1.0, -50 - (int)(rng(s) % 10)));
    auto cmp = [&](int op) {
      bool ok = true;
      for (int i = 0; i < K; ++i) ok = ok && same(o1[i], o2[i]);
      if (!ok) atomicAdd(&bad[op], 1ull);
    };
    mpk::add<K>(x, y, o1);
    mpkref::add<K>(x, y, o2);
    cmp(0);
    mpk::mul<K>(x, y, o1);
    mpkref::mul<K>(x, y, o2);
    cmp(1);
    mpk::mul_lf<K>(x[0], y, o1);
    mpkref::mul_lf<K>(x[0], y, o2);
    cmp(2);
    mpk::add2<K>(x, y[0], y[1], o1);
    mpkref::add2<K>(x, y[0], y[1], o2);
    cmp(3);
    if ((it & 7) == 0) {
      mpk::div<K>(x, y, o1);
      mpkref::div<K>(x, y, o2);
      cmp(4);
      mpk::sqrt_mc<K>(x, o1);
      mpkref::sqrt_mc<K>(x, o2);
      cmp(5);
    }
    {
      double t[7], t2[7];
      for (int i = 0; i < 7; ++i) t[i] = t2[i] = (i < K) ? x[i] : y[i % K] * ldexp(1.0, -20 * i);
      mpk::renorm<7, K>(t, o1);
      mpkref::renorm<7, K>(t2, o2);
      cmp(6);
    }
    atomicAdd(&bad[7], 1ull);
  }
}

template <int K>
void run(int blocks, int iters) {
  unsigned long long *d, h[8];
  cudaMalloc(&d, sizeof h);
  cudaMemset(d, 0, sizeof h);
  check<K><<<blocks, 128>>>(1234567ull + K, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("k=%d cases %llu mismatches: add %llu mul %llu mul_lf %llu add2 %llu div %llu sqrt %llu renorm7 %llu  %s\n",
         K, h[7], h[0], h[1], h[2], h[3], h[4], h[5], h[6], cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<2>(592, 400);
  run<3>(592, 300);
  run<4>(592, 200);
  return 0;
}
