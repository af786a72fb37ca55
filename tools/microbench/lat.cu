// Dependent-chain latencies on sm_100a (one warp): DFMA, DADD, FFMA, SHFL (double), LDS.64, sqrt, division.
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  sm[threadIdx.x] = threadIdx.x;
  __syncwarp();
  double x = threadIdx.x * 1e-3 + 1.0;
  float f = (float)x;
  long long t0, t1;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = fma(x, a, b); t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = x + b; t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) f = fmaf(f, (float)a, (float)b); t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 0.0 * i; t1 = clock64(); cyc[3] = t1 - t0;
  int idx = threadIdx.x;
  t0 = clock64(); for (int i = 0; i < N; ++i) idx = (int)sm[idx & 31]; t1 = clock64(); cyc[4] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = sqrt(x) + 1.0; t1 = clock64(); cyc[5] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = 3.0 / x + 0.5; t1 = clock64(); cyc[6] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = x * a; t1 = clock64(); cyc[7] = t1 - t0;
  out[threadIdx.x] = x + f + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 16 * 8);
  k<<<1, 32>>>(o, c, 1.0000001, 1e-9);
  k<<<1, 32>>>(o, c, 1.0000001, 1e-9);
  long long h[8]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "DADD", "FFMA", "SHFL.f64 (+DFMA)", "LDS (+cvt)", "sqrt f64 (+DADD)", "div f64 (+DADD)", "DMUL"};
  for (int i = 0; i < 8; ++i) printf("%-20s %.1f cycles per dependent op\n", nm[i], (double)h[i] / N);
}
