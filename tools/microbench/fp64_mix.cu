// FP64 instruction throughput on sm_100a (DFMA / DADD / DMUL, and the sketch's 2:1 DFMA:DADD mix)
// and the calibration of ncu's sm__pipe_fp64_cycles_active for a pipe-saturating loop.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 8192
template <int OP>
__global__ void k(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = threadIdx.x + u;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) x[u] = fma(x[u], a, b);
      else if (OP == 1) x[u] = x[u] + b;
      else if (OP == 2) x[u] = x[u] * a;
      else { x[u] = fma(x[u], a, b); x[u] = fma(x[u], a, b); x[u] = x[u] - b; }
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += x[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 8);
  const char* names[] = {"DFMA", "DADD", "DMUL", "2 DFMA + 1 DADD"};
  for (int op = 0; op < 4; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (op == 0) k<0><<<148 * 8, 256>>>(o, 1.0000001, 1e-9);
      if (op == 1) k<1><<<148 * 8, 256>>>(o, 1.0000001, 1e-9);
      if (op == 2) k<2><<<148 * 8, 256>>>(o, 1.0000001, 1e-9);
      if (op == 3) k<3><<<148 * 8, 256>>>(o, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 148.0 * 8 * 256 * ITERS * 8 * (op == 3 ? 3 : 1);
      if (rep) printf("%-18s %.2f ms  %.2f T lane-ops/s  %.2f lane-ops/clk/SM (1.965 GHz)\n", names[op], ms,
                      ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
