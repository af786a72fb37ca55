// DMMA.8x8x4 (mma.sync m8n8k4 f64) throughput on sm_100a vs independent accumulators per warp
// (ACC) and warps per SM: how much ILP / occupancy the BSR kernel needs to keep the FP64 pipe busy.
// Operands in registers (no memory traffic).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void k(double* out, int iters) {
  double c0[ACC], c1[ACC];
#pragma unroll
  for (int u = 0; u < ACC; ++u) c0[u] = c1[u] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < ACC; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[u]), "+d"(c1[u]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < ACC; ++u) s += c0[u] + c1[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC>
void run(int warps_per_sm) {
  double* o;
  cudaMalloc(&o, 148 * 2048 * 8);
  const int threads = 32 * warps_per_sm;
  const int iters = 20000 / ACC * 8;
  k<ACC><<<148, threads>>>(o, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ACC><<<148, threads>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * ACC * (double)iters * warps_per_sm * 148;
  printf("ACC %2d warps/SM %2d: %6.2f TFLOP/s\n", ACC, warps_per_sm, flops / ms / 1e9);
  cudaFree(o);
}

int main() {
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<1>(w); run<2>(w); run<4>(w); run<8>(w); run<16>(w);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
