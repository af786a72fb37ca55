// Throughput of the exp-kernel entry evaluation chain alone (no MMA): entries/s and FP64 ops/s.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2506_16759_b200/csrc/common.cuh"
using namespace h2;

template <int ILP>
__global__ void k_eval(double* out, int iters, const double* __restrict__ tabg) {
  __shared__ double tab[256];
  for (int j = threadIdx.x; j < 256; j += blockDim.x) tab[j] = tabg[j];
  __syncthreads();
  double xi = threadIdx.x * 1e-3, yi = blockIdx.x * 1e-4, zi = 0.3;
  double acc = 0;
  double xj[ILP];
#pragma unroll
  for (int q = 0; q < ILP; ++q) xj[q] = q * 0.01;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < ILP; ++q) {
      double r2 = dist2(xi, yi, zi, xj[q], 0.2, 0.1);
      acc += kernel_scaled<H2_K_EXP>(r2, 0.0, tab);
      xj[q] += 1e-6;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * 8);
  double* tab; cudaMalloc(&tab, 256 * 8);
  double h[256]; for (int j = 0; j < 256; ++j) h[j] = exp2(j / 256.0);
  cudaMemcpy(tab, h, 2048, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int threads : {256, 512, 1024}) for (int blocksPerSM : {1, 2, 4}) {
    if (threads * blocksPerSM > 2048) continue;
    int grid = 148 * blocksPerSM, iters = 2000;
    k_eval<8><<<grid, threads>>>(out, 10, tab);
    cudaEventRecord(a);
    k_eval<8><<<grid, threads>>>(out, iters, tab);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ents = (double)grid * threads * iters * 8;
    printf("threads %4d x %d/SM: %.3f ms, %.3f Gentries/s, per SM per clk %.2f entries\n", threads, blocksPerSM, ms,
           ents / ms / 1e6, ents / (ms * 1e-3) / (148 * 1.965e9));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
