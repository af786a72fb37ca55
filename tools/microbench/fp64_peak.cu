// FP64 pipe microbenchmark for sm_100a: DFMA vs DMMA (mma.sync m8n8k4 f64) throughput,
// and whether the two overlap when interleaved in one warp / split across warps.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double a, double b) {
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = 0;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma(c[2 * u], c[2 * u + 1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// interleaved in one warp: 8 DMMA + 32 DFMA per iteration
__global__ void k_mix(double* out, double a, double b) {
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = 0;
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma(c[2 * u], c[2 * u + 1], a, b);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// split: even warps DMMA, odd warps DFMA
__global__ void k_split(double* out, double a, double b) {
  int w = threadIdx.x >> 5;
  double s = 0;
  if (w & 1) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
      }
    }
    s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  } else {
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = 0;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) dmma(c[2 * u], c[2 * u + 1], a, b);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP64 exp + sqrt throughput (libdevice)
__global__ void k_exp(double* out, double a) {
  double s = 0, x = threadIdx.x * 1e-3;
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) { s += exp(-sqrt(x * x + a) * 5.0); x += 1e-7; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  int blocks = p.multiProcessorCount * 8, threads = 256;
  double* out; cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*launch)(), double flops) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-8s %8.3f ms  %8.2f TFLOP/s\n", name, best, flops / (best * 1e-3) / 1e12);
  };
  static int B, T; B = blocks; T = threads; static double* O; O = out;
  double nthreads = (double)blocks * threads;
  run("dfma", [] { k_dfma<<<B, T>>>(O, 0.999, 1e-3); }, nthreads * ITERS * 32 * 2.0);
  run("dmma", [] { k_dmma<<<B, T>>>(O, 0.999, 1e-3); }, nthreads / 32 * ITERS * 8 * 512.0);
  run("mix", [] { k_mix<<<B, T>>>(O, 0.999, 1e-3); }, nthreads / 32 * ITERS * 8 * 512.0 + nthreads * ITERS * 32 * 2.0);
  run("split", [] { k_split<<<B, T>>>(O, 0.999, 1e-3); }, nthreads / 64 * ITERS * 8 * 512.0 + nthreads / 2 * ITERS * 32 * 2.0);
  run("exp+sqrt", [] { k_exp<<<B, T>>>(O, 0.5); }, nthreads * ITERS);  // reported as G-evals/s x1e3
  cudaError_t err = cudaGetLastError(); printf("err %s\n", cudaGetErrorString(err));
  return 0;
}
