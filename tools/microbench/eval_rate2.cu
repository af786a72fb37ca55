// Ceiling of the sketch_tc evaluation chain (expk_fixed52, 19 FP64 ops/entry) without the MMA
// pipeline: entries/clk/SM for 1 CTA/SM of T threads, ILP independent entries per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o eval_rate2 eval_rate2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint2 expk(double r2, const double* __restrict__ tab, uint32_t lane8) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double r0 = r2 * y0;
  const double e = fma(-r0, y0, 1.0);
  const double pc = fma(e, 0.375, 0.5);
  const double r = fma(r0 * e, pc, r0);
  const double SH = 6755399441055744.0;
  const double t = fma(r, -369.32993046757464, SH);
  const double kf = t - SH;
  const int n = __double2loint(t);
  const double g = fma(kf, -0.0027076061740622863, -r);
  double p = fma(g, 1.0 / 24.0, 1.0 / 6.0);
  p = fma(p, g, 0.5);
  p = fma(p, g, 1.0);
  p = fma(p, g, 1.0);
  uint32_t idx;
  asm("lop3.b32 %0, %1, 0x7F80, %2, 0xEA;" : "=r"(idx) : "r"((uint32_t)n << 7), "r"(lane8));
  const double tv = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(tab) + idx);
  int th;
  asm("{\n .reg .s32 e;\n shr.s32 e, %1, 8;\n mad.lo.s32 %0, e, 1048576, %2;\n}\n" : "=r"(th) : "r"(n), "r"(__double2hiint(tv)));
  const double w = fma(__hiloint2double(th, __double2loint(tv)), p, 4503599627370496.0);
  return make_uint2((uint32_t)__double2loint(w), (uint32_t)(__double2hiint(w) - 0x43300000));
}

__device__ __forceinline__ void transpose4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t* o) {
  uint32_t p = __byte_perm(a, b, 0x5140), q = __byte_perm(c, d, 0x5140);
  uint32_t r = __byte_perm(a, b, 0x7362), t = __byte_perm(c, d, 0x7362);
  o[0] = __byte_perm(p, q, 0x5410);
  o[1] = __byte_perm(p, q, 0x7632);
  o[2] = __byte_perm(r, t, 0x5410);
  o[3] = __byte_perm(r, t, 0x7632);
}

// evaluation + byte slicing + 7 STS.64 per 8 entries (the sketch_tc producer body, no barriers)
template <int RPT>
__global__ void ks(uint32_t* out, int iters, const double4* __restrict__ C) {
  __shared__ __align__(128) double tab[16 * 256];
  __shared__ double4 cs[128];
  __shared__ __align__(16) uint8_t A[7 * 1024];
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) tab[e] = exp2((double)(e >> 4) / 256.0 + 52.0);
  for (int e = threadIdx.x; e < 128; e += blockDim.x) cs[e] = C[e];
  __syncthreads();
  const uint32_t lane8 = 8u * (threadIdx.x & 15);
  double4 ci[RPT];
  for (int k = 0; k < RPT; ++k) ci[k] = C[(threadIdx.x + 37 * k) & 127];
  const int off = (threadIdx.x * 8) & 1023;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      uint32_t lo[8], hi[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double4 p = cs[(q + it * 8) & 127];
        const double dx = ci[k].x - p.x, dy = ci[k].y - p.y, dz = ci[k].z - p.z;
        const double r2 = fma(dz, dz, fma(dy, dy, fma(dx, dx, 9.332636185032189e-302)));
        const uint2 m = expk(r2, tab, lane8);
        lo[q] = m.x; hi[q] = m.y;
      }
      uint32_t w[4][4];
      transpose4(lo[0], lo[1], lo[2], lo[3], w[0]);
      transpose4(lo[4], lo[5], lo[6], lo[7], w[1]);
      transpose4(hi[0], hi[1], hi[2], hi[3], w[2]);
      transpose4(hi[4], hi[5], hi[6], hi[7], w[3]);
#pragma unroll
      for (int s = 0; s < 4; ++s) *reinterpret_cast<uint2*>(A + s * 1024 + ((off + k * 256 + it * 8) & 1023)) = make_uint2(w[0][s], w[1][s]);
#pragma unroll
      for (int s = 0; s < 3; ++s) *reinterpret_cast<uint2*>(A + (s + 4) * 1024 + ((off + k * 256 + it * 8) & 1023)) = make_uint2(w[2][s], w[3][s]);
    }
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int e = 0; e < 7 * 1024; e += 97) acc += A[(e + threadIdx.x) % (7 * 1024)];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int ILP>
__global__ void k(uint32_t* out, int iters, const double4* __restrict__ C) {
  __shared__ __align__(128) double tab[16 * 256];
  __shared__ double4 cs[128];
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) tab[e] = exp2((double)(e >> 4) / 256.0 + 52.0);
  for (int e = threadIdx.x; e < 128; e += blockDim.x) cs[e] = C[e];
  __syncthreads();
  const double4 ci = C[threadIdx.x & 127];
  const uint32_t lane8 = 8u * (threadIdx.x & 15);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < ILP; ++q) {
      const double4 p = cs[(q + it * ILP) & 127];
      const double dx = ci.x - p.x, dy = ci.y - p.y, dz = ci.z - p.z;
      const double r2 = fma(dz, dz, fma(dy, dy, fma(dx, dx, 9.332636185032189e-302)));
      const uint2 m = expk(r2, tab, lane8);
      acc ^= m.x + m.y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 1024 * 4);
  double4* C; cudaMalloc(&C, 128 * sizeof(double4));
  double4 h[128]; for (int i = 0; i < 128; ++i) h[i] = make_double4((i * 37 % 101) * 0.05, (i * 11 % 89) * 0.05, (i % 7) * 0.5, 0);
  cudaMemcpy(C, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int threads : {256, 384, 512, 768, 1024}) {
    for (int ilp : {8, 16}) {
      const int iters = 4000 / (ilp / 8);
      auto run = [&](int it) { if (ilp == 8) k<8><<<148, threads>>>(out, it, C); else k<16><<<148, threads>>>(out, it, C); };
      run(10);
      cudaEventRecord(a); run(iters); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ents = 148.0 * threads * iters * ilp;
      printf("threads %4d ilp %2d: %.3f ms, %.1f Gentries/s, %.2f entries/clk/SM, FP64 pipe %.1f %%\n", threads, ilp, ms,
             ents / ms / 1e6, ents / (ms * 1e-3) / (148 * 1.965e9), 100.0 * 19 * ents / (ms * 1e-3) / (148 * 64 * 1.965e9));
    }
  }
  for (int threads : {256, 512, 1024}) {
    const int iters = 1000;
    ks<2><<<148, threads>>>(out, 10, C);
    cudaEventRecord(a); ks<2><<<148, threads>>>(out, iters, C); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ents = 148.0 * threads * iters * 16;
    printf("with slicing+STS: threads %4d rpt 2: %.1f Gentries/s, %.2f entries/clk/SM, FP64 pipe %.1f %%\n", threads,
           ents / ms / 1e6, ents / (ms * 1e-3) / (148 * 1.965e9), 100.0 * 19 * ents / (ms * 1e-3) / (148 * 64 * 1.965e9));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
