// What limits the sketch_tc evaluation chain (19 FP64 ops/entry) to ~76 % of the FP64 pipe?
// Variants of the eval_rate2 chain (timing only; V1-V3 compute wrong values on purpose):
//   V0 baseline; V1 no MUFU.RSQ64H (integer seed instead); V2 no table LDS (value synthesised);
//   V3 neither; V4 FP32 MUFU.RSQ seed (double->float by integer ops, float->double by integer ops);
//   V5 = V0 with the r^2 floor dropped from the first FMA (DMUL + 2 DFMA, same count).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o eval_rate3 eval_rate3.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ uint2 expk(double r2, const double* __restrict__ tab, uint32_t lane8) {
  double y0;
  if (V == 1 || V == 3) {
    y0 = __hiloint2double(0x5FE6EB50 - (__double2hiint(r2) >> 1), 0);
  } else if (V == 4) {
    // float(r2) by integer ops: exponent rebias (r2 >= 2^-100 assumed here), mantissa top 23 bits
    const int hi = __double2hiint(r2);
    const uint32_t fb = ((uint32_t)(hi - (896 << 20)) << 3) | ((uint32_t)__double2loint(r2) >> 29);
    const float yf = rsqrtf(__uint_as_float(fb));
    const uint32_t yb = __float_as_uint(yf);
    y0 = __hiloint2double((int)((yb >> 3) + (896u << 20)), (int)(yb << 29));
  } else {
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  }
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
  double tv;
  if (V == 2 || V == 3) tv = __hiloint2double(0x43300000 + (idx & 0xFF), idx);
  else tv = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(tab) + idx);
  int th;
  asm("{\n .reg .s32 e;\n shr.s32 e, %1, 8;\n mad.lo.s32 %0, e, 1048576, %2;\n}\n" : "=r"(th) : "r"(n), "r"(__double2hiint(tv)));
  const double w = fma(__hiloint2double(th, __double2loint(tv)), p, 4503599627370496.0);
  return make_uint2((uint32_t)__double2loint(w), (uint32_t)(__double2hiint(w) - 0x43300000));
}

// pure FP64 chain of the same shape: 19 dependent-ish FP64 ops per entry, nothing else
__device__ __forceinline__ uint2 fp64only(double r2) {
  const double y0 = r2 * 0.5;
  const double r0 = r2 * y0;
  const double e = fma(-r0, y0, 1.0);
  const double pc = fma(e, 0.375, 0.5);
  const double r = fma(r0 * e, pc, r0);
  const double t = fma(r, -369.32993046757464, 6755399441055744.0);
  const double kf = t - 6755399441055744.0;
  const double g = fma(kf, -0.0027076061740622863, -r);
  double p = fma(g, 1.0 / 24.0, 1.0 / 6.0);
  p = fma(p, g, 0.5);
  p = fma(p, g, 1.0);
  p = fma(p, g, 1.0);
  const double w = fma(t, p, 4503599627370496.0);
  return make_uint2((uint32_t)__double2loint(w), (uint32_t)__double2hiint(w));
}

template <int V, int ILP>
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
      double r2;
      if (V == 5) r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      else r2 = fma(dz, dz, fma(dy, dy, fma(dx, dx, 9.332636185032189e-302)));
      const uint2 m = V == 6 ? fp64only(r2) : expk<V == 5 ? 0 : V>(r2, tab, lane8);
      acc ^= m.x + m.y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V>
void run(const char* name, uint32_t* out, const double4* C) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int threads : {512, 1024}) {
    const int iters = 4000;
    k<V, 8><<<148, threads>>>(out, 10, C);
    cudaEventRecord(a); k<V, 8><<<148, threads>>>(out, iters, C); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ents = 148.0 * threads * iters * 8;
    printf("%-34s threads %4d: %.2f entries/clk/SM, FP64 pipe %.1f %% (19 ops/entry)\n", name, threads,
           ents / (ms * 1e-3) / (148 * 1.965e9), 100.0 * 19 * ents / (ms * 1e-3) / (148 * 64 * 1.965e9));
  }
}

int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 1024 * 4);
  double4* C; cudaMalloc(&C, 128 * sizeof(double4));
  double4 h[128]; for (int i = 0; i < 128; ++i) h[i] = make_double4((i * 37 % 101) * 0.05, (i * 11 % 89) * 0.05, (i % 7) * 0.5, 0);
  cudaMemcpy(C, h, sizeof(h), cudaMemcpyHostToDevice);
  run<0>("V0 baseline", out, C);
  run<1>("V1 no MUFU.RSQ64H", out, C);
  run<2>("V2 no table LDS", out, C);
  run<3>("V3 no MUFU, no LDS", out, C);
  run<4>("V4 FP32 MUFU.RSQ seed", out, C);
  run<5>("V5 no r2 floor", out, C);
  run<6>("V6 FP64 ops only (+coords)", out, C);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
