// Do int8 tcgen05.mma and FP64 (DFMA) work overlap on an sm_100a SM?
// One CTA per SM: 16 DFMA warps (independent FMA chains) + 1 MMA warp issuing
// tcgen05.mma.kind::i8 M=128 N=NCOL K=32 from fixed shared-memory operands (K-major, no swizzle,
// the sketch_tc layout).  Modes: 1 = MMA only, 2 = DFMA only, 3 = both (same amounts of work).
// Also the same with DADD/DMUL mixes and the pure UMMA rate for N = 64..256.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_fp64_overlap mma_fp64_overlap.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int TM, int NCOL) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(NCOL >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(addr), "r"(parity));
}

template <int NCOL, int NPAIR>
__global__ void __launch_bounds__(544, 1) kern(int mode, int mma_batches, int fma_iters, double* out, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  constexpr int ABYTES = 128 * 128;        // M = 128 x 128 j (4 k-steps)
  constexpr int BBYTES = NCOL * 128;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < (NPAIR * ABYTES + BBYTES) / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(smem)[e] = e * 2654435761u;
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_a));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_a + 8));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  double acc = 0;
  if (warp == 16) {
    if ((mode & 1) && lane == 0) {
      constexpr uint32_t ID = idesc_i8(128, NCOL);
      for (int b = 0; b < mma_batches; ++b) {
#pragma unroll
        for (int p = 0; p < NPAIR; ++p)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = umma_desc(sbase + p * ABYTES + kk * 2 * 2048, 2048, 128);
            const uint64_t bd = umma_desc(sbase + NPAIR * ABYTES + kk * 2 * (NCOL * 16), NCOL * 16, 128);
            const uint32_t en = (kk == 0 && b == 0) ? 0u : 1u;
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem + (uint32_t)(p * NCOL)), "l"(ad), "l"(bd), "r"(ID), "r"(en));
          }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar_a + 8 * (b & 1)));
        if (b >= 1) mbar_wait(bar_a + 8 * ((b - 1) & 1), ((b - 1) >> 1) & 1);   // two batches in flight
      }
      if (mma_batches >= 1) mbar_wait(bar_a + 8 * ((mma_batches - 1) & 1), ((mma_batches - 1) >> 1) & 1);
      {
      }
    }
  } else if (mode & 4) {   // FP32 chains instead (does the UMMA stream slow the FP32 pipe too?)
    float x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = tid + u;
    for (int i = 0; i < fma_iters; ++i) {
#pragma unroll
      for (int u = 0; u < 16; ++u) x[u] = fmaf(x[u], 1.0000001f, 1e-9f);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += x[u];
  } else if (mode & 2) {
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = tid + u;
    const double a = 1.0000001, c = 1e-9;
    for (int i = 0; i < fma_iters; ++i) {
#pragma unroll
      for (int u = 0; u < 16; ++u) x[u] = fma(x[u], a, c);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += x[u];
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  out[blockIdx.x * blockDim.x + tid] = acc;
  if (lane == 0) cyc[blockIdx.x * 17 + warp] = t1 - t0;
}

template <int NCOL, int NPAIR>
void run(const char* label, int mode, int batches, int iters) {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 544 * 8);
  cudaMalloc(&cyc, 148 * 17 * 8);
  const int sm = NPAIR * 128 * 128 + NCOL * 128;
  cudaFuncSetAttribute(kern<NCOL, NPAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  kern<NCOL, NPAIR><<<148, 544, sm>>>(mode, 2, 2, out, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<NCOL, NPAIR><<<148, 544, sm>>>(mode, batches, iters, out, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[17]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double mmaops = 2.0 * 128 * NCOL * 32 * 4 * NPAIR * (double)batches * 148 * ((mode & 1) ? 1 : 0);
  const double fops = 2.0 * 16 * 16 * 32 * (double)iters * 148 * ((mode & 6) ? 1 : 0);
  printf("%-28s mode %d: %8.3f ms  int8 %7.1f TOPS  fp64 %6.2f TFLOP/s  mma-warp cyc %lld  fma-warp cyc %lld  err %s\n",
         label, mode, ms, mmaops / ms / 1e9, fops / ms / 1e9, h[16], h[0], cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  // pure UMMA rate vs N
  run<64, 3>("i8 M128 N64", 1, 20000, 0);
  run<128, 3>("i8 M128 N128", 1, 10000, 0);
  run<160, 3>("i8 M128 N160", 1, 8000, 0);
  run<192, 2>("i8 M128 N192", 1, 8000, 0);
  run<256, 1>("i8 M128 N256", 1, 10000, 0);
  // the sketch mix: 12 UMMAs N = 160 per batch vs DFMA chains, alone and together
  const int B = 8000, F = 60000;
  run<160, 3>("N160 x12 / DFMA", 1, B, F);
  run<160, 3>("N160 x12 / DFMA", 2, B, F);
  run<160, 3>("N160 x12 / DFMA", 3, B, F);
  run<160, 3>("N160 x12 / FFMA", 4, B, 2 * F);
  run<160, 3>("N160 x12 / FFMA", 5, B, 2 * F);
  run<128, 3>("N128 x12 / DFMA", 1, B, F);
  run<128, 3>("N128 x12 / DFMA", 3, B, F);
  run<64, 3>("N64 x12 / DFMA", 1, 2 * B, F);
  run<64, 3>("N64 x12 / DFMA", 3, 2 * B, F);
  return 0;
}
