// Dense-kernel sketch Y = K Omega on the 5th-generation tensor cores (tcgen05.mma kind::i8),
// exact in integer arithmetic (Algorithm 1 line 1; BASELINE configs[0..2]).
//
// FP64 has no tcgen05 kind, and on B200 DMMA shares the FP64 pipe with DFMA, so a DMMA sketch
// spends ~64 % of its FP64 issue on the contraction.  Here the contraction leaves the FP64 pipe:
//   * Omega entries are exact quarters q/4, q in [-32, 32] (the centred binomial, R8):
//     one signed int8 operand.
//   * every kernel entry K in (0, 1] (exp kernel) is generated in FP64 registers and converted
//     to the fixed-point integer m = round(K 2^47) (6 bytes; 2^52 / 7 bytes with H2_TC_SLICES=7;
//     Helmholtz: a signed 53-bit format, 7 bytes, R32) by one FMA; its bytes are the
//     int8 slices A_s (K-major UMMA core-matrix layout in shared memory).
//   * tcgen05.mma.kind::i8 accumulates D_s = A_s B exactly in int32 TMEM; every 65536 j the
//     accumulators are drained: Y += sum_s 2^(8s - 47 - 2) D_s in FP64.
//   * 160-column passes (exp): 64 rows per CTA, slices s and s + 3 stacked as one M = 128 A
//     operand, so each K evaluation feeds 160 columns at the tensor core's full M = 128 rate.
// The result is the exact product of the grid-rounded K with Omega, rounded only at the drains
// (the grid rounding is at the level of an FP64 GEMM's own accumulated rounding), and the FP64
// pipe only evaluates K.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "alloc.hpp"
#include "common.cuh"
#include "kernels.hpp"

namespace h2 {
namespace {


// Byte slices NS of the fixed-point K: 7 (52-bit grid, K 2^52 / v 2^51) or 6 (47-bit grid, K 2^47 /
// v 2^46: its rounding, <= 2^-48 max|K| per entry, stays below the accumulated rounding of an FP64
// GEMM of the same sums, and 6 slices leave TMEM room for 160-column passes).  The low-half /
// high-half split of the slices (summation chains and TMEM lane halves) is NSPLIT.
#ifndef H2_TC_NPW
#define H2_TC_NPW 16
#endif
#ifndef H2_TC_PACK
#define H2_TC_PACK 1
#endif
template <int NS> struct SliceFmt {
  static constexpr int NSPLIT = 3;                 // chains (s0..s2) + (s3..s{NS-1})
  static constexpr int KEXP = NS == 7 ? 52 : 47;   // exp: m = round(K 2^KEXP)
  static constexpr int HEXP = NS == 7 ? 51 : 46;   // Helmholtz: m = round(v 2^HEXP), |v| < 1
};
constexpr int TC_NB = 4;                       // coordinate / B ring depth
constexpr int TC_DRAIN_J = 65536;              // j per TMEM drain: 65536 * 255 * 32 < 2^31

// Shared-memory plan of one (TM rows x NCOL columns x JC j per chunk) configuration:
//   A: NA buffers of 7 byte slices (TM x JC each), B ring: NB x (NCOL x JC) int8,
//   coordinate ring NB x CBUF, mbarriers (the 32 KB lane-replicated exp table is static shared
//   memory: its address is an immediate of the table loads).
template <int TM, int NCOL, int JC, int NS>
struct TcPlan {
  static constexpr int SLICE = TM * JC;                    // bytes of one slice
  static constexpr int ABUF = NS * SLICE;                  // 56 / 48 KB (TM x JC = 8192), 28 / 24 KB (4096)
  static constexpr int NA = ABUF > 32768 ? (NCOL > 64 ? 2 : 3) : 4;   // A buffers
  static constexpr int BBUF = NCOL * JC;
  static constexpr int CBUF = JC * 32 + JC * 2;            // JC x (x, y, z, pad) doubles, +16 B per 8 j (bank skew)
  static constexpr int DRAIN = TC_DRAIN_J / JC;            // chunks per TMEM drain
  static constexpr int A0 = 0;
  static constexpr int B0 = NA * ABUF;
  static constexpr int C0 = B0 + TC_NB * BBUF;
  static constexpr int T0 = C0 + TC_NB * CBUF;
  static constexpr int BAR = T0;                         // full[NA], empty[NA], loaded[NB], drain
  static constexpr int TOTAL = BAR + 8 * (2 * NA + TC_NB + 1) + 16;
  static_assert(TOTAL + 16 * 256 * 8 <= 227 * 1024, "shared memory plan exceeds 227 KB");
};

// UMMA shared-memory descriptor, K-major, no swizzle (canonical ((8,m),(16B,2)):((16B,SBO),(1,LBO)))
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);   // version 1 (sm_100)
}

// instruction descriptor: D s32, A u8, B s8, both K-major, N = NCOL, M = TM
template <int TM, int NCOL>
__host__ __device__ constexpr uint32_t idesc_i8() {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(NCOL >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

// TMEM address offset of the int32 accumulator of byte slice s.
//   TM = 128: all 128 lanes, slice s at columns [s NCOL, (s+1) NCOL).
//   TM = 64 : an M = 64 accumulator occupies lanes 0-15 of each 32-lane sub-partition (row
//             16 q + l -> lane 32 q + l); a second one interleaves in lanes 16-31 at the same
//             columns.  Slices 0-3 take the low half at columns s*NCOL, slices 4-6 the high
//             half (lane offset 16) at columns (s-4)*NCOL: 7 x 128 columns in 4 x 128.
template <int TM, int NCOL, int NS>
__device__ __forceinline__ uint32_t tmem_slice(int s) {
  constexpr int H = SliceFmt<NS>::NSPLIT;
  if constexpr (TM == 128) return (uint32_t)(s * NCOL);
  else return (s < H) ? (uint32_t)(s * NCOL) : ((16u << 16) | (uint32_t)((s - H) * NCOL));
}

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(addr), "r"(count));
}
// with a suspend-time hint (ns): the waiting warp is parked by the hardware until the phase
// completes (or the hint expires) instead of re-issuing try_wait, which keeps issue slots free
// for the evaluating warps (the kernel is issue-bound: ~1 non-FP64 instruction per FP64 one)
__device__ __forceinline__ void mbar_wait_hint(uint32_t addr, uint32_t parity, uint32_t hint) {
  asm volatile(
      "{\n .reg .pred p;\n WAITH_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAITH_%=;\n}\n" ::"r"(addr),
      "r"(parity), "r"(hint));
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(addr),
      "r"(parity));
}


// r'^2 = |x'-y'|^2 + 2^-1000: the floor (folded into the first FMA, no extra operation) keeps
// 1/sqrt finite at x' = y' and is below half an ulp of every r'^2 >= 2^-947.
__device__ __forceinline__ double dist2_floor(double xi, double yi, double zi, double xj, double yj, double zj) {
  const double dx = xi - xj, dy = yi - yj, dz = zi - zj;
  return fma(dz, dz, fma(dy, dy, fma(dx, dx, 9.332636185032189e-302)));   // 2^-1000
}

// m = round(exp(-r') 2^52) for r2 = r'^2 (scaled coordinates) as (lo 32, hi 21 bits).
// Domain: r' <= 650 (host-checked: sketch_tc_supported), so n = rint(-256 r'/ln2) > -2^18 and the
// exponent arithmetic below stays in the normal range.
//   r' = r2 y0 (1 + e/2 + 3e^2/8), e = 1 - r2 y0^2, y0 = MUFU.RSQ64H(r2) (~2^-20): the cubic
//       correction applied to r2 y0 directly (error 5e^3/16 ~ 2^-60);
//   e^{-r'} = 2^(n/256) p(g), g = -r' - n ln2/256 (|g| <= ln2/512), p = degree-4 Taylor;
//   w = T_n p + 2^52 with T_n = 2^(52 + n/256) (table 2^(52 + j/256), lane-replicated: entry j of
//       copy l at byte 128 j + 8 l, so the 32 lookups of a warp are bank-conflict free; exponent
//       n >> 8 added to its high word): one DFMA, one rounding = the fixed-point rounding of
//       K 2^52;
//   m = bits(w) - bits(2^52): the FP64 bit pattern is monotonic, so for w in [2^52, 2^53] this
//       is exactly w - 2^52, including K -> 1 (w = 2^53, m = 2^52, slice 6 = 0x10).
// FP64 pipe: 6 (r'^2, caller) + 5 (r') + 7 (g, p) + 1 (w) = 19.
// H2_TC_EXP1024 (default): a 1024-entry table 2^(KEXP + j/1024) in 4 lane-interleaved copies
// (entry j of copy c at byte 32 j + 8 c, copy = lane & 3) and a degree-3 polynomial on
// |g| <= ln2/2048 constrained to p(0) = 1 (minimax for the relative error: 2.2e-16, i.e. 0.03
// units of the 2^-47 grid), one FP64 operation less than the degree-4 / 256-entry form:
// FP64 pipe 6 (r'^2) + 5 (r') + 6 (g, p) + 1 (w) = 18.
#ifndef H2_TC_EXP1024
#define H2_TC_EXP1024 1
#endif
constexpr int TC_TAB_SHIFT = H2_TC_EXP1024 ? 2 : 4;        // log2(copies): 4 copies x 1024 or 16 x 256
constexpr double TC_TAB_STEP = H2_TC_EXP1024 ? 1.0 / 1024.0 : 1.0 / 256.0;
__device__ __forceinline__ uint32_t tc_lane8(int lane) { return 8u * (uint32_t)(lane & ((1 << TC_TAB_SHIFT) - 1)); }

__device__ __forceinline__ uint2 expk_fixed52_t1024(double r2, const double* __restrict__ tab, uint32_t lane8) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double r0 = r2 * y0;
  const double e = fma(-r0, y0, 1.0);
  const double pc = fma(e, 0.375, 0.5);
  const double r = fma(r0 * e, pc, r0);
  const double SH = 6755399441055744.0;
  const double t = fma(r, -1477.3197218702985, SH);       // -1024/ln2
  const double kf = t - SH;
  const int n = __double2loint(t);
  const double g = fma(kf, -0.0006769015435155716, -r);   // |g| <= ln2/2048
  double q = fma(g, 0.16666666522088344, 0.5000000039549349);
  q = fma(q, g, 1.0000000000000002);
  const double p = fma(q, g, 1.0);
  uint32_t idx;   // ((n & 1023) << 5) | lane8 in one LOP3
  asm("lop3.b32 %0, %1, 0x7FE0, %2, 0xEA;" : "=r"(idx) : "r"((uint32_t)n << 5), "r"(lane8));
  const double tv = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(tab) + idx);
  int th;   // hi(T_j) + (n >> 10) 2^20
  asm("{\n .reg .s32 e;\n shr.s32 e, %1, 10;\n mad.lo.s32 %0, e, 1048576, %2;\n}\n"
      : "=r"(th) : "r"(n), "r"(__double2hiint(tv)));
  const double w = fma(__hiloint2double(th, __double2loint(tv)), p, 4503599627370496.0);
  return make_uint2((uint32_t)__double2loint(w), (uint32_t)(__double2hiint(w) - 0x43300000));
}

__device__ __forceinline__ uint2 expk_fixed52_t256(double r2, const double* __restrict__ tab, uint32_t lane8) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double r0 = r2 * y0;
  const double e = fma(-r0, y0, 1.0);
  const double pc = fma(e, 0.375, 0.5);
  const double r = fma(r0 * e, pc, r0);
  const double SH = 6755399441055744.0;
  const double t = fma(r, -369.32993046757464, SH);      // -256/ln2
  const double kf = t - SH;
  const int n = __double2loint(t);
  const double g = fma(kf, -0.0027076061740622863, -r);
  double p = fma(g, 1.0 / 24.0, 1.0 / 6.0);
  p = fma(p, g, 0.5);
  p = fma(p, g, 1.0);
  p = fma(p, g, 1.0);
  uint32_t idx;   // ((n & 255) << 7) | lane8 in one LOP3
  asm("lop3.b32 %0, %1, 0x7F80, %2, 0xEA;" : "=r"(idx) : "r"((uint32_t)n << 7), "r"(lane8));
  const double tv = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(tab) + idx);
  int th;   // hi(T_j) + (n >> 8) 2^20 as SHF + LEA (the compiler's default is 3 integer operations)
  asm("{\n .reg .s32 e;\n shr.s32 e, %1, 8;\n mad.lo.s32 %0, e, 1048576, %2;\n}\n"
      : "=r"(th) : "r"(n), "r"(__double2hiint(tv)));
  const double w = fma(__hiloint2double(th, __double2loint(tv)), p, 4503599627370496.0);
  return make_uint2((uint32_t)__double2loint(w), (uint32_t)(__double2hiint(w) - 0x43300000));
}

__device__ __forceinline__ uint2 expk_fixed52(double r2, const double* __restrict__ tab, uint32_t lane8) {
  if constexpr (H2_TC_EXP1024) return expk_fixed52_t1024(r2, tab, lane8);
  else return expk_fixed52_t256(r2, tab, lane8);
}

// Helmholtz (PAPER.md Eq. ie, R20): K = cos(k r)/r, 0 at r = 0, in scaled coordinates
// r' = k r: K = k cos(r')/r'.  Signed 53-bit fixed point with a power-of-two scale 2^E >= max|K|
// (hs = k / 2^E): m = round(v 2^51), v = hs cos(r') / r' in (-1, 1):
//   w = v 2^51 + 3 2^51 in (2^52, 2^53): one FMA, the fixed-point rounding;
//   m = bits(w) - bits(2^52) - 2^51 (hi word - 0x43380000): the 64-bit two's complement of m,
//       whose bytes 0..5 are the unsigned slices and byte 6 (bits 48-55, sign-extended) the
//       signed top slice (tcgen05.mma a_format s8);
//   |v| >= 1 (a pair closer than the scale assumed) is flagged: the caller redoes the pass on
//       the FP64 DMMA path.
// cos(r'): n = rint(2 r'/pi), x = r' - n pi/2 (fdlibm two-term Cody-Waite), cos / sin Taylor
// polynomials on |x| <= pi/4 (to x^16 / x^17: truncation < 1e-16), quadrant by n & 3.
// 1/r': the cubic-corrected rsqrt.  r' = 0 (the diagonal; r2 = the 2^-1000 floor) gives 0.
// FP64 pipe: 6 (r'^2) + 5 (1/r') + 1 (r') + 4 (reduction) + 1 (x^2) + 8 (cos) + 9 (sin) + 2 + 1.
template <int HEXP>
__device__ __forceinline__ uint2 helm_fixed51(double r2, double hs, uint32_t& ovf) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double e = fma(-r2, y0 * y0, 1.0);
  const double y = fma(fma(e, 0.375, 0.5), y0 * e, y0);            // 1/r'
  const double r = r2 * y;
  const double SH = 6755399441055744.0;
  const double t = fma(r, 0.63661977236758134308, SH);             // 2/pi
  const double nf = t - SH;
  const int n = __double2loint(t);
  double x = fma(nf, -1.57079632673412561417e+00, r);              // pio2_1
  x = fma(nf, -6.07710050650619224932e-11, x);                     // pio2_1t
  const double z = x * x;
  double c = fma(z, 4.7794773323873852974e-14, -1.1470745597729724714e-11);   // 1/16!, -1/14!
  c = fma(c, z, 2.0876756987868098979e-09);                        // 1/12!
  c = fma(c, z, -2.7557319223985890653e-07);                       // -1/10!
  c = fma(c, z, 2.4801587301587301587e-05);                        // 1/8!
  c = fma(c, z, -1.3888888888888888889e-03);                       // -1/6!
  c = fma(c, z, 4.1666666666666666667e-02);                        // 1/4!
  c = fma(c, z, -0.5);
  c = fma(c, z, 1.0);
  double sn = fma(z, 2.8114572543455207632e-15, -7.6471637318198164759e-13);  // 1/17!, -1/15!
  sn = fma(sn, z, 1.6059043836821614599e-10);                      // 1/13!
  sn = fma(sn, z, -2.5052108385441718775e-08);                     // -1/11!
  sn = fma(sn, z, 2.7557319223985890653e-06);                      // 1/9!
  sn = fma(sn, z, -1.9841269841269841270e-04);                     // -1/7!
  sn = fma(sn, z, 8.3333333333333333333e-03);                      // 1/5!
  sn = fma(sn, z, -0.16666666666666666667);                        // -1/3!
  sn = fma(sn * z, x, x);
  // quadrant: 0 cos, 1 -sin, 2 -cos, 3 sin
  const bool odd = n & 1;
  const uint32_t neg = (uint32_t)((n + 1) & 2) << 30;              // sign for quadrants 1, 2
  const double tr = __hiloint2double((int)((uint32_t)__double2hiint(odd ? sn : c) ^ neg),
                                     __double2loint(odd ? sn : c));
  double v = (hs * tr) * y;
  if (__double2hiint(r2) < 0x03B00000) v = 0.0;                    // r2 < 2^-900: x' = y'
  const double w = fma(v, (double)(1ull << HEXP), 6755399441055744.0);  // v 2^HEXP + 3 2^51
  const int mh = __double2hiint(w) - 0x43380000;
  ovf |= (uint32_t)(mh + (1 << (HEXP - 32))) > (2u << (HEXP - 32));
  return make_uint2((uint32_t)__double2loint(w), (uint32_t)mh);
}

// H2_TC_HTAB (default): cos(r') from a table of (cos, sin)(2 pi j / 1024), j < 1024, in 2
// lane-interleaved copies (16-byte entries; the exp table's 32 KB of static shared memory), and
// short polynomials on the remainder |g| <= pi/1024:  cos(a + g) = C_j c(g) - S_j s(g) with
// c = 1 - g^2/2 + g^4/24 (truncation g^6/720 < 1.2e-18) and s = g - g^3/6 + g^5/120 (< 5e-22);
// reduction g = r' - n (2 pi / 1024) by a 2-term Cody-Waite split (hi has 36 significant bits:
// n hi is exact for n < 2^17, i.e. r' <= 650, the host-checked range).  FP64 pipe: 6 (r'^2)
// + 5 (1/r') + 1 (r') + 4 (reduction) + 1 (g^2) + 2 (c) + 3 (s) + 2 (C c - S s) + 2 (v) + 1 (w)
// = 27 instead of 37 (Taylor to x^16 / x^17 on |x| <= pi/4 with the quadrant logic).
#ifndef H2_TC_HTAB
#define H2_TC_HTAB 1
#endif
constexpr int TC_HTAB_N = 1024;
__device__ __forceinline__ void fill_cs_table(double* tab, int tid, int nth) {
  // entry j, copy c at doubles 4 j + 2 c: (cos, sin)(2 pi j / 1024); sincospi of the exact 2j/1024
  for (int e = tid; e < 2 * TC_HTAB_N; e += nth) {
    double sv, cv;
    sincospi((double)(e >> 1) * (2.0 / TC_HTAB_N), &sv, &cv);
    tab[2 * e] = cv;
    tab[2 * e + 1] = sv;
  }
}
template <int HEXP>
__device__ __forceinline__ uint2 helm_fixed51_tab(double r2, double hs, uint32_t& ovf, const double* __restrict__ tab,
                                                  uint32_t lane16) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double e = fma(-r2, y0 * y0, 1.0);
  const double y = fma(fma(e, 0.375, 0.5), y0 * e, y0);            // 1/r'
  const double r = r2 * y;
  const double SH = 6755399441055744.0;
  const double t = fma(r, 162.97466172610083, SH);                 // 1024 / (2 pi)
  const double nf = t - SH;
  const int n = __double2loint(t);
  double g = fma(nf, -0.006135923151532552, r);                    // 2 pi / 1024, 36-bit head
  g = fma(nf, -1.001306309216609e-14, g);                          // tail
  const double z = g * g;
  const double c = fma(fma(z, 4.1666666666666666667e-02, -0.5), z, 1.0);
  const double sn = fma(fma(z, 8.3333333333333333333e-03, -0.16666666666666666667) * z, g, g);
  uint32_t idx;   // byte offset 32 (n & 1023) + 16 (lane & 1)
  asm("lop3.b32 %0, %1, 0x7FE0, %2, 0xEA;" : "=r"(idx) : "r"((uint32_t)n << 5), "r"(lane16));
  const double2 cs = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(tab) + idx);
  const double tr = fma(cs.x, c, -(cs.y * sn));                    // cos(r')
  double v = (hs * tr) * y;
  if (__double2hiint(r2) < 0x03B00000) v = 0.0;                    // r2 < 2^-900: x' = y'
  const double w = fma(v, (double)(1ull << HEXP), 6755399441055744.0);  // v 2^HEXP + 3 2^51
  const int mh = __double2hiint(w) - 0x43380000;
  ovf |= (uint32_t)(mh + (1 << (HEXP - 32))) > (2u << (HEXP - 32));
  return make_uint2((uint32_t)__double2loint(w), (uint32_t)mh);
}
template <int HEXP>
__device__ __forceinline__ uint2 helm_eval(double r2, double hs, uint32_t& ovf, const double* __restrict__ tab,
                                           int lane) {
  if constexpr (H2_TC_HTAB) return helm_fixed51_tab<HEXP>(r2, hs, ovf, tab, 16u * (uint32_t)(lane & 1));
  else return helm_fixed51<HEXP>(r2, hs, ovf);
}

// Explicit dense operator (H2_S_DENSE_MATRIX): the producers read A(i, j)
// from HBM instead of evaluating a kernel; with a power-of-two scale 2^E >= max|A| (hs = 2^-E,
// exact), v = A hs in [-1, 1] takes the signed 53-bit format of the Helmholtz path:
// w = v 2^51 + 3 2^51 (one FMA: the fixed-point rounding, <= 2^-52 max|A| per entry),
// m = bits(w) - bits(2^52) - 2^51, 7 byte slices, the top one signed.  FP64 pipe: 2 per entry.
constexpr int KDENSE = 3;
template <int HEXP>
__device__ __forceinline__ uint2 dense_fixed(double x, double hs, uint32_t& ovf) {
  const double w = fma(x * hs, (double)(1ull << HEXP), 6755399441055744.0);
  const int mh = __double2hiint(w) - 0x43380000;
  ovf |= (uint32_t)(mh + (1 << (HEXP - 32))) > (2u << (HEXP - 32));
  return make_uint2((uint32_t)__double2loint(w), (uint32_t)mh);
}

// 4x4 byte transpose: out[s] = bytes s of (a, b, c, d)
__device__ __forceinline__ void transpose4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t* o) {
  uint32_t p = __byte_perm(a, b, 0x5140), q = __byte_perm(c, d, 0x5140);
  uint32_t r = __byte_perm(a, b, 0x7362), t = __byte_perm(c, d, 0x7362);
  o[0] = __byte_perm(p, q, 0x5410);
  o[1] = __byte_perm(p, q, 0x7632);
  o[2] = __byte_perm(r, t, 0x5410);
  o[3] = __byte_perm(r, t, 0x7632);
}

__global__ void coords_aos_kernel(const double* X, const double* Y, const double* Z, int64_t n, int64_t npad, double cs,
                                  double4* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npad; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < n ? make_double4(X[i] * cs, Y[i] * cs, Z[i] * cs, 0.0) : make_double4(0.0, 0.0, 0.0, 0.0);
}

// Omega (n x ncols doubles q/4) -> int8 q per 64-j chunk in the B core-matrix layout for NCOL
// columns: chunk t, column c, jj: t*NCOL*64 + (jj/16)*(NCOL*16) + (c/8)*128 + (c%8)*16 + jj%16
// (0 beyond n / ncols).  The K-direction core stride (LBO) is NCOL*16 bytes.
__global__ void omega_i8_kernel(const double* __restrict__ Om, int64_t ldo, int64_t n, int ncols, int NCOL, int JC,
                                int64_t nchunks, int8_t* __restrict__ out) {
  const int64_t total = nchunks * JC * NCOL;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / NCOL;
    const int c = (int)(e - j * NCOL);
    const int64_t t = j / JC;
    const int jj = (int)(j - t * JC);
    int q = 0;
    if (j < n && c < ncols) q = __double2int_rn(Om[j * ldo + c] * 4.0);
    out[t * (NCOL * JC) + (jj >> 4) * (NCOL * 16) + (c >> 3) * 128 + (c & 7) * 16 + (jj & 15)] = (int8_t)q;
  }
}

// Warp-specialised, barrier-free pipeline per CTA (TM rows x NCOL sample columns):
//   NPW producer warps: wait loaded[slot] (coordinates + B of the chunk landed) and empty[buf]
//     (the MMA that last read A[buf] finished), evaluate TM/(4 NPW) rows x 8 j each, write the 7
//     byte slices to A[buf], fence.proxy.async, arrive on full[buf];
//   1 control warp: waits full[buf], issues the tcgen05.mma of the chunk (NS x JC/32, or NS/2 x
//     JC/32 packed M = 128 ones), commits empty[buf] (and drain on drain chunks), then refills the
//     coordinate / B ring with cp.async tracked by mbarriers (cp.async.mbarrier.arrive.noinc) two
//     chunks ahead;
//   producer warps 0-3 (TMEM sub-partitions 0-3) drain the int32 accumulators after every drain
//     chunk.
// TM = 128, NCOL <= 64 : NS x NCOL TMEM columns.  TM = 64 : either the M = 64 accumulators of
// two slices share TMEM columns in the two lane halves (tmem_slice), or (PACK) slices s and s + 3
// form one M = 128 accumulator in all 128 lanes; one evaluation of K feeds 128 / 160 columns.
template <int KIND, int TM, int NPW, int NCOL, int JC, int NS, bool NEARM = false>
__global__ void __launch_bounds__(32 * (NPW + 1), 1)
    sketch_tc_kernel(const double4* __restrict__ C, int64_t n, int64_t row0, int64_t row1,
                     const int8_t* __restrict__ Bq, int64_t nchunks, int ncols, double* __restrict__ Yout, int64_t ldy,
                     int64_t split_stride, double hs, int wshift, uint32_t* __restrict__ ovf_flag, int pfd,
                     uint32_t hint, const double* __restrict__ Aop, int64_t lda,
                     const int32_t* __restrict__ nl_ptr = nullptr, const int32_t* __restrict__ nl_chunk = nullptr,
                     const uint8_t* __restrict__ nl_mask = nullptr) {
  using P = TcPlan<TM, NCOL, JC, NS>;
  constexpr int NSPLIT = SliceFmt<NS>::NSPLIT;
  constexpr int G = JC / 16;               // 16-j core-matrix groups per chunk
  constexpr int CBUF = P::CBUF;
  constexpr int NTH = 32 * (NPW + 1);
  constexpr int NA = P::NA;
  constexpr int RPT = TM * G / (16 * NPW); // rows per producer thread (TM rows x JC j / (32 NPW lanes x 8 j))
  constexpr int BBUF = P::BBUF;            // B chunk bytes
  // PACK (exp, 6 slices, 64 rows): slices s and s + 3 stacked as the two 64-row halves of one
  // M = 128 A operand (rows 0-63 slice s, 64-127 slice s + 3): 3 full-rate M = 128 MMAs per k step
  // instead of 6 half-rate M = 64 ones; accumulator of pair p = all 128 lanes x NCOL columns at p NCOL
  constexpr bool PACK = KIND == H2_K_EXP && NS == 6 && TM == 64 && H2_TC_PACK;
  // PACK7 (7 slices, 64 rows: Helmholtz, or exp with H2_TC_SLICES=7): the unsigned slices 0-5 as
  // three packed M = 128 pairs (s, s + 3) and the top slice 6 (s8 for Helmholtz) as one M = 64
  // MMA into the low lane half of TMEM columns [3 NCOL, 4 NCOL)
  constexpr bool PACK7 = KIND != H2_K_EXP && NS == 7 && TM == 64 && H2_TC_PACK;   // exp-7: 196 vs 178 ms unpacked
  constexpr int LBO_A = (PACK || PACK7) ? 2 * TM * 16 : TM * 16;   // K-direction core-matrix stride of A
  constexpr int LBO_B = NCOL * 16;         // K-direction core-matrix stride of B
  constexpr uint32_t TMEM_COLS = (TM == 128 && NCOL * NS <= 256) ? 256 : 512;
  constexpr uint32_t IDESC = (PACK || PACK7) ? idesc_i8<128, NCOL>() : idesc_i8<TM, NCOL>();
  constexpr uint32_t IDESC64 = idesc_i8<64, NCOL>() | (KIND == H2_K_EXP ? 0u : (1u << 7));   // PACK7 top slice
  // Helmholtz: the top slice holds the sign (two's complement of the signed fixed point): s8
  constexpr uint32_t IDESC6 = KIND == H2_K_EXP ? IDESC : (IDESC | (1u << 7));
  static_assert(RPT >= 1 && NPW % G == 0 && TM * JC == RPT * 32 * NPW * 8, "producer tiling");
  static_assert((TM == 128 && NCOL * NS <= 512) || (TM == 64 && NCOL * (NS - NSPLIT > NSPLIT ? NS - NSPLIT : NSPLIT) <= 512),
                "TMEM plan");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(128) double tab[16 * 256];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bar_full = sbase + P::BAR;                // NA
  const uint32_t bar_empty = bar_full + 8 * NA;            // NA
  const uint32_t bar_loaded = bar_empty + 8 * NA;          // NB
  const uint32_t bar_drain = bar_loaded + 8 * TC_NB;       // 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P::BAR + 8 * (2 * NA + TC_NB + 1));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rtile = row0 + (int64_t)blockIdx.x * TM;
  // j-split boundaries in 128-j units (independent of JC), so that every pass shape splits and
  // drains at the same j and produces bit-identical sums
  const int64_t nunits = nchunks / (128 / JC);
  // near-field mode (nl_ptr != NULL, TM = 64 row tiles = leaves of exactly 64 points): the tile's
  // j chunks are its near leaves' 128-j chunks (list nl_chunk[nl_ptr[leaf] ..]), each with a mask of
  // the 64-j halves that belong to near leaves; the result is SUBTRACTED from Yout -- the leaf
  // subtraction Y^loc = Y - sum_{b in N} D_{tau,b} Omega_b (Algorithm 1) on the tensor cores
  constexpr bool nearm = NEARM;   // compile time: the sketch pass itself carries no near-mode code
  const int nl0 = nearm ? nl_ptr[rtile / 64] : 0;
  const int64_t ch_b = nearm ? 0 : nunits * blockIdx.y / gridDim.y * (128 / JC);
  const int64_t ch_e = nunits * (blockIdx.y + 1) / gridDim.y * (128 / JC);
  const int nch = nearm ? nl_ptr[rtile / 64 + 1] - nl0 : (int)(ch_e - ch_b);
  auto chunk_of = [&](int it) -> int64_t { return nearm ? (int64_t)nl_chunk[nl0 + it] : ch_b + it; };
  const bool control = (warp == NPW);

  if (KIND == H2_K_HELMHOLTZ && H2_TC_HTAB) fill_cs_table(tab, tid, NTH);
  else
    for (int e = tid; e < 16 * 256; e += NTH) tab[e] = exp2((double)(e >> TC_TAB_SHIFT) * TC_TAB_STEP + (double)SliceFmt<NS>::KEXP);
  if (tid == 0) {
    for (int b = 0; b < NA; ++b) {
      mbar_init(bar_full + 8 * b, NPW);
      mbar_init(bar_empty + 8 * b, 1);
    }
    for (int s = 0; s < TC_NB; ++s) mbar_init(bar_loaded + 8 * s, 32);
    mbar_init(bar_drain, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;
  double* Yo = Yout + blockIdx.y * split_stride;

  if (control) {
    // chunk it -> ring slot it % 4: B (NCOL x 64 bytes) + coordinates (2 KB) in 16 B pieces
    auto prefetch = [&](int it) {
      if (it >= nch) return;
      const int64_t t = chunk_of(it);
      const int slot = it & (TC_NB - 1);
#pragma unroll
      for (int q = 0; q < BBUF / 16 / 32; ++q) {
        const int e = lane + 32 * q;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + P::B0 + slot * BBUF + e * 16),
                     "l"(Bq + t * BBUF + e * 16));
      }
      if (KIND != KDENSE) {
#pragma unroll
        for (int q = 0; q < JC / 16; ++q) {
          const int e = lane + 32 * q;
          const int jc = e >> 1;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + P::C0 + slot * CBUF + e * 16 +
                                                                            (jc >> 3) * 16),
                       "l"(reinterpret_cast<const char*>(C + t * JC) + e * 16));
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar_loaded + 8 * slot));
    };
    for (int q = 0; q < pfd; ++q) prefetch(q);
    for (int it = 0; it < nch; ++it) {
      const int buf = it % NA;
      const int slot = it & (TC_NB - 1);
      if (hint) mbar_wait_hint(bar_full + 8 * buf, (it / NA) & 1, hint);
      else mbar_wait(bar_full + 8 * buf, (it / NA) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const bool first = (it % P::DRAIN) == 0;
      const bool drain = ((it % P::DRAIN) == P::DRAIN - 1) || (it == nch - 1);
      if (lane == 0) {
        const uint32_t a0 = sbase + P::A0 + buf * P::ABUF;
        const uint32_t b0 = sbase + P::B0 + slot * BBUF;
        if (PACK7) {
#pragma unroll
          for (int kk = 0; kk < JC / 32; ++kk) {
            const uint64_t ad = umma_desc(a0 + 6 * P::SLICE + kk * 2 * (TM * 16), TM * 16, 128);
            const uint64_t bd = umma_desc(b0 + kk * 2 * LBO_B, LBO_B, 128);
            const uint32_t acc = (first && kk == 0) ? 0u : 1u;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)(3 * NCOL)),
                "l"(ad), "l"(bd), "r"(IDESC64), "r"(acc));
          }
        }
#pragma unroll
        for (int s = 0; s < (PACK || PACK7 ? 3 : NS); ++s)
#pragma unroll
          for (int kk = 0; kk < JC / 32; ++kk) {
            const uint64_t ad = umma_desc(a0 + s * (PACK || PACK7 ? 2 : 1) * P::SLICE + kk * 2 * LBO_A, LBO_A, 128);
            const uint64_t bd = umma_desc(b0 + kk * 2 * LBO_B, LBO_B, 128);
            const uint32_t acc = (first && kk == 0) ? 0u : 1u;
            const uint32_t dcol = (PACK || PACK7) ? (uint32_t)(s * NCOL) : tmem_slice<TM, NCOL, NS>(s);
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + dcol),
                "l"(ad), "l"(bd), "r"(!PACK && !PACK7 && s == NS - 1 ? IDESC6 : IDESC), "r"(acc));
          }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            bar_empty + 8 * buf));
        if (drain)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              bar_drain));
      }
      __syncwarp();
      // slot of chunk it+2 was last used by chunk it-2: its coordinates were consumed before
      // full(it-2) and its B by MMA(it-2) -> wait for that MMA.  With NA <= 2 the producers of
      // chunk it already waited for MMA(it-NA) before arriving on full(it), and waiting here
      // could alias: MMA(it) commits to the same barrier and may complete its phase too.
      if (pfd == 3) {
        // prefetch distance 3 (TC_NB = 4 slots): the slot of chunk it+3 was last used by chunk
        // it-1, whose coordinates were consumed before full(it-1) and its B by MMA(it-1): wait for
        // MMA(it-1) (its empty barrier is not the one MMA(it) just committed to)
        if (it >= 1) mbar_wait(bar_empty + 8 * ((it - 1) % NA), ((it - 1) / NA) & 1);
        prefetch(it + 3);
      } else {
        if (NA > 2 && it >= 2) mbar_wait(bar_empty + 8 * ((it - 2) % NA), ((it - 2) / NA) & 1);
        prefetch(it + 2);
      }
    }
  } else {
    // producer: rows rs*16 + pair + k*16*(NPW/G) (k < RPT), 8 consecutive j (half h of 16-j group g)
    const int g = warp % G;
    const int rs = warp / G;
    const int h = lane & 1;
    const int r0 = 16 * rs + (lane >> 1);
    double4 ci[RPT];
    const double* arow[RPT];   // KDENSE: the operator rows
    int off[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = r0 + k * 16 * (NPW / G);
      const int64_t ri = (rtile + r < row1) ? (rtile + r) : (row1 - 1);
      if (KIND == KDENSE) arow[k] = Aop + ri * lda;
      else ci[k] = C[ri];
      off[k] = g * LBO_A + (r >> 3) * 128 + (r & 7) * 16 + 8 * h;
    }
    // PACK7: the M = 64 layout of the top slice (64 rows x 16 B per k group)
    const int off6d = g * (TM * 16) - g * LBO_A;
    const uint32_t lane8 = tc_lane8(lane);
    uint32_t ovf = 0;
    int drains = 0;
    // KDENSE: the next chunk's operator entries are loaded into registers while this chunk is
    // converted (one chunk of HBM reads in flight per thread: latency hidden, bandwidth-bound)
    double xa[KIND == KDENSE ? RPT : 1][8];
    auto load_a = [&](int itx, double (&dst)[KIND == KDENSE ? RPT : 1][8]) {
      if constexpr (KIND == KDENSE) {
        const int64_t j0 = (ch_b + itx) * JC + 16 * g + 8 * h;
        if (itx < nch && j0 + 8 <= n && (lda & 1) == 0) {   // 16-byte loads (even lda, even j0)
#pragma unroll
          for (int k = 0; k < RPT; ++k)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double2 v = __ldg(reinterpret_cast<const double2*>(arow[k] + j0) + u);
              dst[k][2 * u] = v.x;
              dst[k][2 * u + 1] = v.y;
            }
        } else {
#pragma unroll
          for (int k = 0; k < RPT; ++k)
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[k][q] = (itx < nch && j0 + q < n) ? __ldg(arow[k] + j0 + q) : 0.0;
        }
      }
    };
    load_a(0, xa);
    for (int it = 0; it < nch; ++it) {
      const int buf = it % NA;
      const int slot = it & (TC_NB - 1);
      if (hint) {
        mbar_wait_hint(bar_loaded + 8 * slot, (it / TC_NB) & 1, hint);
        if (it >= NA) mbar_wait_hint(bar_empty + 8 * buf, ((it - NA) / NA) & 1, hint);
      } else {
        mbar_wait(bar_loaded + 8 * slot, (it / TC_NB) & 1);
        if (it >= NA) mbar_wait(bar_empty + 8 * buf, ((it - NA) / NA) & 1);
      }
      const uint8_t* cb = smem + P::C0 + slot * CBUF;
      uint8_t* Ab = smem + P::A0 + buf * P::ABUF;
      const int jj0 = 16 * g + 8 * h;
      uint32_t lo[RPT][8], hi[RPT][8];
      if constexpr (KIND == KDENSE) {
        // 8 consecutive j of each row (loaded one chunk ahead); columns beyond n are 0
        double xn[RPT][8];
        load_a(it + 1, xn);
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint2 m = dense_fixed<SliceFmt<NS>::HEXP>(xa[k][q], hs, ovf);
            lo[k][q] = m.x;
            hi[k][q] = m.y;
          }
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
          for (int q = 0; q < 8; ++q) xa[k][q] = xn[k][q];
      } else if (nearm && !((nl_mask[nl0 + it] >> (jj0 >> 6)) & 1)) {
        // this warp's 64-j half of the chunk is not a near leaf of the tile: zero slices
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
          for (int q = 0; q < 8; ++q) lo[k][q] = hi[k][q] = 0u;
      } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int jj = jj0 + q;
        const double4 p = *reinterpret_cast<const double4*>(cb + jj * 32 + (jj >> 3) * 16);
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const double r2 = dist2_floor(ci[k].x, ci[k].y, ci[k].z, p.x, p.y, p.z);
          const uint2 m = KIND == H2_K_EXP ? expk_fixed52(r2, tab, lane8)
                                           : helm_eval<SliceFmt<NS>::HEXP>(r2, hs, ovf, tab, lane);
          lo[k][q] = m.x;
          hi[k][q] = m.y;
        }
      }
      }
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        uint32_t w[4][4];
        transpose4(lo[k][0], lo[k][1], lo[k][2], lo[k][3], w[0]);
        transpose4(lo[k][4], lo[k][5], lo[k][6], lo[k][7], w[1]);
        transpose4(hi[k][0], hi[k][1], hi[k][2], hi[k][3], w[2]);
        transpose4(hi[k][4], hi[k][5], hi[k][6], hi[k][7], w[3]);
        // slice s at s SLICE, or (PACK) pair s % 3, half s / 3 (64 rows x 16 B per k group)
        auto sa = [&](int sl) {
          if (PACK7 && sl == 6) return 6 * P::SLICE + off6d;
          return (PACK || PACK7) ? (sl % 3) * 2 * P::SLICE + (sl / 3) * TM * 16 : sl * P::SLICE;
        };
#pragma unroll
        for (int s = 0; s < 4; ++s)
          *reinterpret_cast<uint2*>(Ab + sa(s) + off[k]) = make_uint2(w[0][s], w[1][s]);
#pragma unroll
        for (int s = 0; s < NS - 4; ++s)
          *reinterpret_cast<uint2*>(Ab + sa(s + 4) + off[k]) = make_uint2(w[2][s], w[3][s]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar_full + 8 * buf));

      const bool drain = ((it % P::DRAIN) == P::DRAIN - 1) || (it == nch - 1);
      // near-field mode: its only drain is the final one (a few chunks per CTA), and every producer
      // warp has finished -- all NPW / 4 warp quartets drain, each a quarter of the column groups
      // (the same per-entry arithmetic; the A buffers, idle after the last MMA, hold the hand-off)
      constexpr int NREP = (nearm && NPW % 4 == 0) ? NPW / 4 : 1;
      const bool all_drain = NREP > 1 && it == nch - 1;
      if (PACK && drain && (warp < 4 || all_drain)) {
        mbar_wait(bar_drain, drains & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        // lane 32 w + l: row 32 (w & 1) + l; warps 0-1 hold slices 0-2 (pairs' low halves), warps
        // 2-3 slices 3-5.  Chains (s0..s2) and (s3..s5) as in the other shapes; the high warps hand
        // theirs to the low warps through the coordinate slot of this chunk (consumed, and not
        // refilled before chunk it + 4), 8 columns at a time.
        const int wq = warp & 3, rep = all_drain ? warp >> 2 : 0;
        const int i_stride = all_drain ? 8 * NREP : 8;
        const int64_t i = rtile + 32 * (wq & 1) + lane;
        const bool high = wq >= 2;
        double* xb = all_drain ? reinterpret_cast<double*>(smem + P::A0) + rep * 512 + (32 * (wq & 1) + lane) * 8
                               : reinterpret_cast<double*>(smem + P::C0 + slot * CBUF) + (32 * (warp & 1) + lane) * 8;
        double* y = Yo + (i - row0) * ldy;
#pragma unroll 1
        for (int c0 = 8 * rep; c0 < NCOL; c0 += i_stride) {
          double v[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = 0.0;
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            uint32_t r[8];
            const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(p * NCOL + c0);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                           "=r"(r[7])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
            const double wgt = ldexp(1.0, 8 * (p + (high ? 3 : 0)) + wshift);
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = fma((double)(int)r[c], wgt, v[c]);
          }
          if (high) {
#pragma unroll
            for (int c = 0; c < 8; ++c) xb[c] = v[c];
          }
          asm volatile("bar.sync %0, 128;\n" ::"r"(1 + rep));
          if (!high && i < row1) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const double t = v[c] + xb[c];
              if (c0 + c < ncols) y[c0 + c] = nearm ? y[c0 + c] - t : drains == 0 ? t : y[c0 + c] + t;
            }
          }
          asm volatile("bar.sync %0, 128;\n" ::"r"(1 + rep));
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      } else if (PACK7 && drain && warp < 4) {
        mbar_wait(bar_drain, drains & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        // pairs: lane 32 w + l holds row 32 (w & 1) + l, slices 0-2 (w < 2) or 3-5 (w >= 2); the
        // top slice (M = 64 layout) holds row 16 w + l in lanes l < 16.  Chains (s0..s2) and
        // (s3..s6): the top slice goes to the high warps and their chain to the low warps through
        // the consumed coordinate slot of this chunk, 4 columns at a time.
        const int row = 32 * (warp & 1) + lane;
        const int64_t i = rtile + row;
        const bool high = warp >= 2;
        int32_t* xs6 = reinterpret_cast<int32_t*>(smem + P::C0 + slot * CBUF);   // 64 x 4 int32
        double* xu = reinterpret_cast<double*>(smem + P::C0 + slot * CBUF + 64 * 4 * 4);   // 64 x 4
        double* y = Yo + (i - row0) * ldy;
#pragma unroll 1
        for (int c0 = 0; c0 < NCOL; c0 += 4) {
          uint32_t r6[4];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                       : "=r"(r6[0]), "=r"(r6[1]), "=r"(r6[2]), "=r"(r6[3])
                       : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(3 * NCOL + c0)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
          if (lane < 16) {
#pragma unroll
            for (int c = 0; c < 4; ++c) xs6[(16 * warp + lane) * 4 + c] = (int32_t)r6[c];
          }
          double v[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) v[c] = 0.0;
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            uint32_t r[4];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                         : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(p * NCOL + c0)));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
            const double wgt = ldexp(1.0, 8 * (p + (high ? 3 : 0)) + wshift);
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] = fma((double)(int)r[c], wgt, v[c]);
          }
          asm volatile("bar.sync 1, 128;\n" ::);
          if (high) {
            const double w6 = ldexp(1.0, 8 * 6 + wshift);
#pragma unroll
            for (int c = 0; c < 4; ++c) xu[row * 4 + c] = fma((double)xs6[row * 4 + c], w6, v[c]);
          }
          asm volatile("bar.sync 1, 128;\n" ::);
          if (!high && i < row1) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double t = v[c] + xu[row * 4 + c];
              if (c0 + c < ncols) y[c0 + c] = nearm ? y[c0 + c] - t : drains == 0 ? t : y[c0 + c] + t;
            }
          }
          asm volatile("bar.sync 1, 128;\n" ::);
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      } else if (drain && warp < 4) {
        mbar_wait(bar_drain, drains & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        // TM = 128: lane l of warp w holds row 32 w + l, all slices.
        // TM = 64 : lanes l < 16 hold row 16 w + l (slices 0-2), lanes 16 + l the same row
        //           (slices 3..NS-1); the halves are summed with one shuffle.
        // Every shape sums the slices as (s0..s2 chain) + (s3..s{NS-1} chain), so the sketch is
        // bitwise independent of the pass width.
        const int64_t i = TM == 128 ? rtile + warp * 32 + lane : rtile + warp * 16 + (lane & 15);
        const bool writer = TM == 128 || lane < 16;
        double* y = Yo + (i - row0) * ldy;
#pragma unroll 1
        for (int c0 = 0; c0 < NCOL; c0 += 16) {   // 16 columns at a time (register budget)
          double v[16], u[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = u[c] = 0.0;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            if (TM == 64 && s >= (NS - NSPLIT > NSPLIT ? NS - NSPLIT : NSPLIT)) break;
            uint32_t r[16];
            // TM = 64: column s NCOL holds slice s (low lanes, s < NSPLIT) and slice s + NSPLIT (high)
            const uint32_t col = TM == 64 ? (uint32_t)(s * NCOL) : tmem_slice<TM, NCOL, NS>(s);
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + col + (uint32_t)c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];\n"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
            // slice weight 2^(8 sl) * 2^-KEXP * (1/4); at TM = 64 the high lanes hold slice s + NSPLIT
            const int sl = (TM == 128 || lane < 16) ? s : s + NSPLIT;
            const bool valid = (TM == 128 || lane >= 16) ? sl < NS : s < NSPLIT;
            const double wgt = valid ? ldexp(1.0, 8 * sl + wshift) : 0.0;
            if (TM == 128 && s >= NSPLIT) {
#pragma unroll
              for (int c = 0; c < 16; ++c) u[c] = fma((double)(int)r[c], wgt, u[c]);
            } else {
#pragma unroll
              for (int c = 0; c < 16; ++c) v[c] = fma((double)(int)r[c], wgt, v[c]);
            }
          }
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] += (TM == 64) ? __shfl_xor_sync(0xffffffffu, v[c], 16) : u[c];
          if (writer && i < row1) {
#pragma unroll
            for (int c = 0; c < 16; ++c)
              if (c0 + c < ncols) y[c0 + c] = nearm ? y[c0 + c] - v[c] : drains == 0 ? v[c] : y[c0 + c] + v[c];
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      }
      if (drain) ++drains;
    }
    if (KIND != H2_K_EXP && ovf) atomicOr(ovf_flag, 1u);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
}


// ------------------------------------------------------------------------------------------
// CTA-pair variant of the 128-column pass (cta_group::2): two CTAs of
// a cluster own adjacent 64-row tiles and the same j range; the leader issues
// tcgen05.mma.cta_group::2 with M = 128 (64 rows per SM) x N = 128 x K = 32, whose A operand is
// each CTA's own K slices and whose B operand is split by columns (CTA r holds Omega columns
// [64 r, 64 r + 64) of the chunk).  Each SM's 64 x 128 accumulator of a slice occupies all 128
// TMEM lanes x 64 columns (lanes 64 h + m: row m, columns [64 h, 64 h + 64)), 7 slices in 448
// columns, and an M = 128 dispatch runs the tensor core at its full rate (an M = 64 single-CTA
// dispatch costs the same cycles for half the rows).  Producers, ring and drain as above; the
// peer's producers arrive on the leader's full barrier (cluster scope) and the MMA completion is
// multicast to the empty / drain barriers of both CTAs.
// ------------------------------------------------------------------------------------------
constexpr int PR_TM = 64, PR_NCOL = 128, PR_NH = 64, PR_JC = 128;
template <int NS>
struct PairPlan {
  static constexpr int SLICE = PR_TM * PR_JC;              // 8 KB
  static constexpr int ABUF = NS * SLICE;                  // 56 / 48 KB
  static constexpr int NA = 2;
  static constexpr int BBUF = PR_NH * PR_JC;               // this CTA's half of B: 8 KB
  static constexpr int CBUF = PR_JC * 32 + PR_JC * 2;
  static constexpr int DRAIN = TC_DRAIN_J / PR_JC;
  static constexpr int A0 = 0;
  static constexpr int B0 = NA * ABUF;
  static constexpr int C0 = B0 + TC_NB * BBUF;
  static constexpr int BAR = C0 + TC_NB * CBUF;
  static constexpr int TOTAL = BAR + 8 * (2 * NA + TC_NB + 1) + 16;
  static_assert(TOTAL + 16 * 256 * 8 <= 227 * 1024, "shared memory plan exceeds 227 KB");
};

__device__ __forceinline__ void mbar_wait_cluster(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITC_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAITC_%=;\n}\n" ::"r"(addr),
      "r"(parity));
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::);
}

template <int KIND, int NPW, int NS>
__global__ void __launch_bounds__(32 * (NPW + 1), 1)
    sketch_tc_pair_kernel(const double4* __restrict__ C, int64_t n, int64_t row0, int64_t row1,
                          const int8_t* __restrict__ Bq, int64_t nchunks, int ncols, double* __restrict__ Yout,
                          int64_t ldy, int64_t split_stride, double hs, int wshift, uint32_t* __restrict__ ovf_flag) {
  using P = PairPlan<NS>;
  constexpr int NSPLIT = SliceFmt<NS>::NSPLIT;
  constexpr int TM = PR_TM, JC = PR_JC;
  constexpr int G = JC / 16;
  constexpr int CBUF = P::CBUF;
  constexpr int NA = P::NA;
  constexpr int RPT = TM * G / (16 * NPW);
  constexpr int BBUF = P::BBUF;
  constexpr int LBO_A = TM * 16;
  constexpr int LBO_B = PR_NH * 16;
  constexpr uint32_t IDESC = idesc_i8<128, PR_NCOL>();   // M = 128 over the CTA pair
  constexpr uint32_t IDESC6 = KIND == H2_K_EXP ? IDESC : (IDESC | (1u << 7));
  static_assert(RPT >= 1 && NPW % G == 0 && TM * JC == RPT * 32 * NPW * 8, "producer tiling");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(128) double tab[16 * 256];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bar_full = sbase + P::BAR;
  const uint32_t bar_empty = bar_full + 8 * NA;
  const uint32_t bar_loaded = bar_empty + 8 * NA;
  const uint32_t bar_drain = bar_loaded + 8 * TC_NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P::BAR + 8 * (2 * NA + TC_NB + 1));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
  const bool leader = crank == 0;
  const int64_t rtile = row0 + (int64_t)blockIdx.x * TM;
  const int64_t nunits = nchunks / (128 / JC);
  const int64_t ch_b = nunits * blockIdx.y / gridDim.y * (128 / JC);
  const int64_t ch_e = nunits * (blockIdx.y + 1) / gridDim.y * (128 / JC);
  const int nch = (int)(ch_e - ch_b);
  const bool control = (warp == NPW);
  const int8_t* Bh = Bq + (int64_t)crank * nchunks * BBUF;   // this CTA's column half

  if (KIND == H2_K_HELMHOLTZ && H2_TC_HTAB) fill_cs_table(tab, tid, 32 * (NPW + 1));
  else
    for (int e = tid; e < 16 * 256; e += 32 * (NPW + 1)) tab[e] = exp2((double)(e >> TC_TAB_SHIFT) * TC_TAB_STEP + (double)SliceFmt<NS>::KEXP);
  if (tid == 0) {
    for (int b = 0; b < NA; ++b) {
      mbar_init(bar_full + 8 * b, leader ? 2 * NPW : NPW);   // leader: both CTAs' producers
      mbar_init(bar_empty + 8 * b, 1);
    }
    for (int q = 0; q < TC_NB; ++q) mbar_init(bar_loaded + 8 * q, 32);
    mbar_init(bar_drain, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  cluster_sync_all();   // peer barriers initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;
  double* Yo = Yout + blockIdx.y * split_stride;

  if (control) {
    auto prefetch = [&](int it) {
      if (it >= nch) return;
      const int64_t t = ch_b + it;
      const int slot = it & (TC_NB - 1);
#pragma unroll
      for (int q = 0; q < BBUF / 16 / 32; ++q) {
        const int e = lane + 32 * q;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + P::B0 + slot * BBUF + e * 16),
                     "l"(Bh + t * BBUF + e * 16));
      }
#pragma unroll
      for (int q = 0; q < JC / 16; ++q) {
        const int e = lane + 32 * q;
        const int jc = e >> 1;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + P::C0 + slot * CBUF + e * 16 +
                                                                          (jc >> 3) * 16),
                     "l"(reinterpret_cast<const char*>(C + t * JC) + e * 16));
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar_loaded + 8 * slot));
    };
    prefetch(0);
    prefetch(1);
    for (int it = 0; it < nch; ++it) {
      const int buf = it % NA;
      const int slot = it & (TC_NB - 1);
      // full(it): both CTAs' producers (leader) / this CTA's producers (peer) finished chunk it,
      // hence MMA(it - 2) completed and ring slot (it + 2) % 4 is free in this CTA
      mbar_wait_cluster(bar_full + 8 * buf, (it / NA) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      if (leader && lane == 0) {
        const bool first = (it % P::DRAIN) == 0;
        const bool drain = ((it % P::DRAIN) == P::DRAIN - 1) || (it == nch - 1);
        const uint32_t a0 = sbase + P::A0 + buf * P::ABUF;
        const uint32_t b0 = sbase + P::B0 + slot * BBUF;
#pragma unroll
        for (int sl = 0; sl < NS; ++sl)
#pragma unroll
          for (int kk = 0; kk < JC / 32; ++kk) {
            const uint64_t ad = umma_desc(a0 + sl * P::SLICE + kk * 2 * LBO_A, LBO_A, 128);
            const uint64_t bd = umma_desc(b0 + kk * 2 * LBO_B, LBO_B, 128);
            const uint32_t acc = (first && kk == 0) ? 0u : 1u;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)(sl * PR_NH)),
                "l"(ad), "l"(bd), "r"(sl == NS - 1 ? IDESC6 : IDESC), "r"(acc));
          }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                bar_empty + 8 * buf),
            "h"((uint16_t)3));
        if (drain)
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                  bar_drain),
              "h"((uint16_t)3));
      }
      __syncwarp();
      prefetch(it + 2);
    }
  } else {
    const int g = warp % G;
    const int rs = warp / G;
    const int h = lane & 1;
    const int r0 = 16 * rs + (lane >> 1);
    double4 ci[RPT];
    int off[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = r0 + k * 16 * (NPW / G);
      ci[k] = C[(rtile + r < row1) ? (rtile + r) : (row1 - 1)];
      off[k] = g * LBO_A + (r >> 3) * 128 + (r & 7) * 16 + 8 * h;
    }
    uint32_t full_remote = 0;
    if (!leader)
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(full_remote) : "r"(bar_full), "r"(0));
    const uint32_t lane8 = tc_lane8(lane);
    uint32_t ovf = 0;
    int drains = 0;
    for (int it = 0; it < nch; ++it) {
      const int buf = it % NA;
      const int slot = it & (TC_NB - 1);
      mbar_wait(bar_loaded + 8 * slot, (it / TC_NB) & 1);
      if (it >= NA) mbar_wait(bar_empty + 8 * buf, ((it - NA) / NA) & 1);
      const uint8_t* cb = smem + P::C0 + slot * CBUF;
      uint8_t* Ab = smem + P::A0 + buf * P::ABUF;
      const int jj0 = 16 * g + 8 * h;
      uint32_t lo[RPT][8], hi[RPT][8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int jj = jj0 + q;
        const double4 p = *reinterpret_cast<const double4*>(cb + jj * 32 + (jj >> 3) * 16);
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const double r2 = dist2_floor(ci[k].x, ci[k].y, ci[k].z, p.x, p.y, p.z);
          const uint2 m = KIND == H2_K_EXP ? expk_fixed52(r2, tab, lane8)
                                           : helm_eval<SliceFmt<NS>::HEXP>(r2, hs, ovf, tab, lane);
          lo[k][q] = m.x;
          hi[k][q] = m.y;
        }
      }
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        uint32_t w[4][4];
        transpose4(lo[k][0], lo[k][1], lo[k][2], lo[k][3], w[0]);
        transpose4(lo[k][4], lo[k][5], lo[k][6], lo[k][7], w[1]);
        transpose4(hi[k][0], hi[k][1], hi[k][2], hi[k][3], w[2]);
        transpose4(hi[k][4], hi[k][5], hi[k][6], hi[k][7], w[3]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint2*>(Ab + q * P::SLICE + off[k]) = make_uint2(w[0][q], w[1][q]);
#pragma unroll
        for (int q = 0; q < NS - 4; ++q)
          *reinterpret_cast<uint2*>(Ab + (q + 4) * P::SLICE + off[k]) = make_uint2(w[2][q], w[3][q]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::);
      __syncwarp();
      if (lane == 0) {
        asm volatile("mbarrier.arrive.release.cluster.shared::cta.b64 _, [%0];\n" ::"r"(bar_full + 8 * buf));
        if (!leader)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(full_remote + 8 * buf));
      }

      const bool drain = ((it % P::DRAIN) == P::DRAIN - 1) || (it == nch - 1);
      if (drain && warp < 4) {
        mbar_wait(bar_drain, drains & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        // lane 32 w + l holds row 32 (w & 1) + l, columns [64 (w >> 1), +64), all 7 slices at
        // columns 64 s; summed as (s0..s3 chain) + (s4..s6 chain) like the other pass shapes
        const int64_t i = rtile + 32 * (warp & 1) + lane;
        const int ch = 64 * (warp >> 1);
        double* y = Yo + (i - row0) * ldy + ch;
#pragma unroll 1
        for (int c0 = 0; c0 < PR_NH; c0 += 8) {   // 8 columns at a time (register budget)
          double v[8], u[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = u[c] = 0.0;
#pragma unroll
          for (int sl = 0; sl < NS; ++sl) {
            uint32_t r[8];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(sl * PR_NH + c0);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                           "=r"(r[7])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
            const double wgt = ldexp(1.0, 8 * sl + wshift);
            if (sl >= NSPLIT) {
#pragma unroll
              for (int c = 0; c < 8; ++c) u[c] = fma((double)(int)r[c], wgt, u[c]);
            } else {
#pragma unroll
              for (int c = 0; c < 8; ++c) v[c] = fma((double)(int)r[c], wgt, v[c]);
            }
          }
          if (i < row1) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int col = ch + c0 + c;
              if (col < ncols) y[c0 + c] = drains == 0 ? v[c] + u[c] : y[c0 + c] + (v[c] + u[c]);
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      }
      if (drain) ++drains;
    }
    if (KIND != H2_K_EXP && ovf) atomicOr(ovf_flag, 1u);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  cluster_sync_all();   // no CTA leaves while its peer may still arrive or MMA into it
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

}  // namespace

// exp: a point set whose scaled diameter keeps n = rint(-256 r'/ln2) in the range of the exponent
// arithmetic of expk_fixed52 (r' <= 650; K < 1e-282 there, far below the 2^-53 grid).
// Helmholtz: a known minimum point distance (the fixed-point scale) and r' = k r <= 650.
bool sketch_tc_supported(const KernelParams& kp) {
  if (kp.kind == H2_K_EXP) return kp.rmax > 0 && kp.rmax <= 650.0;
  return kp.kind == H2_K_HELMHOLTZ && kp.rmax > 0 && kp.rmax <= 650.0 && kp.rmin > 0;
}

// CTA-pair (cta_group::2) 128-column pass, opt-in (H2_TC_PAIR=1): bitwise identical, but 200 vs
// 178 ms per 128 columns at N = 2^18 (the full-rate M = 128 dispatch does not pay: the pass is
// not bound by the tensor-core rate, and the pair couples two CTAs' producers per chunk)
bool sketch_tc_pair() {
  return env_int("H2_TC_PAIR", 0) != 0;
}

// byte slices of the fixed-point K (SliceFmt): exp 6 (H2_TC_SLICES=7: 7); Helmholtz 7 (its scale
// 2^E >= 4 max|K| leaves 2^-45 max|K| per entry at 6 slices, above the FP64-GEMM-level bound)
int sketch_tc_slices(int kind) {
  if (kind != H2_K_EXP) return 7;
  return env_int("H2_TC_SLICES", 6) == 7 ? 7 : 6;
}

// widest pass: 160 columns with 6 slices (3 x 160 TMEM columns per lane half), 128 with 7;
// H2_TC_WIDE=0: 64
int sketch_tc_pass_cols(int kind) {
  const char* e = getenv("H2_TC_WIDE");
  if (e && atoi(e) == 0) return 64;
  return sketch_tc_slices(kind) == 6 ? 160 : 128;
}

namespace {
template <int KIND, int TM, int NCOL, int JC, int NS, bool NEARM = false>
void tc_launch(dim3 grid, cudaStream_t st, const double4* C, int64_t n, int64_t row0, int64_t row1, const int8_t* Bq,
               int64_t nchunks, int nc, double* yo, int64_t ld, int64_t sstride, double hs, int wshift, uint32_t* ovf,
               const double* Aop = nullptr, int64_t lda = 0, const int32_t* nl_ptr = nullptr,
               const int32_t* nl_chunk = nullptr, const uint8_t* nl_mask = nullptr) {
  // producer warps: 16 (8 measured slower: 170 vs 163 ms at 32 columns, 180 vs 172 at 128; 32
  // would exceed 1024 threads per CTA with the control warp)
  constexpr int smem = TcPlan<TM, NCOL, JC, NS>::TOTAL;
  static const int pfd = env_int("H2_TC_PF", 2) == 3 ? 3 : 2;   // cp.async ring prefetch distance
  static const uint32_t hint = (uint32_t)env_int("H2_TC_HINT", 0); // mbarrier wait suspend hint (ns), 0 = none
  constexpr int NPW = 16;
  // per launch: the attribute is per device (a process may drive several GPUs)
  H2_CUDA(cudaFuncSetAttribute(sketch_tc_kernel<KIND, TM, NPW, NCOL, JC, NS, NEARM>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  sketch_tc_kernel<KIND, TM, NPW, NCOL, JC, NS, NEARM><<<grid, 32 * (NPW + 1), smem, st>>>(C, n, row0, row1, Bq, nchunks, nc,
                                                                                    yo, ld, sstride, hs, wshift, ovf, pfd, hint,
                                                                                    Aop, lda, nl_ptr, nl_chunk, nl_mask);
}

template <int KIND, int NS>
void tc_launch_pair(dim3 grid, cudaStream_t st, const double4* C, int64_t n, int64_t row0, int64_t row1,
                    const int8_t* Bq, int64_t nchunks, int nc, double* yo, int64_t ld, int64_t sstride, double hs,
                    int wshift, uint32_t* ovf) {
  constexpr int NPW = 16;
  constexpr int smem = PairPlan<NS>::TOTAL;
  H2_CUDA(cudaFuncSetAttribute(sketch_tc_pair_kernel<KIND, NPW, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(32 * (NPW + 1));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  H2_CUDA(cudaLaunchKernelEx(&cfg, sketch_tc_pair_kernel<KIND, NPW, NS>, C, n, row0, row1, Bq, nchunks, nc, yo, ld,
                             sstride, hs, wshift, ovf));
}

template <int KIND, int NS>
void tc_dispatch(int NCOL, dim3 grid, cudaStream_t st, const double4* C, int64_t n, int64_t row0, int64_t row1,
                 const int8_t* Bq, int64_t nchunks, int nc, double* yo, int64_t ld, int64_t ss, double hs, int wshift,
                 uint32_t* ovf, const double* Aop = nullptr, int64_t lda = 0) {
  if constexpr (NS == 6) {
    if (NCOL == 160) {
      tc_launch<KIND, 64, 160, 128, NS>(grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
      return;
    }
  }
  if (NCOL == 128)
    tc_launch<KIND, 64, 128, 128, NS>(grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf, Aop, lda);
  else if (NCOL == 64)
    tc_launch<KIND, 128, 64, 64, NS>(grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf, Aop, lda);
  else
    tc_launch<KIND, 128, 32, 64, NS>(grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf, Aop, lda);
}

// j-split S fills the last wave (1 CTA / SM)
int pick_split(int tiles, int64_t nunits, int sms) {
  int S = 1;
  double best = 0;
  for (int s = 1; s <= 4; ++s) {
    if (s > 1 && nunits / s < 32) break;
    const int64_t units = (int64_t)tiles * s;
    const double eff = (double)units / ((double)sms * ((units + sms - 1) / sms)) - 0.01 * (s - 1);
    if (eff > best + 1e-9) {
      best = eff;
      S = s;
    }
  }
  return S;
}
}  // namespace

// Omega columns are processed sketch_tc_pass_cols() at a time: a pass of more than 64 columns
// runs the 64-row / 128-column kernel (K evaluated once per 128 columns), narrower passes the
// 128-row kernel with 32 or 64 columns.  Returns false if a Helmholtz entry overflowed the
// fixed-point scale (the caller then recomputes on the FP64 DMMA path).
bool launch_dense_sketch_tc(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, int64_t n,
                            int64_t row0, int64_t row1, const double* Om, int64_t ldo, int ncols, double* Yout,
                            int64_t ldy, cudaStream_t st) {
  if (row1 <= row0 || ncols <= 0) return true;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int wmax = sketch_tc_pass_cols(kp.kind);
  const int64_t npad = ((n + 127) / 128) * 128;   // 128-j units: every chunk shape tiles it
  const int64_t rows = row1 - row0;
  const bool helm = kp.kind == H2_K_HELMHOLTZ;
  // Helmholtz scale 2^E >= 4 max|K| (max|K| <= 1 / r_min): hs = k / 2^E, slice weight
  // 2^(8s) 2^E 2^-51 / 4; exp: K in (0, 1], weight 2^(8s) 2^-52 / 4
  const int E = helm ? (int)std::ceil(std::log2(1.0 / kp.rmin)) + 2 : 0;
  const double hs = helm ? std::ldexp(kp.param, -E) : 0.0;
  const int NS = sketch_tc_slices(kp.kind);
  // slice weight 2^(8 s) x 2^-KEXP / 4 (exp) or 2^E 2^-HEXP / 4 (Helmholtz)
  const int wshift = helm ? E - (NS == 7 ? 51 : 46) - 2 : -(NS == 7 ? 52 : 47) - 2;
  double4* C = static_cast<double4*>(cache_alloc(sizeof(double4) * npad, st));
  int8_t* Bq = static_cast<int8_t*>(cache_alloc((size_t)npad * 160, st));
  uint32_t* ovf = static_cast<uint32_t*>(cache_alloc(sizeof(uint32_t), st));
  H2_CUDA(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), st));
  double* part = nullptr;
  int64_t part_elems = 0;
  coords_aos_kernel<<<(int)std::min<int64_t>((npad + 255) / 256, (int64_t)sms * 16), 256, 0, st>>>(
      X, Yc, Zc, n, npad, helm ? kp.param : kp.inv, C);
  H2_CHECK_LAUNCH();
  for (int c0 = 0; c0 < ncols; c0 += wmax) {
    const int nc = std::min(wmax, ncols - c0);
    const int NCOL = nc > 128 ? 160 : nc > 64 ? 128 : nc > 32 ? 64 : 32;
    const int TM = NCOL >= 128 ? 64 : 128;
    const int JC = NCOL >= 128 ? 128 : 64;
    const int64_t nchunks = npad / JC;
    const int tiles = div_up(rows, TM);
    // the split is chosen from n only -- for the row shard of the largest rank count of one box
    // (8 GPUs: its 64-row tiles fill the waves there; one GPU just runs more waves) -- and shared
    // by all pass shapes and row shards: bitwise identical sketches for any P <= 8
    const int S = pick_split(div_up(n, 64 * 8), npad / 128, sms);
    if (S > 1 && part_elems < rows * nc * S) {
      if (part) cache_free(part, st);
      part_elems = rows * nc * S;
      part = static_cast<double*>(cache_alloc(sizeof(double) * part_elems, st));
    }
    const bool pair = NCOL == 128 && sketch_tc_pair();
    double* yo = S > 1 ? part : Yout + c0;
    const int64_t ld = S > 1 ? nc : ldy;
    const int64_t ss = S > 1 ? rows * nc : 0;
    if (pair) {
      // B split by columns: halves [0, 64) and [64, nc) packed as two 64-column operands
      for (int hlf = 0; hlf < 2; ++hlf) {
        const int nch = std::max(0, std::min(64, nc - 64 * hlf));
        omega_i8_kernel<<<(int)std::min<int64_t>((nchunks * JC * 64 + 255) / 256, (int64_t)sms * 32), 256, 0, st>>>(
            Om + c0 + 64 * hlf, ldo, n, nch, 64, JC, nchunks, Bq + (int64_t)hlf * nchunks * JC * 64);
        H2_CHECK_LAUNCH();
      }
      const dim3 grid((unsigned)(2 * div_up(tiles, 2)), S);   // CTA pairs along x
      if (NS == 7) {
        if (helm) tc_launch_pair<H2_K_HELMHOLTZ, 7>(grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
        else tc_launch_pair<H2_K_EXP, 7>(grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
      } else {
        if (helm) tc_launch_pair<H2_K_HELMHOLTZ, 6>(grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
        else tc_launch_pair<H2_K_EXP, 6>(grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
      }
    } else {
      omega_i8_kernel<<<(int)std::min<int64_t>((nchunks * JC * NCOL + 255) / 256, (int64_t)sms * 32), 256, 0, st>>>(
          Om + c0, ldo, n, nc, NCOL, JC, nchunks, Bq);
      H2_CHECK_LAUNCH();
      const dim3 grid(tiles, S);
      if (NS == 7) {
        if (helm) tc_dispatch<H2_K_HELMHOLTZ, 7>(NCOL, grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
        else tc_dispatch<H2_K_EXP, 7>(NCOL, grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
      } else {
        if (helm) tc_dispatch<H2_K_HELMHOLTZ, 6>(NCOL, grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
        else tc_dispatch<H2_K_EXP, 6>(NCOL, grid, st, C, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift, ovf);
      }
    }
    H2_CHECK_LAUNCH();
    if (S > 1) launch_sketch_combine(part, S, rows, nc, Yout + c0, ldy, st);
  }
  uint32_t h_ovf = 0;
  if (helm) {
    H2_CUDA(cudaMemcpyAsync(&h_ovf, ovf, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    H2_CUDA(cudaStreamSynchronize(st));
  }
  cache_free(C, st);
  cache_free(Bq, st);
  cache_free(ovf, st);
  if (part) cache_free(part, st);
  return h_ovf == 0;
}

// Near-field product on the tensor cores (the leaf subtraction of Algorithm 1, fused with the
// entry evaluation: SURVEY §8(a) a3+a4): Y(rows) -= sum_{b in N(leaf)} K(rows, I_b) Omega(I_b, :)
// with the same fixed-point K and exact int8 contraction as the dense sketch, over each leaf's near
// leaves only (nl_*: per leaf, the 128-j chunks holding its near leaves and a 2-bit mask of the
// 64-j halves).  Requires leaves of exactly 64 points at multiples of 64 (row tiles = leaves) and a
// 128- or 160-column pass (64-row tiles); ncols <= sketch_tc_pass_cols.  Returns false on a
// Helmholtz scale overflow (the caller then uses the BSR path).
bool launch_near_sketch_tc(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, int64_t n,
                           int64_t row0, int64_t row1, const double* Om, int64_t ldo, int ncols, double* Y, int64_t ldy,
                           const int32_t* nl_ptr, const int32_t* nl_chunk, const uint8_t* nl_mask, cudaStream_t st) {
  if (row1 <= row0 || ncols <= 0) return true;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t npad = ((n + 127) / 128) * 128;
  const bool helm = kp.kind == H2_K_HELMHOLTZ;
  const int E = helm ? (int)std::ceil(std::log2(1.0 / kp.rmin)) + 2 : 0;
  const double hs = helm ? std::ldexp(kp.param, -E) : 0.0;
  const int NS = sketch_tc_slices(kp.kind);
  const int wshift = helm ? E - (NS == 7 ? 51 : 46) - 2 : -(NS == 7 ? 52 : 47) - 2;
  const int NCOL = ncols > 128 ? 160 : 128;
  double4* C = static_cast<double4*>(cache_alloc(sizeof(double4) * npad, st));
  int8_t* Bq = static_cast<int8_t*>(cache_alloc((size_t)npad * 160, st));
  uint32_t* ovf = static_cast<uint32_t*>(cache_alloc(sizeof(uint32_t), st));
  H2_CUDA(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), st));
  coords_aos_kernel<<<(int)std::min<int64_t>((npad + 255) / 256, (int64_t)sms * 16), 256, 0, st>>>(
      X, Yc, Zc, n, npad, helm ? kp.param : kp.inv, C);
  H2_CHECK_LAUNCH();
  const int64_t nchunks = npad / 128;
  omega_i8_kernel<<<(int)std::min<int64_t>((nchunks * 128 * NCOL + 255) / 256, (int64_t)sms * 32), 256, 0, st>>>(
      Om, ldo, n, ncols, NCOL, 128, nchunks, Bq);
  H2_CHECK_LAUNCH();
  const dim3 grid((unsigned)div_up(row1 - row0, 64), 1);
  if (NS == 6 && NCOL == 160) {
    tc_launch<H2_K_EXP, 64, 160, 128, 6, true>(grid, st, C, n, row0, row1, Bq, nchunks, ncols, Y, ldy, 0, hs, wshift,
                                               ovf, nullptr, 0, nl_ptr, nl_chunk, nl_mask);
  } else if (NS == 6) {
    tc_launch<H2_K_EXP, 64, 128, 128, 6, true>(grid, st, C, n, row0, row1, Bq, nchunks, ncols, Y, ldy, 0, hs, wshift,
                                               ovf, nullptr, 0, nl_ptr, nl_chunk, nl_mask);
  } else if (helm) {
    tc_launch<H2_K_HELMHOLTZ, 64, 128, 128, 7, true>(grid, st, C, n, row0, row1, Bq, nchunks, ncols, Y, ldy, 0, hs,
                                                     wshift, ovf, nullptr, 0, nl_ptr, nl_chunk, nl_mask);
  } else {
    tc_launch<H2_K_EXP, 64, 128, 128, 7, true>(grid, st, C, n, row0, row1, Bq, nchunks, ncols, Y, ldy, 0, hs, wshift,
                                               ovf, nullptr, 0, nl_ptr, nl_chunk, nl_mask);
  }
  H2_CHECK_LAUNCH();
  uint32_t h_ovf = 0;
  if (helm) {
    H2_CUDA(cudaMemcpyAsync(&h_ovf, ovf, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    H2_CUDA(cudaStreamSynchronize(st));
  }
  cache_free(C, st);
  cache_free(Bq, st);
  cache_free(ovf, st);
  return h_ovf == 0;
}

// ------------------------------------------------------------------------------------------
// Explicit dense operator on the int8 tensor cores (H2_S_DENSE_MATRIX):
// Y(rows) = A(rows, :) Omega for the h2 Omega stream.  A (row-major, lda, tree order) is read
// once per pass of up to 128 columns and converted to the 7-slice signed fixed point of scale
// 2^E >= max|A| (dense_fixed); the contraction is exact in int32 TMEM accumulators, so the only
// rounding is the grid (<= 2^-52 max|A| per entry) and the FP64 drains -- the normwise error
// level of an FP64 GEMM.  HBM-bound (8 bytes per entry per pass) instead of DGEMM-bound.
// ------------------------------------------------------------------------------------------
__global__ void absmax_kernel(const double* __restrict__ A, int64_t lda, int64_t n, unsigned long long* out) {
  double m = 0.0;
  // one row per CTA iteration, 4 independent loads in flight per thread
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double* a = A + i * lda;
    for (int64_t j = threadIdx.x; j < n; j += 4 * blockDim.x) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = j + u * blockDim.x < n ? fabs(__ldg(a + j + u * blockDim.x)) : 0.0;
      m = fmax(m, fmax(fmax(v[0], v[1]), fmax(v[2], v[3])));
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));   // m >= 0: bit order
}

double dense_absmax(const double* A, int64_t lda, int64_t n, cudaStream_t st) {
  unsigned long long* d = static_cast<unsigned long long*>(cache_alloc(8, st));
  H2_CUDA(cudaMemsetAsync(d, 0, 8, st));
  absmax_kernel<<<148 * 8, 256, 0, st>>>(A, lda, n, d);
  H2_CHECK_LAUNCH();
  unsigned long long h = 0;
  H2_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st));
  H2_CUDA(cudaStreamSynchronize(st));
  cache_free(d, st);
  double v;
  std::memcpy(&v, &h, 8);
  return v;
}

void launch_dense_op_tc(const double* A, int64_t lda, int64_t n, int64_t row0, int64_t row1, double amax,
                        const double* Om, int64_t ldo, int ncols, double* Yout, int64_t ldy, cudaStream_t st) {
  if (row1 <= row0 || ncols <= 0) return;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t npad = ((n + 127) / 128) * 128;
  const int64_t rows = row1 - row0;
  // scale 2^E >= max|A|: v = A 2^-E in [-1, 1]; slice weight 2^(8 s) 2^E 2^-51 / 4
  const int E = amax > 0 ? (int)std::ceil(std::log2(amax)) : 0;
  const double hs = std::ldexp(1.0, -E);
  const int wshift = E - 51 - 2;
  int8_t* Bq = static_cast<int8_t*>(cache_alloc((size_t)npad * 128, st));
  uint32_t* ovf = static_cast<uint32_t*>(cache_alloc(sizeof(uint32_t), st));
  H2_CUDA(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), st));
  double* part = nullptr;
  int64_t part_elems = 0;
  for (int c0 = 0; c0 < ncols; c0 += 128) {
    const int nc = std::min(128, ncols - c0);
    const int NCOL = nc > 64 ? 128 : nc > 32 ? 64 : 32;
    const int TM = NCOL >= 128 ? 64 : 128;
    const int JC = NCOL >= 128 ? 128 : 64;
    const int64_t nchunks = npad / JC;
    const int tiles = div_up(rows, TM);
    const int S = pick_split(div_up(n, 64 * 8), npad / 128, sms);
    if (S > 1 && part_elems < rows * nc * S) {
      if (part) cache_free(part, st);
      part_elems = rows * nc * S;
      part = static_cast<double*>(cache_alloc(sizeof(double) * part_elems, st));
    }
    double* yo = S > 1 ? part : Yout + c0;
    const int64_t ld = S > 1 ? nc : ldy;
    const int64_t ss = S > 1 ? rows * nc : 0;
    omega_i8_kernel<<<(int)std::min<int64_t>((nchunks * JC * NCOL + 255) / 256, (int64_t)sms * 32), 256, 0, st>>>(
        Om + c0, ldo, n, nc, NCOL, JC, nchunks, Bq);
    H2_CHECK_LAUNCH();
    tc_dispatch<KDENSE, 7>(NCOL, dim3(tiles, S), st, nullptr, n, row0, row1, Bq, nchunks, nc, yo, ld, ss, hs, wshift,
                           ovf, A, lda);
    H2_CHECK_LAUNCH();
    if (S > 1) launch_sketch_combine(part, S, rows, nc, Yout + c0, ldy, st);
  }
  cache_free(Bq, st);
  cache_free(ovf, st);
  if (part) cache_free(part, st);
}

// minimum squared distance between distinct points over the near-field leaf pairs (the closest
// pair of a point set lies in adjacent, hence inadmissible, leaves): one CTA per leaf
__global__ void min_dist2_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                                 const double* __restrict__ Z, const int64_t* __restrict__ lb,
                                 const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                 unsigned long long* __restrict__ out) {
  const int c = blockIdx.x;
  double best = INFINITY;
  for (int e = ptr[c]; e < ptr[c + 1]; ++e) {
    const int b = idx[e];
    const int64_t i0 = lb[c], i1 = lb[c + 1], j0 = lb[b], j1 = lb[b + 1];
    const int64_t nj = j1 - j0;
    for (int64_t q = threadIdx.x; q < (i1 - i0) * nj; q += blockDim.x) {
      const int64_t i = i0 + q / nj, j = j0 + q % nj;
      if (i == j) continue;
      const double dx = X[i] - X[j], dy = Y[i] - Y[j], dz = Z[i] - Z[j];
      best = fmin(best, fma(dz, dz, fma(dy, dy, dx * dx)));
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best < INFINITY) atomicMin(out, (unsigned long long)__double_as_longlong(best));
}

double min_near_dist2(const double* X, const double* Y, const double* Z, const int64_t* leaf_begin, int nleaf,
                      const int32_t* near_ptr, const int32_t* near_idx, cudaStream_t st) {
  unsigned long long* d = static_cast<unsigned long long*>(cache_alloc(sizeof(unsigned long long), st));
  H2_CUDA(cudaMemsetAsync(d, 0x7f, sizeof(unsigned long long), st));   // 0x7f7f.. = a huge positive double
  min_dist2_kernel<<<nleaf, 256, 0, st>>>(X, Y, Z, leaf_begin, near_ptr, near_idx, d);
  H2_CHECK_LAUNCH();
  unsigned long long h = 0;
  H2_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  H2_CUDA(cudaStreamSynchronize(st));
  cache_free(d, st);
  double v;
  std::memcpy(&v, &h, sizeof(v));
  return v;
}

}  // namespace h2
