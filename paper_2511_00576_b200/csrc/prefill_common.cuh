// prefill_common.cuh -- small device helpers shared by the tcgen05 prefill kernels
// (prefill_sm100.cu): MUFU exp2, bf16 packing, column-range bit masks, packed
// fp32x2 arithmetic.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace eva {
namespace pfx {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}


// Bits [lo, hi) of a 64-column tile (clamped).
__device__ __forceinline__ uint64_t range_bits(int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, 64);
  if (hi <= lo) return 0ull;
  const uint64_t a = hi >= 64 ? ~0ull : ((1ull << hi) - 1ull);
  const uint64_t b = (1ull << lo) - 1ull;
  return a & ~b;
}
// ---- packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2: two lanes per issue slot)
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float f2lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for x <= 0 on the FMA/ALU pipes (the MUFU pipe does 16 ex2 per clock per SM, a quarter of
// what the softmax would need to keep pace with the tensor core at d = 64): x = n + f with
// n = rint(x) via the 1.5*2^23 shifter, 2^f on [-1/2, 1/2] by a degree-3 polynomial (relative
// error 7.5e-5, far below the bf16 rounding of P), and n added to the exponent field.  x is
// clamped at -126 so that -inf (masked columns) gives a value below 2^-125 instead of garbage.
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
  const float lo = fmaxf(f2lo(x), -126.f), hi = fmaxf(f2hi(x), -126.f);
  const uint64_t xc = f2pack(lo, hi);
  const uint64_t SH = f2pack(12582912.f, 12582912.f), NSH = f2pack(-12582912.f, -12582912.f);
  const uint64_t j = fadd2(xc, SH);                    // low mantissa bits hold rint(x)
  const uint64_t f = ffma2(fadd2(j, NSH), f2pack(-1.f, -1.f), xc);  // x - rint(x), exact
  uint64_t p = ffma2(f2pack(0.055171627551317215f, 0.055171627551317215f), f,
                     f2pack(0.24261116981506348f, 0.24261116981506348f));
  p = ffma2(p, f, f2pack(0.6932610273361206f, 0.6932610273361206f));
  p = ffma2(p, f, f2pack(0.9999280571937561f, 0.9999280571937561f));
  const uint32_t rlo = (uint32_t)p + ((uint32_t)j << 23);
  const uint32_t rhi = (uint32_t)(p >> 32) + ((uint32_t)(j >> 32) << 23);
  return (uint64_t)rlo | ((uint64_t)rhi << 32);
}

}  // namespace pfx
}  // namespace eva
