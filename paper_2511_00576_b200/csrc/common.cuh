// common.cuh -- device helpers shared by the FlashEVA kernels (sm_100a).
// No code here is shared with oracle/ (the oracle has its own Philox, mask and
// arithmetic); see DESIGN.md §4 for the independence rule.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/eva.h"

namespace eva {

// ---------------------------------------------------------------- element I/O
template <typename T> struct Elem;
template <> struct Elem<float> {
  static __device__ __forceinline__ float to_f(float x) { return x; }
  static __device__ __forceinline__ float from_f(float x) { return x; }
};
template <> struct Elem<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// Load N contiguous elements starting at p (N in {1,2,4,8}) into floats.
template <typename T, int N> __device__ __forceinline__ void load_vec(const T* p, float* out) {
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = Elem<T>::to_f(p[i]);
}
template <> __device__ __forceinline__ void load_vec<float, 4>(const float* p, float* out) {
  float4 v = *reinterpret_cast<const float4*>(p);
  out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
}
template <> __device__ __forceinline__ void load_vec<__nv_bfloat16, 4>(const __nv_bfloat16* p, float* out) {
  uint2 v = *reinterpret_cast<const uint2*>(p);
  __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&v.x), b = *reinterpret_cast<__nv_bfloat162*>(&v.y);
  float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
  out[0] = fa.x; out[1] = fa.y; out[2] = fb.x; out[3] = fb.y;
}
template <> __device__ __forceinline__ void load_vec<__nv_bfloat16, 8>(const __nv_bfloat16* p, float* out) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
    out[2 * i] = f.x; out[2 * i + 1] = f.y;
  }
}

// Unpack one 16-byte piece (16/sizeof(T) elements) into floats.
template <typename T> __device__ __forceinline__ void unpack16(const uint4& v, float* out);
template <> __device__ __forceinline__ void unpack16<float>(const uint4& v, float* out) {
  out[0] = __uint_as_float(v.x); out[1] = __uint_as_float(v.y);
  out[2] = __uint_as_float(v.z); out[3] = __uint_as_float(v.w);
}
template <> __device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4& v, float* out) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = __uint_as_float(w[i] << 16);
    out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 ldg16_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <typename T, int N> __device__ __forceinline__ void store_vec(T* p, const float* in) {
#pragma unroll
  for (int i = 0; i < N; ++i) p[i] = Elem<T>::from_f(in[i]);
}

// ---------------------------------------------------------------- warp helpers
template <int WIDTH> __device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) { return group_sum<32>(v); }

// ---------------------------------------------------------------- partition (reading R7)
// Query n sees locals [lo, n] and summaries c < nsum.  Integer-exact.
struct Range { int64_t lo, nsum; };
__host__ __device__ __forceinline__ Range mask_range(int64_t n, int C, int W, int mode) {
  Range r;
  if (mode == EVA_WINDOW_SLIDING) {
    int64_t s = n / C - W / C + 1;
    r.nsum = s > 0 ? s : 0;
    r.lo = r.nsum * C;
  } else {
    r.lo = (n / W) * W;
    r.nsum = r.lo / C;
  }
  return r;
}

// Visible set of query n in a sequence of T positions, every mode (R7, R15): locals
// [lo, hi) and summaries [0, s1) U [s2, nC).  Causal modes: hi = n + 1, s2 = "never".
struct Vis { int64_t lo, hi, s1, s2; };
__host__ __device__ __forceinline__ Vis visible_set(int64_t n, int C, int W, int mode, int64_t T) {
  Vis v;
  if (mode == EVA_NONCAUSAL) {
    v.lo = (n / W) * W;
    v.hi = v.lo + W < T ? v.lo + W : T;
    v.s1 = v.lo / C;
    v.s2 = (v.lo + W) / C;
  } else {
    const Range r = mask_range(n, C, W, mode);
    v.lo = r.lo;
    v.hi = n + 1;
    v.s1 = r.nsum;
    v.s2 = INT64_MAX;
  }
  return v;
}

// ---------------------------------------------------------------- Philox4x32-10 (reading R9)
struct U4 { uint32_t x, y, z, w; };
__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
    const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
#endif
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Four N(0,1) draws eps[c][4i .. 4i+3] of unit bh: Philox block (i, c, bh, layer),
// u = ((x >> 8) + 0.5) * 2^-24, Box-Muller pairs (u0,u1) and (u2,u3).
__device__ __forceinline__ float4 philox_normal4(uint64_t seed, uint32_t layer, uint32_t bh,
                                                 uint32_t c, uint32_t i) {
  U4 x = philox4x32_10(U4{i, c, bh, layer}, (uint32_t)seed, (uint32_t)(seed >> 32));
  const float s = 5.9604644775390625e-08f;  // 2^-24
  float u0 = ((float)(x.x >> 8) + 0.5f) * s, u1 = ((float)(x.y >> 8) + 0.5f) * s;
  float u2 = ((float)(x.z >> 8) + 0.5f) * s, u3 = ((float)(x.w >> 8) + 0.5f) * s;
  float r0 = sqrtf(-2.0f * logf(u0)), r1 = sqrtf(-2.0f * logf(u2));
  float s0, c0, s1, c1;
  sincospif(2.0f * u1, &s0, &c0);
  sincospif(2.0f * u3, &s1, &c1);
  return make_float4(r0 * c0, r0 * s0, r1 * c1, r1 * s1);
}

// eps component j of chunk c (used where a lane holds a non-multiple-of-4 channel group).
__device__ __forceinline__ float philox_normal1(uint64_t seed, uint32_t layer, uint32_t bh,
                                                uint32_t c, uint32_t j) {
  float4 z = philox_normal4(seed, layer, bh, c, j >> 2);
  switch (j & 3) { case 0: return z.x; case 1: return z.y; case 2: return z.z; default: return z.w; }
}

// Eq.15 with mu_c = k~_c; reading R3 selects the composition.
__device__ __forceinline__ float omega_of(float kt, float e, const eva_config& cfg) {
  if (cfg.omega_mode == EVA_OMEGA_AS_PRINTED)
    return cfg.lambda * fminf(fmaxf(kt + e, -cfg.clip), cfg.clip);
  return kt + cfg.lambda * fminf(fmaxf(e, -cfg.clip), cfg.clip);
}

// ---------------------------------------------------------------- programmatic dependent launch
// Kernels of the hot path are launched with programmatic stream serialisation: the next
// kernel on the stream may be scheduled as soon as every CTA of this one has executed
// pdl_trigger(), and it runs its prologue (barrier init, TMEM alloc, descriptor prefetch)
// while this one drains.  pdl_wait() blocks until the previous grid has COMPLETED and its
// memory is visible, so every kernel calls it before its first global-memory access --
// the overlap is launch latency and prologue only, never data.  Both are no-ops when the
// launch carried no programmatic dependency.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kern, std::forward<Args>(args)...);
}

// Launch counter (eva_launch_count): incremented on the host per enqueue.
void note_launch(int n = 1);

}  // namespace eva
