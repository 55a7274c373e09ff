// summarize_cta.cuh -- one CTA (128 threads) computes one chunk summary (k~_c, beta^_c).
// Same formulas as summarize.cuh (Eq.10, Eq.15, P:49 xi, Eq.9 with
// S = 1), but bandwidth-shaped: the chunk's C key rows and C value rows are staged in
// shared memory with cp.async (every 16-byte piece in flight at once), then
//   k~      : column sums over the rows             (thread per channel x row group)
//   omega   : Eq.15 per channel                     (Philox in-kernel or caller eps)
//   a_i     : omega . k_i - |k_i|^2 / 2              (warp per row, shuffle reduce)
//   softmax : max / sum over the C logits           (warp 0)
//   beta^   : sum_i w_i v_i                          (thread per channel x row group)
// Row addresses come from a functor so the cache append can summarise chunks that
// straddle the ring and the newly appended tokens.
#pragma once
#include "common.cuh"

namespace eva {

constexpr int SUMM_THREADS = 128;

__host__ __device__ constexpr size_t summ_smem_bytes(int C, int D, int elem) {
  return (size_t)2 * C * D * elem + (size_t)C * 4 + (size_t)D * 4 + (size_t)SUMM_THREADS * 4 + 64;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

template <typename T, int D, typename RowK, typename RowV>
__device__ __forceinline__ void summarize_chunk_cta(const RowK& rowK, const RowV& rowV, int C,
                                                    const float* eps_c, uint32_t bh_global,
                                                    uint32_t chunk, const eva_config& cfg,
                                                    T* ksum_out, T* vsum_out, uint8_t* smem) {
  constexpr int VEC = 16 / sizeof(T);          // elements per 16-byte piece
  constexpr int PPR = D / VEC;                 // pieces per row
  constexpr int GROUPS = SUMM_THREADS / D;     // row groups in the column passes (D <= 128)
  static_assert(D <= SUMM_THREADS && SUMM_THREADS % D == 0, "D must divide 128");
  T* Ks = reinterpret_cast<T*>(smem);
  T* Vs = Ks + (size_t)C * D;
  float* a = reinterpret_cast<float*>(Vs + (size_t)C * D);
  float* om = a + C;
  float* part = om + D;  // [SUMM_THREADS]
  float* stat = part + SUMM_THREADS;  // [2]: max, 1/sum
  const int tid = threadIdx.x;

  // stage K and V rows
  for (int i = tid; i < C * PPR; i += SUMM_THREADS) {
    const int r = i / PPR, p = i % PPR;
    cp_async16(Ks + (size_t)r * D + p * VEC, rowK(r) + p * VEC);
    cp_async16(Vs + (size_t)r * D + p * VEC, rowV(r) + p * VEC);
  }
  cp_async_wait_all();
  __syncthreads();

  // k~ = column mean; thread (g, ch) sums rows g, g+GROUPS, ...
  const int ch = tid % D, g = tid / D;
  {
    float s = 0.f;
    for (int r = g; r < C; r += GROUPS) s += Elem<T>::to_f(Ks[(size_t)r * D + ch]);
    part[tid] = s;
  }
  __syncthreads();
  if (tid < D) {
    float s = 0.f;
#pragma unroll
    for (int gg = 0; gg < GROUPS; ++gg) s += part[gg * D + tid];
    const float kt = s * (1.0f / (float)C);
    float e;
    if (eps_c) e = eps_c[tid];
    else e = philox_normal1(cfg.seed, cfg.layer, bh_global, chunk, (uint32_t)tid);
    om[tid] = omega_of(kt, e, cfg);
    ksum_out[tid] = Elem<T>::from_f(kt);
  }
  __syncthreads();

  // a_i = omega . k_i - |k_i|^2 / 2 : warp w takes rows w, w+4, ...
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int r = warp; r < C; r += SUMM_THREADS / 32) {
      float s = 0.f;
      for (int c2 = lane; c2 < D; c2 += 32) {
        const float k = Elem<T>::to_f(Ks[(size_t)r * D + c2]);
        s += k * (om[c2] - 0.5f * k);
      }
      s = warp_sum(s);
      if (lane == 0) a[r] = s;
    }
  }
  __syncthreads();
  // softmax statistics over the C logits (warp 0)
  if (tid < 32) {
    float m = -INFINITY;
    for (int r = tid; r < C; r += 32) m = fmaxf(m, a[r]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float z = 0.f;
    for (int r = tid; r < C; r += 32) {
      const float w = __expf(a[r] - m);
      a[r] = w;
      z += w;
    }
    z = warp_sum(z);
    if (tid == 0) stat[1] = 1.0f / z;
  }
  __syncthreads();
  // beta^ = sum_i w_i v_i / sum_i w_i
  {
    float s = 0.f;
    for (int r = g; r < C; r += GROUPS) s += a[r] * Elem<T>::to_f(Vs[(size_t)r * D + ch]);
    part[tid] = s;
  }
  __syncthreads();
  if (tid < D) {
    float s = 0.f;
#pragma unroll
    for (int gg = 0; gg < GROUPS; ++gg) s += part[gg * D + tid];
    vsum_out[tid] = Elem<T>::from_f(s * stat[1]);
  }
}

}  // namespace eva
