// summarize_cta.cuh -- one CTA (128 threads) computes one chunk summary (k~_c, beta^_c).
// Same formulas as summarize.cuh (Eq.10, Eq.15, P:49 xi, Eq.9 with
// S = 1), but bandwidth-shaped: the chunk's C key rows and C value rows are staged in
// shared memory with cp.async (every 16-byte piece in flight at once), then read back
// as 16-byte vectors by "row groups": thread t owns the VEC channels of piece t % TPR
// (TPR = pieces per row) of the rows g, g + G, g + 2G, ... (g = t / TPR, G = 128 / TPR):
//   k~      : column sums over the rows, groups combined through shared memory
//   omega   : Eq.15 per channel (Philox in-kernel or caller eps)
//   a_i     : omega . k_i - |k_i|^2 / 2 (partial per piece, reduced over the TPR lanes)
//   softmax : max / sum over the C logits (warp 0)
//   beta^   : sum_i w_i v_i, groups combined through shared memory
// Row addresses come from a functor so the cache append can summarise chunks that
// straddle the ring and the newly appended tokens.
#pragma once
#include "common.cuh"

namespace eva {

constexpr int SUMM_THREADS = 128;

__host__ __device__ constexpr size_t summ_smem_bytes(int C, int D, int elem) {
  return (size_t)2 * C * D * elem + (size_t)C * 4 + (size_t)D * 4 + (size_t)SUMM_THREADS * 16 * 4 + 64;
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

// Stage the chunk's C key rows and C value rows into kv_smem ([C][D] K then [C][D] V)
// with cp.async; the caller commits / waits the group.
template <typename T, int D, typename RowK, typename RowV>
__device__ __forceinline__ void summarize_stage(const RowK& rowK, const RowV& rowV, int C, T* kv_smem) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int TPR = D / VEC;
  T* Ks = kv_smem;
  T* Vs = Ks + (size_t)C * D;
  for (int i = threadIdx.x; i < C * TPR; i += SUMM_THREADS) {
    const int r = i / TPR, p = i % TPR;
    cp_async16(Ks + (size_t)r * D + p * VEC, rowK(r) + p * VEC);
    cp_async16(Vs + (size_t)r * D + p * VEC, rowV(r) + p * VEC);
  }
}

// Compute (k~, beta^) of a staged chunk.  work: scratch of summ_work_bytes(C, D) bytes.
__host__ __device__ constexpr size_t summ_work_bytes(int C, int D) {
  return (size_t)C * 4 + (size_t)D * 4 + (size_t)SUMM_THREADS * 16 * 4 + 64;
}
template <typename T, int D>
__device__ __forceinline__ void summarize_compute(const T* kv_smem, int C, const float* eps_c,
                                                  uint32_t bh_global, uint32_t chunk,
                                                  const eva_config& cfg, T* ksum_out, T* vsum_out,
                                                  uint8_t* work) {
  constexpr int VEC = 16 / sizeof(T);          // elements per 16-byte piece
  constexpr int TPR = D / VEC;                 // pieces (threads) per row
  constexpr int G = SUMM_THREADS / TPR;        // row groups
  static_assert(TPR >= 1 && TPR <= 32 && SUMM_THREADS % TPR == 0, "bad D");
  const T* Ks = kv_smem;
  const T* Vs = Ks + (size_t)C * D;
  float* a = reinterpret_cast<float*>(work);
  float* om = a + C;
  float* part = om + D;  // [G][D]
  float* stat = part + G * D;
  const int tid = threadIdx.x;
  const int pc = tid % TPR, g = tid / TPR;
  const int ch0 = pc * VEC;

  // k~: column mean
  {
    float s[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) s[j] = 0.f;
    for (int r = g; r < C; r += G) {
      float k[VEC];
      load_vec<T, VEC>(Ks + (size_t)r * D + ch0, k);
#pragma unroll
      for (int j = 0; j < VEC; ++j) s[j] += k[j];
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) part[g * D + ch0 + j] = s[j];
  }
  __syncthreads();
  if (tid < D) {
    float s = 0.f;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) s += part[gg * D + tid];
    const float kt = s * (1.0f / (float)C);
    const float e = eps_c ? eps_c[tid]
                          : philox_normal1(cfg.seed, cfg.layer, bh_global, chunk, (uint32_t)tid);
    om[tid] = omega_of(kt, e, cfg);
    ksum_out[tid] = Elem<T>::from_f(kt);
  }
  __syncthreads();

  // a_i = omega . k_i - |k_i|^2 / 2
  {
    float o[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) o[j] = om[ch0 + j];
    const int nit = (C + G - 1) / G;  // uniform trip count for the shuffles
    for (int it = 0; it < nit; ++it) {
      const int r = g + it * G;
      float s = 0.f;
      if (r < C) {
        float k[VEC];
        load_vec<T, VEC>(Ks + (size_t)r * D + ch0, k);
#pragma unroll
        for (int j = 0; j < VEC; ++j) s += k[j] * (o[j] - 0.5f * k[j]);
      }
      s = group_sum<TPR>(s);
      if (pc == 0 && r < C) a[r] = s;
    }
  }
  __syncthreads();
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
    if (tid == 0) stat[0] = 1.0f / z;
  }
  __syncthreads();
  // beta^ = sum_i w_i v_i / sum_i w_i
  {
    float s[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) s[j] = 0.f;
    for (int r = g; r < C; r += G) {
      float v[VEC];
      load_vec<T, VEC>(Vs + (size_t)r * D + ch0, v);
      const float w = a[r];
#pragma unroll
      for (int j = 0; j < VEC; ++j) s[j] += w * v[j];
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) part[g * D + ch0 + j] = s[j];
  }
  __syncthreads();
  if (tid < D) {
    float s = 0.f;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) s += part[gg * D + tid];
    vsum_out[tid] = Elem<T>::from_f(s * stat[0]);
  }
}

template <typename T, int D, typename RowK, typename RowV>
__device__ __forceinline__ void summarize_chunk_cta(const RowK& rowK, const RowV& rowV, int C,
                                                    const float* eps_c, uint32_t bh_global,
                                                    uint32_t chunk, const eva_config& cfg,
                                                    T* ksum_out, T* vsum_out, uint8_t* smem) {
  T* kv = reinterpret_cast<T*>(smem);
  summarize_stage<T, D>(rowK, rowV, C, kv);
  cp_async_wait_all();
  __syncthreads();
  summarize_compute<T, D>(kv, C, eps_c, bh_global, chunk, cfg, ksum_out, vsum_out,
                          smem + (size_t)2 * C * D * sizeof(T));
}

}  // namespace eva
