// summarize.cuh -- one warp computes one chunk summary (k~_c, beta^_c).
//
//   k~_c    = (1/C) sum_i k_{cC+i}                       P:99 Eq.10 (reading R1)
//   omega_c = lambda * clip(k~_c + eps_c)                 P:311-314 Eq.15 (R2, R3)
//   a_i     = omega_c . k_i - |k_i|^2 / 2                 log xi
//   beta^_c = sum_i softmax(a)_i v_i                      P:92 Eq.9, S = 1
//
// The softmax over the chunk is evaluated online (running max / running sum),
// i.e. log-domain with max subtraction -- the linear-domain xi underflows at
// d = 128 (R12).  Lane l owns CPL contiguous channels.
#pragma once
#include "common.cuh"

namespace eva {

template <int D> struct LaneMap {
  static constexpr int CPL = D >= 32 ? D / 32 : 1;  // channels per lane
  static constexpr int LANES = D / CPL;              // active lanes
};

// RowK(i) / RowV(i): pointer to row i (0..C-1) of the chunk's keys / values.
template <typename T, int D, typename RowK, typename RowV>
__device__ __forceinline__ void summarize_chunk_warp(const RowK& rowK, const RowV& rowV, int C,
                                                     const float* eps_c, uint32_t bh_global,
                                                     uint32_t chunk, const eva_config& cfg,
                                                     T* ksum_out, T* vsum_out) {
  using LM = LaneMap<D>;
  constexpr int CPL = LM::CPL;
  const int lane = threadIdx.x & 31;
  const bool act = lane < LM::LANES;
  const int ch0 = lane * CPL;

  // pass 1: mean key
  float kt[CPL];
#pragma unroll
  for (int j = 0; j < CPL; ++j) kt[j] = 0.f;
  if (act) {
    for (int i = 0; i < C; ++i) {
      float k[CPL];
      load_vec<T, CPL>(rowK(i) + ch0, k);
#pragma unroll
      for (int j = 0; j < CPL; ++j) kt[j] += k[j];
    }
  }
  const float invC = 1.0f / (float)C;
#pragma unroll
  for (int j = 0; j < CPL; ++j) kt[j] *= invC;

  // omega (Eq.15)
  float om[CPL];
  if (act) {
    float e[CPL];
    if (eps_c) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) e[j] = eps_c[ch0 + j];
    } else {
      if constexpr (CPL == 4) {
        float4 z = philox_normal4(cfg.seed, cfg.layer, bh_global, chunk, (uint32_t)lane);
        e[0] = z.x; e[1] = z.y; e[2] = z.z; e[3] = z.w;
      } else {
#pragma unroll
        for (int j = 0; j < CPL; ++j)
          e[j] = philox_normal1(cfg.seed, cfg.layer, bh_global, chunk, ch0 + j);
      }
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) om[j] = omega_of(kt[j], e[j], cfg);
  } else {
#pragma unroll
    for (int j = 0; j < CPL; ++j) om[j] = 0.f;
  }

  // pass 2: online log-domain softmax over the chunk's log-xi logits
  float m = -INFINITY, l = 0.f, acc[CPL];
#pragma unroll
  for (int j = 0; j < CPL; ++j) acc[j] = 0.f;
  for (int i = 0; i < C; ++i) {
    float k[CPL], v[CPL];
    float part = 0.f;
    if (act) {
      load_vec<T, CPL>(rowK(i) + ch0, k);
      load_vec<T, CPL>(rowV(i) + ch0, v);
#pragma unroll
      for (int j = 0; j < CPL; ++j) part += k[j] * (om[j] - 0.5f * k[j]);
    } else {
#pragma unroll
      for (int j = 0; j < CPL; ++j) v[j] = 0.f;
    }
    const float a = warp_sum(part);
    const float mn = fmaxf(m, a);
    const float corr = __expf(m - mn);  // m = -inf on the first row -> 0
    const float p = __expf(a - mn);
    l = l * corr + p;
#pragma unroll
    for (int j = 0; j < CPL; ++j) acc[j] = acc[j] * corr + p * v[j];
    m = mn;
  }
  if (act) {
    const float il = 1.0f / l;
#pragma unroll
    for (int j = 0; j < CPL; ++j) acc[j] *= il;
    store_vec<T, CPL>(ksum_out + ch0, kt);
    store_vec<T, CPL>(vsum_out + ch0, acc);
  }
}

}  // namespace eva
