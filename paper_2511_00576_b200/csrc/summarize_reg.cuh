// summarize_reg.cuh -- the register-resident chunk summariser (one chunk per 128-thread CTA),
// shared by eva_summarize, the cache append, the ragged decode step, the RoPE producer and the
// bulk-copy summariser, so all of them produce the same summaries bit for bit.
#pragma once
#include "common.cuh"

namespace eva {

// Rows per lane slot of the register summariser for (C, D, T); > 16 means "too large".
template <typename T, int D>
constexpr int summ_reg_ni(int C) {
  return (C + 4 * (32 / (D * (int)sizeof(T) / 16)) - 1) / (4 * (32 / (D * (int)sizeof(T) / 16)));
}

// Register-resident variant (the default when C <= 32 * 128 * 16 / (D * sizeof(T))):
// one CTA (4 warps) per chunk; a row is read by TPR = D*sizeof(T)/16 lanes with one 16-byte
// load each, a warp covers RPW = 32/TPR rows per load and warp w owns the row slots
// w*RPW + 4*RPW*i.  Every K and V piece of the chunk is loaded up front (up to 2*NI
// 16-byte loads in flight per lane) and kept in registers: column sums -> k~ (smem merge
// of the 4 warps), Eq.15 -> omega, per-row log-xi logits (group shuffles), per-warp
// online softmax of the rows -> partial (m, l, acc), merged across warps in smem.
// Pk (may be nullptr): the learned summary-key projection of NEXT row 4 (reading R17),
// k~ = Pk mean(k) with Pk [D, D] row-major fp32 of this unit's head; omega uses mu = k~.
struct NoKXform {
  __device__ __forceinline__ void operator()(int, int, uint4&, bool) const {}
};
// LD: the 16-byte load of a key / value piece (global streaming loads by default; the bulk-copy
// summariser passes shared-memory loads, so every path runs the same arithmetic bit for bit).
struct LdGlobalStream {
  template <typename P>
  __device__ __forceinline__ uint4 operator()(const P* p) const { return ldg16_stream(p); }
};
// KX (optional): applied to every loaded 16-byte key piece (row r, channel ch0, valid = r < C)
// before any use, by every lane of the warp -- the fused RoPE producer rotates (exchanging the
// half-split partner pieces by shuffles) and stores the keys there.
// RELOAD: re-read every piece through LD where it is used instead of holding the chunk in
// registers (the rows sit in shared memory: same arithmetic in the same order, ~60 fewer
// registers, so more chunks are computed at once per SM).  Only with the identity KX.
template <typename T, int D, int NI, typename RowK, typename RowV, typename KX = NoKXform,
          typename LD = LdGlobalStream, bool RELOAD = false>
__device__ __forceinline__ void summarize_chunk_reg(const RowK& rowK, const RowV& rowV, int C,
                                                    const float* eps_c, uint32_t bh_global,
                                                    uint32_t chunk, const eva_config& cfg,
                                                    T* ksum_out, T* vsum_out, const float* Pk = nullptr,
                                                    const KX& kxf = KX(), const LD& ld = LD()) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int TPR = D / VEC;
  constexpr int RPW = 32 / TPR;
  __shared__ float sh_sum[4][D];
  __shared__ float sh_om[D];
  __shared__ float sh_m[4], sh_l[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / TPR, gl = lane % TPR, ch0 = gl * VEC;
  uint4 kx[RELOAD ? 1 : NI], vx[RELOAD ? 1 : NI];
  auto kpiece = [&](int i, int r) -> uint4 { if constexpr (RELOAD) return ld(rowK(r) + ch0); else return kx[i]; };
  auto vpiece = [&](int i, int r) -> uint4 { if constexpr (RELOAD) return ld(rowV(r) + ch0); else return vx[i]; };
  if constexpr (!RELOAD) {
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int r = warp * RPW + 4 * RPW * i + grp;
      if (r < C) {
        kx[i] = ld(rowK(r) + ch0);
        vx[i] = ld(rowV(r) + ch0);
      } else {
        kx[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      kxf(r, ch0, kx[i], r < C);  // every lane (a transform may exchange pieces by shuffles)
    }
  } else {
    static_assert(sizeof(KX) == sizeof(NoKXform), "RELOAD takes no key transform");
  }
  // column sums
  float cs[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) cs[j] = 0.f;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = warp * RPW + 4 * RPW * i + grp;
    if (r < C) {
      float k[VEC];
      unpack16<T>(kpiece(i, r), k);
#pragma unroll
      for (int j = 0; j < VEC; ++j) cs[j] += k[j];
    }
  }
#pragma unroll
  for (int o = TPR; o < 32; o <<= 1)
#pragma unroll
    for (int j = 0; j < VEC; ++j) cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], o);
  if (grp == 0) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) sh_sum[warp][ch0 + j] = cs[j];
  }
  __syncthreads();
  __shared__ float sh_mean[D];
  if (Pk != nullptr) {  // the chunk mean first: every projected channel reads all of it
    if (threadIdx.x < D) {
      const int ch = threadIdx.x;
      sh_mean[ch] = (sh_sum[0][ch] + sh_sum[1][ch] + sh_sum[2][ch] + sh_sum[3][ch]) * (1.0f / (float)C);
    }
    __syncthreads();
  }
  // k~ and omega (Eq.15); one Philox block per 4 channels
  if (threadIdx.x < D / 4) {
    const int q = threadIdx.x;
    float e[4];
    if (eps_c) {
      const float* ep = eps_c + 4 * q;
      e[0] = ep[0]; e[1] = ep[1]; e[2] = ep[2]; e[3] = ep[3];
    } else {
      const float4 z = philox_normal4(cfg.seed, cfg.layer, bh_global, chunk, (uint32_t)q);
      e[0] = z.x; e[1] = z.y; e[2] = z.z; e[3] = z.w;
    }
    T* ko = ksum_out + 4 * q;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ch = 4 * q + j;
      float kt;
      if (Pk == nullptr) {
        kt = (sh_sum[0][ch] + sh_sum[1][ch] + sh_sum[2][ch] + sh_sum[3][ch]) * (1.0f / (float)C);
      } else {
        const float4* prow = reinterpret_cast<const float4*>(Pk + (size_t)ch * D);
        kt = 0.f;
#pragma unroll 4
        for (int l4 = 0; l4 < D / 4; ++l4) {
          const float4 w = __ldg(prow + l4);
          kt = fmaf(w.x, sh_mean[4 * l4], kt);
          kt = fmaf(w.y, sh_mean[4 * l4 + 1], kt);
          kt = fmaf(w.z, sh_mean[4 * l4 + 2], kt);
          kt = fmaf(w.w, sh_mean[4 * l4 + 3], kt);
        }
      }
      sh_om[ch] = omega_of(kt, e[j], cfg);
      ko[j] = Elem<T>::from_f(kt);
    }
  }
  __syncthreads();
  float om[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) om[j] = sh_om[ch0 + j];
  // logits a_r = omega . k_r - |k_r|^2 / 2 and the warp's online softmax over its rows
  float a[NI];
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = warp * RPW + 4 * RPW * i + grp;
    float part = 0.f;
    if (r < C) {
      float k[VEC];
      unpack16<T>(kpiece(i, r), k);
#pragma unroll
      for (int j = 0; j < VEC; ++j) part += k[j] * (om[j] - 0.5f * k[j]);
    }
    part = group_sum<TPR>(part);
    a[i] = r < C ? part : -INFINITY;
    m = fmaxf(m, a[i]);
  }
#pragma unroll
  for (int o = TPR; o < 32; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float l = 0.f, acc[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = warp * RPW + 4 * RPW * i + grp;
    if (r < C) {
      const float p = __expf(a[i] - m);
      l += p;
      float v[VEC];
      unpack16<T>(vpiece(i, r), v);
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] += p * v[j];
    }
  }
#pragma unroll
  for (int o = TPR; o < 32; o <<= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
  }
  if (lane == 0) { sh_m[warp] = m; sh_l[warp] = l; }
  __syncthreads();  // sh_sum is free again: reuse it for the partial accumulators
  if (grp == 0) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) sh_sum[warp][ch0 + j] = acc[j];
  }
  __syncthreads();
  if (threadIdx.x < D) {
    const int ch = threadIdx.x;
    float M = fmaxf(fmaxf(sh_m[0], sh_m[1]), fmaxf(sh_m[2], sh_m[3]));
    float L = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float f = sh_m[w] == -INFINITY ? 0.f : __expf(sh_m[w] - M);
      L += f * sh_l[w];
      o += f * sh_sum[w][ch];
    }
    vsum_out[ch] = Elem<T>::from_f(o / L);
  }
}



}  // namespace eva
