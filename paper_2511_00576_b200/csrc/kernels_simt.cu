// kernels_simt.cu -- SIMT kernels of the FlashEVA hot path (sm_100a):
//   summarize (one warp per chunk), the fp32 parity prefill, cache append,
//   split-K decode + merge, and the debug mask / Philox / eps dumps.
// The bf16 tensor-core prefill lives in prefill_sm100.cu.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "launch.h"
#include "summarize.cuh"
#include "summarize_cta.cuh"
#include "summarize_reg.cuh"

namespace eva {

// ============================================================================ summarize
// grid: (ceil(nC / 4), bh_count); block 128 = 4 warps, warp w -> chunk 4*blockIdx.x + w.
template <typename T, int D>
__global__ void __launch_bounds__(128) summarize_kernel(eva_config cfg, const T* __restrict__ K,
                                                        const T* __restrict__ V,
                                                        const float* __restrict__ eps,
                                                        T* __restrict__ Ksum, T* __restrict__ Vsum, int c0) {
  const int nC = cfg.T / cfg.chunk;
  const int c = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int u = blockIdx.y;
  if (c >= nC) return;
  const int C = cfg.chunk;
  const T* Kc = K + ((size_t)u * cfg.T + (size_t)c * C) * D;
  const T* Vc = V + ((size_t)u * cfg.T + (size_t)c * C) * D;
  auto rowK = [&](int i) { return Kc + (size_t)i * D; };
  auto rowV = [&](int i) { return Vc + (size_t)i * D; };
  const float* e = eps ? eps + ((size_t)u * nC + c) * D : nullptr;
  summarize_chunk_warp<T, D>(rowK, rowV, C, e, (uint32_t)(cfg.bh_begin + u), (uint32_t)(c0 + c), cfg,
                             Ksum + ((size_t)u * nC + c) * D, Vsum + ((size_t)u * nC + c) * D);
}

// grid: (nC, bh_count); block 128; one CTA per chunk, rows staged in shared memory.
template <typename T, int D>
__global__ void __launch_bounds__(SUMM_THREADS) summarize_cta_kernel(eva_config cfg, const T* __restrict__ K,
                                                                   const T* __restrict__ V,
                                                                   const float* __restrict__ eps,
                                                                   T* __restrict__ Ksum,
                                                                   T* __restrict__ Vsum, int c0) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int nC = cfg.T / cfg.chunk;
  const int c = blockIdx.x, u = blockIdx.y, C = cfg.chunk;
  const T* Kc = K + ((size_t)u * cfg.T + (size_t)c * C) * D;
  const T* Vc = V + ((size_t)u * cfg.T + (size_t)c * C) * D;
  auto rowK = [&](int i) { return Kc + (size_t)i * D; };
  auto rowV = [&](int i) { return Vc + (size_t)i * D; };
  const float* e = eps ? eps + ((size_t)u * nC + c) * D : nullptr;
  summarize_chunk_cta<T, D>(rowK, rowV, C, e, (uint32_t)(cfg.bh_begin + u), (uint32_t)(c0 + c), cfg,
                            Ksum + ((size_t)u * nC + c) * D, Vsum + ((size_t)u * nC + c) * D, smem);
}

template <typename T, int D, int NI>
__global__ void __launch_bounds__(128) summarize_reg_kernel(eva_config cfg, const T* __restrict__ K,
                                                           const T* __restrict__ V,
                                                           const float* __restrict__ eps,
                                                           T* __restrict__ Ksum, T* __restrict__ Vsum, int c0,
                                                           const float* __restrict__ Pk = nullptr) {
  pdl_wait();
  pdl_trigger();
  const int C = cfg.chunk, nC = cfg.T / C;
  const int c = blockIdx.x, u = blockIdx.y;
  const T* Kc = K + ((size_t)u * cfg.T + (size_t)c * C) * D;
  const T* Vc = V + ((size_t)u * cfg.T + (size_t)c * C) * D;
  summarize_chunk_reg<T, D, NI>([&](int r) { return Kc + (size_t)r * D; }, [&](int r) { return Vc + (size_t)r * D; },
                                C, eps ? eps + ((size_t)u * nC + c) * D : nullptr,
                                (uint32_t)(cfg.bh_begin + u), (uint32_t)(c0 + c), cfg,
                                Ksum + ((size_t)u * nC + c) * D, Vsum + ((size_t)u * nC + c) * D,
                                Pk ? Pk + (size_t)((cfg.bh_begin + u) % cfg.H) * D * D : nullptr);
}

// Summaries broadcast to n_dst destination buffers (context parallelism: every rank's copy
// of the global summary list, reached through NVLink peer pointers): the summary of chunk
// c0 + c is computed once into shared memory and stored to row (c0 + c) of unit u of each
// destination [units, dst_rows, D] -- the compute and the all-gather in one kernel.
// ------------------------------------------------------------ RoPE (NEXT row 4, R18 / R19)
// The first rd channels of a row at position pos rotate in pairs j < rd/2 by the angle
// pos * base^(-2j/rd): pair (2j, 2j+1) (interleaved, style 0) or (j, j + rd/2) (GPT-NeoX
// half-split, style 1); channels >= rd pass through.  sign = -1: the transposed rotation (the
// gradient through RoPE).  The angle is reduced mod 2 pi in double so fp32 keeps its accuracy
// at long positions.  rd is a multiple of 2 * (16 / sizeof(T)), so a 16-byte piece is either
// inside [0, rd) or outside it, and a half-split piece's partner is a whole piece rd/2 later.
// theta_j = base^(-2j/rd) comes from a double table the host fills (the kernels take the spec as
// a __grid_constant__ parameter, so th[j] is a constant-bank load, not a per-element exp2).
struct RopeSpec {
  double th[64];     // double: at positions ~2^31 a float theta alone shifts the angle by radians
  int rd;
  int style;
  float sign;
  int pad;
};
inline RopeSpec make_rope_spec(double base, int rd, int style, float sign) {
  RopeSpec rs{};
  rs.rd = rd;
  rs.style = style;
  rs.sign = sign;
  for (int j = 0; j < rd / 2 && j < 64; ++j) rs.th[j] = std::exp2(std::log2(base) * (-2.0 * (double)j / (double)rd));
  return rs;
}

__device__ __forceinline__ void rope_cs(int64_t pos, int j, const RopeSpec& rs, float& c, float& s) {
  const double theta = rs.th[j];
  double a = (double)pos * theta;
  a -= 6.283185307179586 * rint(a * 0.15915494309189535);
  __sincosf((float)a, &s, &c);  // |a| <= pi after the reduction: the MUFU form is ~1e-6 absolute
  s *= rs.sign;
}

template <typename T>
__device__ __forceinline__ uint4 pack16(const float* v) {
  constexpr int VEC = 16 / sizeof(T);
  T o[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) o[j] = Elem<T>::from_f(v[j]);
  return *reinterpret_cast<const uint4*>(o);
}

// interleaved: the pairs inside one piece (channels ch0 .. ch0 + VEC, ch0 < rd)
template <typename T>
__device__ __forceinline__ uint4 rope_piece_il(uint4 x, int64_t pos, int ch0, const RopeSpec& rs) {
  constexpr int VEC = 16 / sizeof(T);
  float v[VEC];
  unpack16<T>(x, v);
#pragma unroll
  for (int j = 0; j < VEC; j += 2) {
    float c, sn;
    rope_cs(pos, (ch0 + j) / 2, rs, c, sn);
    const float x0 = v[j], x1 = v[j + 1];
    v[j] = x0 * c - x1 * sn;
    v[j + 1] = x0 * sn + x1 * c;
  }
  return pack16<T>(v);
}

// half-split: piece a holds channels j0 .. j0 + VEC (< rd/2), piece b their partners + rd/2
template <typename T>
__device__ __forceinline__ void rope_pair_neox(uint4& a, uint4& b, int64_t pos, int j0, const RopeSpec& rs) {
  constexpr int VEC = 16 / sizeof(T);
  float va[VEC], vb[VEC];
  unpack16<T>(a, va);
  unpack16<T>(b, vb);
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    float c, sn;
    rope_cs(pos, j0 + j, rs, c, sn);
    const float x0 = va[j], x1 = vb[j];
    va[j] = x0 * c - x1 * sn;
    vb[j] = x0 * sn + x1 * c;
  }
  a = pack16<T>(va);
  b = pack16<T>(vb);
}

// Work items of one row: rotate items (interleaved: one piece each, rd/VEC of them; half-split:
// a piece pair each, rd/(2 VEC)), then pass-through pieces (D - rd)/VEC.
template <typename T, int D>
__device__ __forceinline__ int rope_items(const RopeSpec& rs) {
  constexpr int VEC = 16 / sizeof(T);
  return (rs.style == EVA_ROPE_NEOX ? rs.rd / (2 * VEC) : rs.rd / VEC) + (D - rs.rd) / VEC;
}
template <typename T, int D>
__device__ __forceinline__ void rope_row_item(const T* src, T* dst, int64_t pos, int it, const RopeSpec& rs) {
  constexpr int VEC = 16 / sizeof(T);
  const int nrot = rs.style == EVA_ROPE_NEOX ? rs.rd / (2 * VEC) : rs.rd / VEC;
  if (it >= nrot) {  // pass-through piece
    const int ch0 = rs.rd + (it - nrot) * VEC;
    if (src != dst) *reinterpret_cast<uint4*>(dst + ch0) = ldg16_stream(src + ch0);
    return;
  }
  if (rs.style == EVA_ROPE_NEOX) {
    const int j0 = it * VEC, h = rs.rd / 2;
    uint4 a = ldg16_stream(src + j0), b = ldg16_stream(src + j0 + h);
    rope_pair_neox<T>(a, b, pos, j0, rs);
    *reinterpret_cast<uint4*>(dst + j0) = a;
    *reinterpret_cast<uint4*>(dst + j0 + h) = b;
  } else {
    const int ch0 = it * VEC;
    *reinterpret_cast<uint4*>(dst + ch0) = rope_piece_il<T>(ldg16_stream(src + ch0), pos, ch0, rs);
  }
}


// eva_rope_ex's kernel: thread (row block, item) walks RB consecutive rows of one item (an
// interleaved piece, a half-split piece pair or a pass-through piece).  The angles of the first
// row of the block (and of the first row of a new unit) come from rope_cs (double reduction);
// every next row multiplies by e^{i theta_j} -- a few fp32 FMAs per pair instead of a double
// reduction and sin/cos per element, so the kernel streams at HBM rate.
constexpr int ROPE_RB = 16;
template <typename T, int D>
__global__ void __launch_bounds__(256) rope_walk_kernel(const T* __restrict__ X, T* __restrict__ Y, int64_t rows,
                                                        int T_, int64_t pos0, const int64_t* __restrict__ pos,
                                                        const __grid_constant__ RopeSpec rs) {
  pdl_wait();
  pdl_trigger();
  constexpr int VEC = 16 / sizeof(T);
  const bool neox = rs.style == EVA_ROPE_NEOX;
  const int nrot = neox ? rs.rd / (2 * VEC) : rs.rd / VEC;
  const int per = nrot + (D - rs.rd) / VEC;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int it = (int)(i % per);
  const int64_t r0 = (i / per) * ROPE_RB;
  if (r0 >= rows) return;
  const int64_t r1 = min(rows, r0 + ROPE_RB);
  if (it >= nrot) {  // pass-through piece
    if (X == Y) return;
    const int ch0 = rs.rd + (it - nrot) * VEC;
    for (int64_t r = r0; r < r1; ++r)
      *reinterpret_cast<uint4*>(Y + r * D + ch0) = ldg16_stream(X + r * D + ch0);
    return;
  }
  const int np = neox ? VEC : VEC / 2;                  // pairs of this item
  const int j0 = neox ? it * VEC : it * (VEC / 2);      // first pair index
  const int cha = neox ? it * VEC : it * VEC, chb = cha + rs.rd / 2;
  float c[VEC], sn[VEC], sc[VEC], ss[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q)
    if (q < np) rope_cs(1, j0 + q, rs, sc[q], ss[q]);  // one-row step (sign included)
  // 8 rows per batch: their loads are issued before any store (the call may run in place, but a
  // thread only ever writes the pieces it has read)
  constexpr int NB = 8;
  for (int64_t rb = r0; rb < r1; rb += NB) {
    uint4 xa[NB], xb[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      if (rb + k < r1) {
        xa[k] = ldg16_stream(X + (rb + k) * D + cha);
        if (neox) xb[k] = ldg16_stream(X + (rb + k) * D + chb);
      }
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int64_t r = rb + k;
      if (r >= r1) break;
      const int64_t u = r / T_, t = r - u * T_;
      if (r == r0 || t == 0) {
        const int64_t p = (pos ? pos[u] : pos0) + t;
#pragma unroll
        for (int q = 0; q < VEC; ++q)
          if (q < np) rope_cs(p, j0 + q, rs, c[q], sn[q]);
      }
      if (neox) {
        float va[VEC], vb[VEC];
        unpack16<T>(xa[k], va);
        unpack16<T>(xb[k], vb);
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          const float x0 = va[q], x1 = vb[q];
          va[q] = x0 * c[q] - x1 * sn[q];
          vb[q] = x0 * sn[q] + x1 * c[q];
        }
        *reinterpret_cast<uint4*>(Y + r * D + cha) = pack16<T>(va);
        *reinterpret_cast<uint4*>(Y + r * D + chb) = pack16<T>(vb);
      } else {
        float v[VEC];
        unpack16<T>(xa[k], v);
#pragma unroll
        for (int q = 0; q < VEC / 2; ++q) {
          const float x0 = v[2 * q], x1 = v[2 * q + 1];
          v[2 * q] = x0 * c[q] - x1 * sn[q];
          v[2 * q + 1] = x0 * sn[q] + x1 * c[q];
        }
        *reinterpret_cast<uint4*>(Y + r * D + cha) = pack16<T>(v);
      }
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        if (q < np) {
          const float cn = c[q] * sc[q] - sn[q] * ss[q];
          sn[q] = sn[q] * sc[q] + c[q] * ss[q];
          c[q] = cn;
        }
      }
    }
  }
}

// The key transform of the fused producer: rotate the piece (row r of the chunk, channels ch0)
// at position r0 + r and store it to Kr.  Half-split pairs live in lanes gl and gl ^ off
// (off = rd / (2 VEC), a power of two), exchanged by shuffles -- every lane takes part.
template <typename T, int D>
struct RopeKX {
  static constexpr int VEC = 16 / sizeof(T);
  const RopeSpec& rs;  // the kernel's __grid_constant__ parameter
  int64_t r0;
  T* Krc;
  int step;            // rows between this lane's consecutive calls (the summariser's 4 * RPW)
  // A lane's calls walk rows r, r + step, ...: the angles of its pairs come from double
  // precision at the first call, then by the recurrence e^{i (p + step) theta} =
  // e^{i p theta} e^{i step theta} (fp32, at most 16 steps).
  mutable float c[VEC], s[VEC], sc[VEC], ss[VEC];
  mutable bool init = false;
  __device__ __forceinline__ void angles(int64_t pos, int j0, int np) const {
#pragma unroll
    for (int jj = 0; jj < VEC; ++jj) {
      if (jj < np) {
        rope_cs(pos, j0 + jj, rs, c[jj], s[jj]);
        rope_cs((int64_t)step, j0 + jj, rs, sc[jj], ss[jj]);
      }
    }
  }
  __device__ __forceinline__ void next(int np) const {
#pragma unroll
    for (int jj = 0; jj < VEC; ++jj) {
      if (jj < np) {
        const float cn = c[jj] * sc[jj] - s[jj] * ss[jj];
        s[jj] = s[jj] * sc[jj] + c[jj] * ss[jj];
        c[jj] = cn;
      }
    }
  }
  __device__ __forceinline__ void operator()(int r, int ch0, uint4& x, bool valid) const {
    if (rs.style == EVA_ROPE_NEOX) {
      const int off = rs.rd / (2 * VEC);
      uint4 y;
      y.x = __shfl_xor_sync(0xffffffffu, x.x, off);
      y.y = __shfl_xor_sync(0xffffffffu, x.y, off);
      y.z = __shfl_xor_sync(0xffffffffu, x.z, off);
      y.w = __shfl_xor_sync(0xffffffffu, x.w, off);
      if (ch0 < rs.rd) {
        const bool first = ch0 < rs.rd / 2;
        if (!init) angles(r0 + r, first ? ch0 : ch0 - rs.rd / 2, VEC);
        else next(VEC);
        float vx[VEC], vy[VEC];
        unpack16<T>(x, vx);
        unpack16<T>(y, vy);
#pragma unroll
        for (int jj = 0; jj < VEC; ++jj)
          vx[jj] = first ? vx[jj] * c[jj] - vy[jj] * s[jj] : vy[jj] * s[jj] + vx[jj] * c[jj];
        x = pack16<T>(vx);
      }
    } else if (ch0 < rs.rd) {
      if (!init) angles(r0 + r, ch0 / 2, VEC / 2);
      else next(VEC / 2);
      float v[VEC];
      unpack16<T>(x, v);
#pragma unroll
      for (int jj = 0; jj < VEC / 2; ++jj) {
        const float x0 = v[2 * jj], x1 = v[2 * jj + 1];
        v[2 * jj] = x0 * c[jj] - x1 * s[jj];
        v[2 * jj + 1] = x0 * s[jj] + x1 * c[jj];
      }
      x = pack16<T>(v);
    }
    init = true;
    if (valid && Krc) *reinterpret_cast<uint4*>(Krc + (size_t)r * D + ch0) = x;
  }
};

// grid (nC + tail, bh_count), 128 threads.  CTA x < nC: chunk x -- its keys are rotated as
// they are loaded (and stored to Kr), summarised from the rotated values, and its query rows
// rotated into Qr; CTA x = nC rotates the trailing partial chunk's rows only.
template <typename T, int D, int NI>
__global__ void __launch_bounds__(128) rope_summarize_kernel(eva_config cfg, const __grid_constant__ RopeSpec rs,
                                                            const T* __restrict__ Q, const T* __restrict__ K,
                                                            const T* __restrict__ V, const float* __restrict__ eps,
                                                            T* __restrict__ Qr, T* __restrict__ Kr,
                                                            T* __restrict__ Ksum, T* __restrict__ Vsum) {
  pdl_wait();
  pdl_trigger();
  const int C = cfg.chunk, Tn = cfg.T, nC = Tn / C;
  const int c = blockIdx.x, u = blockIdx.y;
  const size_t ub = (size_t)u * Tn;
  const int r0 = c * C, r1 = min(Tn, r0 + C);
  const int per = rope_items<T, D>(rs);
  // the query rows of this chunk (and, for the tail CTA, the key rows too).  Qr == Kr == NULL:
  // summaries only (eva_attn_prefill_rope rotates Q and K inside the prefill kernel).
  if (Qr) {
    for (int i = threadIdx.x; i < (r1 - r0) * per; i += blockDim.x) {
      const int r = r0 + i / per, it = i % per;
      rope_row_item<T, D>(Q + (ub + r) * D, Qr + (ub + r) * D, r, it, rs);
      if (c >= nC) rope_row_item<T, D>(K + (ub + r) * D, Kr + (ub + r) * D, r, it, rs);
    }
  }
  if (c >= nC) return;
  const T* Kc = K + (ub + (size_t)r0) * D;
  const T* Vc = V + (ub + (size_t)r0) * D;
  constexpr int RPW_ = 32 / (D / (16 / (int)sizeof(T)));
  RopeKX<T, D> kx{rs, (int64_t)r0, Kr ? Kr + (ub + (size_t)r0) * D : nullptr, 4 * RPW_};
  summarize_chunk_reg<T, D, NI>([&](int r) { return Kc + (size_t)r * D; }, [&](int r) { return Vc + (size_t)r * D; },
                                C, eps ? eps + ((size_t)u * nC + c) * D : nullptr, (uint32_t)(cfg.bh_begin + u),
                                (uint32_t)c, cfg, Ksum + ((size_t)u * nC + c) * D, Vsum + ((size_t)u * nC + c) * D,
                                nullptr, kx);
}

template <typename T, int D, int NI>
__global__ void __launch_bounds__(128) summarize_bcast_kernel(eva_config cfg, const T* __restrict__ K,
                                                             const T* __restrict__ V,
                                                             const float* __restrict__ eps,
                                                             const unsigned long long* __restrict__ dst_k,
                                                             const unsigned long long* __restrict__ dst_v,
                                                             int n_dst, int dst_rows, int c0) {
  __shared__ __align__(16) T sk[D];
  __shared__ __align__(16) T sv[D];
  pdl_wait();
  pdl_trigger();
  const int C = cfg.chunk, nC = cfg.T / C;
  const int c = blockIdx.x, u = blockIdx.y;
  const T* Kc = K + ((size_t)u * cfg.T + (size_t)c * C) * D;
  const T* Vc = V + ((size_t)u * cfg.T + (size_t)c * C) * D;
  summarize_chunk_reg<T, D, NI>([&](int r) { return Kc + (size_t)r * D; }, [&](int r) { return Vc + (size_t)r * D; },
                                C, eps ? eps + ((size_t)u * nC + c) * D : nullptr,
                                (uint32_t)(cfg.bh_begin + u), (uint32_t)(c0 + c), cfg, sk, sv);
  __syncthreads();
  constexpr int PCS = D * (int)sizeof(T) / 16;  // 16-byte pieces per row
  const size_t row = ((size_t)u * dst_rows + (size_t)(c0 + c)) * D;
  for (int i = threadIdx.x; i < n_dst * PCS * 2; i += blockDim.x) {
    const int which = i / (n_dst * PCS), rest = i % (n_dst * PCS), dst = rest / PCS, pc = rest % PCS;
    const uint4 val = reinterpret_cast<const uint4*>(which ? sv : sk)[pc];
    T* base = reinterpret_cast<T*>(which ? dst_v[dst] : dst_k[dst]);
    reinterpret_cast<uint4*>(base + row)[pc] = val;
  }
}


// ============================================================================ SIMT prefill
// One CTA = one unit x QT queries.  G threads cooperate on one query (thread gi
// owns channels gi, gi+G, ... -> conflict-free smem reads); key/value tiles of
// KT rows are staged in shared memory as fp32.  Two segments are walked in
// order: the summary prefix [0, nsum(n_last)) and the local span
// [lo(n_first), n_last]; each query applies its own (lo, nsum) (P:124 mask).
template <typename T, int D>
__global__ void __launch_bounds__(128) prefill_simt_kernel(eva_config cfg, PrefillRange rg,
                                                           const T* __restrict__ Q,
                                                           const T* __restrict__ K,
                                                           const T* __restrict__ V,
                                                           const T* __restrict__ Ksum,
                                                           const T* __restrict__ Vsum,
                                                           T* __restrict__ O, float* __restrict__ lse) {
  constexpr int G = D >= 32 ? D / 32 : 1;
  constexpr int CH = D / G;
  constexpr int QT = 128 / G;
  constexpr int KT = 32;
  __shared__ float Ks[KT][D];
  __shared__ float Vs[KT][D];

  // Absolute positions: query row i is position q0 + i, key/value row r is position k0 + r,
  // summary row c is chunk c (rows per unit: nq, nkv, nsl).
  const int C = cfg.chunk, W = cfg.window;
  const int64_t q0 = rg.q0, k0 = rg.k0, qend = rg.q0 + rg.nq;
  const int u = blockIdx.y;
  const int64_t n0 = q0 + (int64_t)blockIdx.x * QT;
  const int tid = threadIdx.x, qi = tid / G, gi = tid % G;
  const int64_t n = n0 + qi;
  const bool valid = n < qend;
  const int64_t nlast = min(n0 + QT - 1, qend - 1);
  const Vis vme = visible_set(valid ? n : nlast, C, W, cfg.mode, qend);
  const Vis vfirst = visible_set(n0, C, W, cfg.mode, qend);
  const Vis vlast = visible_set(nlast, C, W, cfg.mode, qend);
  const bool noncausal = cfg.mode == EVA_NONCAUSAL;

  float q[CH], acc[CH];
  const T* qp = Q + ((size_t)u * rg.nq + (size_t)((valid ? n : nlast) - q0)) * D;
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    q[j] = Elem<T>::to_f(qp[j * G + gi]) * cfg.scale;
    acc[j] = 0.f;
  }
  float m = -INFINITY, l = 0.f;

  for (int seg = 0; seg < 2; ++seg) {
    // kb/vb indexed by absolute position (local segment) or chunk (summary segment)
    const T* kb = seg == 0 ? Ksum + (size_t)u * rg.nsl * D : K + ((size_t)u * rg.nkv - k0) * D;
    const T* vb = seg == 0 ? Vsum + (size_t)u * rg.nsl * D : V + ((size_t)u * rg.nkv - k0) * D;
    const int64_t beg = seg == 0 ? 0 : vfirst.lo;
    const int64_t end = seg == 0 ? (noncausal ? (int64_t)rg.nsl : vlast.s1) : vlast.hi;
    const float bias = seg == 0 ? cfg.summary_bias : 0.f;
    for (int64_t t0 = beg; t0 < end; t0 += KT) {
      const int nk = (int)min((int64_t)KT, end - t0);
      __syncthreads();
      for (int i = tid; i < nk * D; i += 128) {
        const int r = i / D, cc = i % D;
        Ks[r][cc] = Elem<T>::to_f(kb[(size_t)(t0 + r) * D + cc]);
        Vs[r][cc] = Elem<T>::to_f(vb[(size_t)(t0 + r) * D + cc]);
      }
      __syncthreads();
      for (int j = 0; j < nk; ++j) {
        float s = 0.f;
#pragma unroll
        for (int c2 = 0; c2 < CH; ++c2) s += q[c2] * Ks[j][c2 * G + gi];
        s = group_sum<G>(s) + bias;
        const int64_t t = t0 + j;
        const bool vis = valid && (seg == 0 ? (t < vme.s1 || t >= vme.s2) : (t >= vme.lo && t < vme.hi));
        if (vis) {
          const float mn = fmaxf(m, s);
          const float corr = __expf(m - mn);
          const float p = __expf(s - mn);
          l = l * corr + p;
#pragma unroll
          for (int c2 = 0; c2 < CH; ++c2) acc[c2] = acc[c2] * corr + p * Vs[j][c2 * G + gi];
          m = mn;
        }
      }
    }
  }
  if (valid) {
    const float il = 1.0f / l;
    T* op = O + ((size_t)u * rg.nq + (size_t)(n - q0)) * D;
#pragma unroll
    for (int j = 0; j < CH; ++j) op[j * G + gi] = Elem<T>::from_f(acc[j] * il);
    if (lse && gi == 0) lse[(size_t)u * rg.nq + (n - q0)] = m + logf(l);
  }
}

// ============================================================================ cache append
// One launch, flat grid of 128-thread CTAs:
//   blockIdx.x <  n_copy : ring write of the last min(n_new, W) tokens of every unit
//                          (one 16-byte piece of K and of V per thread; if do_ring)
//   blockIdx.x >= n_copy : CTA summarises (unit, chunk) = divmod(x - n_copy, n_chunks)
//                          (if do_sum)
// Rows of a chunk come from K_new (positions >= pos) or the ring (positions < pos).
template <typename T, int D, int SUMM>  // SUMM: 0 warp, 1 staged CTA, 2/4/8 register NI
__global__ void __launch_bounds__(128) append_kernel(eva_cache c, const T* __restrict__ Kn,
                                                     const T* __restrict__ Vn,
                                                     const float* __restrict__ eps, int n_new,
                                                     int n_copy, int do_sum, int64_t chunk0,
                                                     int n_chunks) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int VEC = 16 / sizeof(T);
  constexpr int PPR = D / VEC;
  const int W = c.cfg.window, C = c.cfg.chunk;
  const int64_t pos = c.pos;
  const int keep = min(n_new, W);
  if ((int)blockIdx.x < n_copy) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // piece index
    const int64_t per_unit = (int64_t)keep * PPR;
    if (i >= per_unit * c.cfg.bh_count) return;
    const int u = (int)(i / per_unit);
    const int rem = (int)(i % per_unit);
    const int r = n_new - keep + rem / PPR, cc = (rem % PPR) * VEC;
    const size_t slot = (size_t)((pos + r) % W);
    T* rk = static_cast<T*>(c.ring_k) + (size_t)u * W * D;
    T* rv = static_cast<T*>(c.ring_v) + (size_t)u * W * D;
    const T* kn = Kn + (size_t)u * n_new * D;
    const T* vn = Vn + (size_t)u * n_new * D;
    *reinterpret_cast<uint4*>(rk + slot * D + cc) = *reinterpret_cast<const uint4*>(kn + (size_t)r * D + cc);
    *reinterpret_cast<uint4*>(rv + slot * D + cc) = *reinterpret_cast<const uint4*>(vn + (size_t)r * D + cc);
    return;
  }
  if (!do_sum) return;
  const int x = (int)blockIdx.x - n_copy;
  constexpr bool CTA_SUMM = SUMM != 0;
  const int per = CTA_SUMM ? n_chunks : (n_chunks + 3) / 4;
  const int u = x / per;
  const int ci = CTA_SUMM ? x % per : (x % per) * 4 + (int)(threadIdx.x >> 5);
  if (u >= c.cfg.bh_count || ci >= n_chunks) return;
  const T* rk = static_cast<const T*>(c.ring_k) + (size_t)u * W * D;
  const T* rv = static_cast<const T*>(c.ring_v) + (size_t)u * W * D;
  const T* kn = Kn + (size_t)u * n_new * D;
  const T* vn = Vn + (size_t)u * n_new * D;
  const int64_t chunk = chunk0 + ci;
  const int64_t p0 = chunk * C;
  auto rowK = [&](int i) -> const T* {
    const int64_t p = p0 + i;
    return p >= pos ? kn + (size_t)(p - pos) * D : rk + (size_t)(p % W) * D;
  };
  auto rowV = [&](int i) -> const T* {
    const int64_t p = p0 + i;
    return p >= pos ? vn + (size_t)(p - pos) * D : rv + (size_t)(p % W) * D;
  };
  const float* e = eps ? eps + ((size_t)u * c.cap_chunks + chunk) * D : nullptr;
  T* sk = static_cast<T*>(c.sum_k) + ((size_t)u * c.cap_chunks + chunk) * D;
  T* sv = static_cast<T*>(c.sum_v) + ((size_t)u * c.cap_chunks + chunk) * D;
  if constexpr (SUMM >= 2)
    summarize_chunk_reg<T, D, (SUMM >= 2 ? SUMM : 2)>(rowK, rowV, C, e, (uint32_t)(c.cfg.bh_begin + u),
                                                       (uint32_t)chunk, c.cfg, sk, sv);
  else if constexpr (SUMM == 1)
    summarize_chunk_cta<T, D>(rowK, rowV, C, e, (uint32_t)(c.cfg.bh_begin + u), (uint32_t)chunk,
                              c.cfg, sk, sv, smem);
  else
    summarize_chunk_warp<T, D>(rowK, rowV, C, e, (uint32_t)(c.cfg.bh_begin + u), (uint32_t)chunk,
                               c.cfg, sk, sv);
}

// ============================================================================ ragged step
// Per-unit positions: unit u holds pos[u] tokens.  One CTA per
// unit appends its new token at position p = pos[u] (ring slot p mod W -- position p - W,
// which query p no longer sees), summarises chunk (p+1)/C - 1 when p completes it (rows from
// the ring, the newest row from Knew: no read-after-write through the read-only path), and
// advances pos[u].  The decode launch that follows reads each unit's own pos.
template <typename T, int D, int NI>
__global__ void __launch_bounds__(128) ragged_append_kernel(eva_cache c, int64_t* __restrict__ pos,
                                                            const T* __restrict__ Knew,
                                                            const T* __restrict__ Vnew,
                                                            const float* __restrict__ eps) {
  pdl_wait();
  pdl_trigger();
  constexpr int VEC = 16 / sizeof(T);
  const int u = blockIdx.x;
  const int W = c.cfg.window, C = c.cfg.chunk;
  const int64_t p = pos[u];
  T* rk = static_cast<T*>(c.ring_k) + (size_t)u * W * D;
  T* rv = static_cast<T*>(c.ring_v) + (size_t)u * W * D;
  const T* kn = Knew + (size_t)u * D;
  const T* vn = Vnew + (size_t)u * D;
  const size_t slot = (size_t)(p % W);
  for (int i = threadIdx.x; i < D / VEC; i += blockDim.x) {
    reinterpret_cast<uint4*>(rk + slot * D)[i] = reinterpret_cast<const uint4*>(kn)[i];
    reinterpret_cast<uint4*>(rv + slot * D)[i] = reinterpret_cast<const uint4*>(vn)[i];
  }
  const int64_t chunk = (p + 1) / C - 1;
  if ((p + 1) % C == 0 && chunk < c.cap_chunks) {  // uniform over the CTA
    const int64_t p0 = chunk * C;
    auto rowK = [&](int i) -> const T* {
      const int64_t q = p0 + i;
      return q == p ? kn : rk + (size_t)(q % W) * D;
    };
    auto rowV = [&](int i) -> const T* {
      const int64_t q = p0 + i;
      return q == p ? vn : rv + (size_t)(q % W) * D;
    };
    summarize_chunk_reg<T, D, NI>(rowK, rowV, C, eps ? eps + ((size_t)u * c.cap_chunks + chunk) * D : nullptr,
                                  (uint32_t)(c.cfg.bh_begin + u), (uint32_t)chunk, c.cfg,
                                  static_cast<T*>(c.sum_k) + ((size_t)u * c.cap_chunks + chunk) * D,
                                  static_cast<T*>(c.sum_v) + ((size_t)u * c.cap_chunks + chunk) * D);
  }
  __syncthreads();
  if (threadIdx.x == 0) pos[u] = p + 1;
}

// ============================================================================ decode
// grid (bh_count, splits), block 128 (4 warps).  The visible list of query
// n = pos-1 is the summary prefix [0, nsum) followed by the ring positions
// [lo, n] (slot p mod W, at most two contiguous ring segments).  Split s takes
// entries [s*E/S, (s+1)*E/S).  Bandwidth layout: a row of D elements is read by a
// group of TPR = D/VEC lanes with one 16-byte load each (VEC elements per lane);
// a warp covers RPW = 32/TPR rows per load and UNROLL row-blocks per iteration, so
// every lane has 2*UNROLL independent 16-byte loads in flight.  Each lane group
// keeps its own online-softmax state (m, l, acc[VEC]); groups and warps are merged
// at the end (shuffles, then shared memory).
// Fused decode step (FUSED): the cache descriptor already counts the new token (pos = p+1)
// and Knew/Vnew hold it; entry n = p is read from Knew/Vnew instead of the ring, and the
// split-0 CTA of each unit writes it to ring slot p mod W (which held position p - W,
// invisible to query p).  Used for steps that do not complete a chunk.
// RoPE of the VEC channels [ch0, ch0 + VEC) a lane holds (as floats) at position pos (R18/R19):
// interleaved pairs are inside the lane; a half-split partner is rd/2 channels away, i.e. in lane
// gl ^ (rd / (2 VEC)) of the same row group (a power of two, checked by the C ABI) -- exchanged by
// shuffles, every lane of the warp taking part.
template <int VEC>
__device__ __forceinline__ void rope_vals(float (&v)[VEC], int64_t pos, int ch0, const RopeSpec& rs) {
  if (rs.style == EVA_ROPE_NEOX) {
    const int off = rs.rd / (2 * VEC);
    float y[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) y[j] = __shfl_xor_sync(0xffffffffu, v[j], off);
    if (ch0 < rs.rd) {
      const bool first = ch0 < rs.rd / 2;
      const int j0 = first ? ch0 : ch0 - rs.rd / 2;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        float c, sn;
        rope_cs(pos, j0 + j, rs, c, sn);
        v[j] = first ? v[j] * c - y[j] * sn : y[j] * sn + v[j] * c;
      }
    }
  } else if (ch0 < rs.rd) {
#pragma unroll
    for (int j = 0; j < VEC; j += 2) {
      float c, sn;
      rope_cs(pos, (ch0 + j) / 2, rs, c, sn);
      const float x0 = v[j], x1 = v[j + 1];
      v[j] = x0 * c - x1 * sn;
      v[j + 1] = x0 * sn + x1 * c;
    }
  }
}

// The summariser's loads in the RoPE ragged step: the newest key row (K_new, un-rotated in
// memory) is served from the lane's rotated piece, every other row from global memory.
template <typename T, int D>
struct LdRopeNew {
  const T* kn;  // K_new row of this unit
  uint4 piece;  // this lane's rotated piece of it (channels ch0 .. ch0 + VEC)
  template <typename P>
  __device__ __forceinline__ uint4 operator()(const P* p) const {
    const T* q = reinterpret_cast<const T*>(p);
    return (q >= kn && q < kn + D) ? piece : ldg16_stream(p);
  }
};

template <typename T, int D, bool FUSED = false, bool RAGGED = false, bool ROPE = false>
__global__ void __launch_bounds__(128, 6) decode_kernel(eva_cache c, const T* __restrict__ Q,
                                                     T* __restrict__ O, float* __restrict__ lse,
                                                     float* __restrict__ ws, int S_,
                                                     const T* __restrict__ Knew,
                                                     const T* __restrict__ Vnew,
                                                     int64_t* __restrict__ pos_dev,
                                                     const float* __restrict__ ragged_eps,
                                                     const __grid_constant__ RopeSpec rs) {
  static_assert(!ROPE || (FUSED && RAGGED), "RoPE is folded into the one-launch ragged step");
  constexpr int VEC = 16 / sizeof(T);
  constexpr int TPR = D / VEC;          // lanes per row
  constexpr int RPW = 32 / TPR;         // rows per warp-wide load
  constexpr int UNROLL = 4;
  constexpr int ROWS_IT = RPW * UNROLL; // rows per warp iteration
  constexpr int NW = 4;
  static_assert(TPR >= 1 && TPR <= 32 && 32 % TPR == 0, "bad D/VEC");
  __shared__ float sm_m[NW], sm_l[NW];
  __shared__ float sm_acc[NW][D];
  pdl_wait();
  pdl_trigger();
  const int u = blockIdx.x, S = S_, s = blockIdx.y;
  const int W = c.cfg.window, C = c.cfg.chunk;
  // workspace layout (split-K only): merge counters at a FIXED offset (one per unit, padded to
  // 16 bytes) then the partials (m, l, acc[D]) per (unit, split).  The split count changes with
  // the position (E/64), so anything placed after the partials would move between calls.
  unsigned* counters = reinterpret_cast<unsigned*>(ws);
  float* parts = ws + ((size_t)gridDim.x + 3) / 4 * 4;
  // ragged (its own instantiations, so the uniform kernel is unchanged): this unit's
  // position; the fused ragged step is called before the advance (pos[u] = p = n)
  const int64_t n = RAGGED ? (FUSED ? pos_dev[u] : pos_dev[u] - 1) : c.pos - 1;
  const Range r = mask_range(n, C, W, c.cfg.mode);
  // 32-bit entry indices: E <= nsum + W stays far below 2^31 for any cache that fits HBM
  const int ns = (int)r.nsum;
  const int E = ns + (int)(n - r.lo + 1);
  const int e0 = (int)((int64_t)E * s / S), e1 = (int)((int64_t)E * (s + 1) / S);
  const int slot0 = (int)(r.lo % W) - ns;  // ring slot of entry e >= ns is slot0 + e (mod W)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / TPR, gl = lane % TPR;
  const int ch0 = gl * VEC;
  const T* sk = static_cast<const T*>(c.sum_k) + (size_t)u * c.cap_chunks * D + ch0;
  const T* sv = static_cast<const T*>(c.sum_v) + (size_t)u * c.cap_chunks * D + ch0;
  const T* rk = static_cast<const T*>(c.ring_k) + (size_t)u * W * D + ch0;
  const T* rv = static_cast<const T*>(c.ring_v) + (size_t)u * W * D + ch0;
  float q[VEC], acc[VEC];
  load_vec<T, VEC>(Q + (size_t)u * D + ch0, q);
  uint4 kn_rot = make_uint4(0u, 0u, 0u, 0u);
  if constexpr (ROPE) {
    // q and the new key at this unit's position n, in registers (RoPE(q), RoPE(k_new) are
    // never written; the rotated key goes to its ring slot in dtype, like the two-pass path)
    rope_vals<VEC>(q, n, ch0, rs);
    float kv[VEC];
    load_vec<T, VEC>(Knew + (size_t)u * D + ch0, kv);
    rope_vals<VEC>(kv, n, ch0, rs);
    kn_rot = pack16<T>(kv);
  }
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    q[j] *= c.cfg.scale;
    acc[j] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int eb = e0 + warp * ROWS_IT; eb < e1; eb += NW * ROWS_IT) {
    uint4 kx[UNROLL], vx[UNROLL];
    bool ok[UNROLL];
#pragma unroll
    for (int i = 0; i < UNROLL; ++i) {
      const int e = eb + i * RPW + grp;
      ok[i] = e < e1;
      const bool is_new = FUSED && e == E - 1;
      const T *kp, *vp;
      if (e < ns) {
        kp = sk + (size_t)e * D;
        vp = sv + (size_t)e * D;
      } else if (FUSED && e == E - 1) {  // the token being appended in this launch
        kp = Knew + (size_t)u * D + ch0;
        vp = Vnew + (size_t)u * D + ch0;
      } else {
        int slot = slot0 + e;
        if (slot >= W) slot -= W;
        kp = rk + (size_t)slot * D;
        vp = rv + (size_t)slot * D;
      }
      if (ok[i]) {
        kx[i] = (ROPE && is_new) ? kn_rot : ldg16_stream(kp);
        vx[i] = ldg16_stream(vp);
      }
    }
    float sc[UNROLL];
    float mx = m;
#pragma unroll
    for (int i = 0; i < UNROLL; ++i) {
      float d = 0.f;
      if (ok[i]) {
        float k[VEC];
        unpack16<T>(kx[i], k);
#pragma unroll
        for (int j = 0; j < VEC; ++j) d += q[j] * k[j];
      }
      d = group_sum<TPR>(d);
      sc[i] = ok[i] ? (eb + i * RPW + grp < ns ? d + c.cfg.summary_bias : d) : -INFINITY;
      mx = fmaxf(mx, sc[i]);
    }
    if (mx == -INFINITY) continue;
    const float corr = __expf(m - mx);
    l *= corr;
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] *= corr;
#pragma unroll
    for (int i = 0; i < UNROLL; ++i) {
      const float p = __expf(sc[i] - mx);
      l += p;
      if (ok[i]) {
        float v[VEC];
        unpack16<T>(vx[i], v);
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] += p * v[j];
      }
    }
    m = mx;
  }
  // merge the RPW lane groups of this warp (butterfly over group ids)
#pragma unroll
  for (int o = TPR; o < 32; o <<= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float l2 = __shfl_xor_sync(0xffffffffu, l, o);
    const float M = fmaxf(m, m2);
    const float f1 = m == -INFINITY ? 0.f : __expf(m - M);
    const float f2 = m2 == -INFINITY ? 0.f : __expf(m2 - M);
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = acc[j] * f1 + __shfl_xor_sync(0xffffffffu, acc[j], o) * f2;
    l = l * f1 + l2 * f2;
    m = M;
  }
  if (lane == 0) { sm_m[warp] = m; sm_l[warp] = l; }
  if (grp == 0) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) sm_acc[warp][ch0 + j] = acc[j];
  }
  if constexpr (FUSED) {
    // append: split 0 writes the new token to ring slot p mod W (position p - W, never read
    // by this launch); issued after the attention loads so it does not delay them
    if (s == 0 && warp == 1) {
      const size_t slot = (size_t)(n % W);
      T* wk = static_cast<T*>(c.ring_k) + ((size_t)u * W + slot) * D;
      T* wv = static_cast<T*>(c.ring_v) + ((size_t)u * W + slot) * D;
      if constexpr (ROPE) {
        if (grp == 0) *reinterpret_cast<uint4*>(wk + ch0) = kn_rot;
        for (int i = lane; i < D; i += 32) wv[i] = Vnew[(size_t)u * D + i];
      } else {
        for (int i = lane; i < D; i += 32) {
          wk[i] = Knew[(size_t)u * D + i];
          wv[i] = Vnew[(size_t)u * D + i];
        }
      }
    }
  }
  __syncthreads();
  if constexpr (FUSED && RAGGED) {
    // the chunk this token completes (per unit): all four warps of split 0 summarise it with the
    // register summariser (re-reading its rows: the decode's 80-register budget) -- rows from the
    // ring, the newest from Knew (its ring slot is written by warp 1 above).  The same arithmetic
    // as the cache append, so the summaries equal eva_decode_step's bit for bit.  (One warp with
    // the warp summariser kept 1/64 of the CTAs ~30 us longer per step at configs[3] with the
    // units 64 tokens apart: 0.87 of HBM vs 0.99 uniform.)
    const int64_t chunk = (n + 1) / C - 1;
    if (s == 0 && (n + 1) % C == 0 && chunk < c.cap_chunks) {
      const int64_t p0 = chunk * C;
      const T* rk0 = static_cast<const T*>(c.ring_k) + (size_t)u * W * D;
      const T* rv0 = static_cast<const T*>(c.ring_v) + (size_t)u * W * D;
      auto rowK = [&](int i) -> const T* {
        const int64_t q = p0 + i;
        return q == n ? Knew + (size_t)u * D : rk0 + (size_t)(q % W) * D;
      };
      auto rowV = [&](int i) -> const T* {
        const int64_t q = p0 + i;
        return q == n ? Vnew + (size_t)u * D : rv0 + (size_t)(q % W) * D;
      };
      if constexpr (ROPE) {
        // the ring rows are rotated already; the newest row's rotated piece comes from kn_rot
        summarize_chunk_reg<T, D, 16, decltype(rowK), decltype(rowV), NoKXform, LdRopeNew<T, D>, true>(
            rowK, rowV, C, ragged_eps ? ragged_eps + ((size_t)u * c.cap_chunks + chunk) * D : nullptr,
            (uint32_t)(c.cfg.bh_begin + u), (uint32_t)chunk, c.cfg,
            static_cast<T*>(c.sum_k) + ((size_t)u * c.cap_chunks + chunk) * D,
            static_cast<T*>(c.sum_v) + ((size_t)u * c.cap_chunks + chunk) * D, nullptr, NoKXform(),
            LdRopeNew<T, D>{Knew + (size_t)u * D, kn_rot});
      } else {
        summarize_chunk_reg<T, D, 16, decltype(rowK), decltype(rowV), NoKXform, LdGlobalStream, true>(
            rowK, rowV, C, ragged_eps ? ragged_eps + ((size_t)u * c.cap_chunks + chunk) * D : nullptr,
            (uint32_t)(c.cfg.bh_begin + u), (uint32_t)chunk, c.cfg,
            static_cast<T*>(c.sum_k) + ((size_t)u * c.cap_chunks + chunk) * D,
            static_cast<T*>(c.sum_v) + ((size_t)u * c.cap_chunks + chunk) * D);
      }
    }
  }
  if (warp != 0) return;
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < NW; ++w) M = fmaxf(M, sm_m[w]);
  float f[NW], L = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    f[w] = sm_m[w] == -INFINITY ? 0.f : __expf(sm_m[w] - M);
    L += f[w] * sm_l[w];
  }
  for (int ch = lane; ch < D; ch += 32) {
    float o = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) o += f[w] * sm_acc[w][ch];
    if (S == 1) {
      O[(size_t)u * D + ch] = Elem<T>::from_f(o / L);
    } else {
      parts[((size_t)u * S + s) * (D + 2) + 2 + ch] = o;
    }
  }
  if (S == 1) {
    if (lane == 0 && lse) lse[u] = M + logf(L);
    if constexpr (RAGGED && FUSED) {
      if (lane == 0) pos_dev[u] = n + 1;
    }
    return;
  }
  if (lane == 0) {
    float* p = parts + ((size_t)u * S + s) * (D + 2);
    p[0] = M;
    p[1] = L;
  }
  // split-K: the last CTA of this unit to finish merges the S partials (no second launch).
  // Counters (at the front of the workspace) are left at zero for the next call.
  __threadfence();
  __syncwarp();
  unsigned prev = 0;
  if (lane == 0) prev = atomicAdd(&counters[u], 1u);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != (unsigned)(S - 1)) return;
  __threadfence();
  const volatile float* pu = parts + (size_t)u * S * (D + 2);
  float Mg = -INFINITY;
  for (int k = 0; k < S; ++k) Mg = fmaxf(Mg, pu[(size_t)k * (D + 2)]);
  float Lg = 0.f;
  for (int k = 0; k < S; ++k) {
    const float mk = pu[(size_t)k * (D + 2)];
    Lg += (mk == -INFINITY ? 0.f : __expf(mk - Mg)) * pu[(size_t)k * (D + 2) + 1];
  }
  for (int ch = lane; ch < D; ch += 32) {
    float o = 0.f;
    for (int k = 0; k < S; ++k) {
      const float mk = pu[(size_t)k * (D + 2)];
      if (mk != -INFINITY) o += __expf(mk - Mg) * pu[(size_t)k * (D + 2) + 2 + ch];
    }
    O[(size_t)u * D + ch] = Elem<T>::from_f(o / Lg);
  }
  if (lane == 0) {
    if (lse) lse[u] = Mg + logf(Lg);
    counters[u] = 0u;
    if constexpr (RAGGED && FUSED) pos_dev[u] = n + 1;  // every split has read pos[u]
  }
}

// ============================================================================ cache load
// Prefill hand-off with summaries already computed: one flat grid of 16-byte copies,
//   pieces [0, n_ring)            : the last keep = min(n, W) tokens -> ring slots (p mod W)
//   pieces [n_ring, n_ring+n_sum) : Ksum/Vsum rows [bh, nC, d] -> sum_k/sum_v rows [bh, cap, d]
template <typename T, int D>
__global__ void __launch_bounds__(256) cache_load_kernel(eva_cache c, const T* __restrict__ K,
                                                         const T* __restrict__ V,
                                                         const T* __restrict__ Ksum,
                                                         const T* __restrict__ Vsum, int n, int nC) {
  pdl_wait();
  pdl_trigger();
  constexpr int PPR = D * (int)sizeof(T) / 16;
  const int W = c.cfg.window;
  const int keep = min(n, W);
  const int64_t n_ring = (int64_t)c.cfg.bh_count * keep * PPR;
  const int64_t n_sum = (int64_t)c.cfg.bh_count * nC * PPR;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_ring) {
    const int u = (int)(i / ((int64_t)keep * PPR));
    const int rem = (int)(i % ((int64_t)keep * PPR));
    const int r = n - keep + rem / PPR, p = rem % PPR;
    const size_t slot = (size_t)((c.pos + r) % W);
    const size_t src = ((size_t)u * n + r) * D * sizeof(T) / 16 + p;
    const size_t dst = ((size_t)u * W + slot) * D * sizeof(T) / 16 + p;
    reinterpret_cast<uint4*>(c.ring_k)[dst] = reinterpret_cast<const uint4*>(K)[src];
    reinterpret_cast<uint4*>(c.ring_v)[dst] = reinterpret_cast<const uint4*>(V)[src];
  } else if (i < n_ring + n_sum) {
    const int64_t k = i - n_ring;
    const int u = (int)(k / ((int64_t)nC * PPR));
    const int rem = (int)(k % ((int64_t)nC * PPR));
    const int row = rem / PPR, p = rem % PPR;
    const size_t src = ((size_t)u * nC + row) * D * sizeof(T) / 16 + p;
    const size_t dst = ((size_t)u * c.cap_chunks + row) * D * sizeof(T) / 16 + p;
    reinterpret_cast<uint4*>(c.sum_k)[dst] = reinterpret_cast<const uint4*>(Ksum)[src];
    reinterpret_cast<uint4*>(c.sum_v)[dst] = reinterpret_cast<const uint4*>(Vsum)[src];
  }
}

// ============================================================================ debug kernels
__global__ void mask_ranges_kernel(int C, int W, int mode, int64_t n0, int64_t count, int64_t* lo,
                                   int64_t* nsum) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const Range r = mask_range(n0 + i, C, W, mode);
  lo[i] = r.lo;
  nsum[i] = r.nsum;
}

__global__ void philox_kernel(const uint32_t* in, uint32_t* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* a = in + (size_t)i * 6;
  U4 r = philox4x32_10(U4{a[0], a[1], a[2], a[3]}, a[4], a[5]);
  out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
}

__global__ void draw_eps_kernel(eva_config cfg, int nC, float* eps) {
  // one thread per (unit, chunk, block of 4 channels)
  const int nb = (cfg.d_head + 3) / 4;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)cfg.bh_count * nC * nb) return;
  const int b4 = (int)(i % nb);
  const int c = (int)((i / nb) % nC);
  const int u = (int)(i / ((int64_t)nb * nC));
  const float4 z = philox_normal4(cfg.seed, cfg.layer, (uint32_t)(cfg.bh_begin + u), c, b4);
  const float zz[4] = {z.x, z.y, z.z, z.w};
  float* e = eps + ((size_t)u * nC + c) * cfg.d_head;
  for (int j = 0; j < 4 && 4 * b4 + j < cfg.d_head; ++j) e[4 * b4 + j] = zz[j];
}

// ============================================================================ launchers
#define EVA_DISPATCH_D(D_, ...)                               \
  switch (D_) {                                               \
    case 16: { constexpr int D = 16; __VA_ARGS__; } break;    \
    case 32: { constexpr int D = 32; __VA_ARGS__; } break;    \
    case 64: { constexpr int D = 64; __VA_ARGS__; } break;    \
    case 128: { constexpr int D = 128; __VA_ARGS__; } break;  \
    default: return cudaErrorInvalidValue;                    \
  }
#define EVA_DISPATCH_T(dt, ...)                                                 \
  if ((dt) == EVA_BF16) { using T = __nv_bfloat16; __VA_ARGS__; }               \
  else { using T = float; __VA_ARGS__; }

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

constexpr size_t kSummSmemMax = 96 * 1024;

// Raise the dynamic shared-memory limit of `fn` to `bytes` (once per device, function and
// size: the attribute belongs to the current device's context).
cudaError_t set_smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t ge = cudaGetDevice(&dev);
  if (ge != cudaSuccess) return ge;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{dev, fn}];
  if (bytes > cur) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    cur = bytes;
  }
  return cudaSuccess;
}

cudaError_t launch_summarize(const eva_config& cfg, const void* K, const void* V, const float* eps,
                             void* Ksum, void* Vsum, cudaStream_t s, int c0, const float* Pk) {
  const int nC = cfg.T / cfg.chunk;
  if (nC == 0 || cfg.bh_count == 0) return cudaSuccess;
  // bf16, d in {64, 128}, C in {16..128}: the persistent bulk-copy summariser (summarize_bulk.cu);
  // EVA_SUMMARIZE_REG=1 keeps the register summariser (comparisons)
  static const bool force_reg = [] {
    const char* e = getenv("EVA_SUMMARIZE_REG");
    return e && atoi(e) == 1;
  }();
  if (Pk == nullptr && !force_reg && summarize_bulk_supported(cfg))
    return launch_summarize_bulk(cfg, K, V, eps, Ksum, Vsum, c0, s);
  cudaError_t err = cudaSuccess;
  EVA_DISPATCH_T(cfg.dtype, EVA_DISPATCH_D(cfg.d_head, {
    const size_t sm = summ_smem_bytes(cfg.chunk, D, sizeof(T));
    const int ni = summ_reg_ni<T, D>(cfg.chunk);  // row slots per lane
    if (ni <= 16) {
      const dim3 grid(nC, cfg.bh_count);
      if (ni <= 2)
        err = launch_pdl(summarize_reg_kernel<T, D, 2>, grid, dim3(128), 0, s, cfg, (const T*)K, (const T*)V, eps, (T*)Ksum, (T*)Vsum, c0, Pk);
      else if (ni <= 4)
        err = launch_pdl(summarize_reg_kernel<T, D, 4>, grid, dim3(128), 0, s, cfg, (const T*)K, (const T*)V, eps, (T*)Ksum, (T*)Vsum, c0, Pk);
      else if (ni <= 8)
        err = launch_pdl(summarize_reg_kernel<T, D, 8>, grid, dim3(128), 0, s, cfg, (const T*)K, (const T*)V, eps, (T*)Ksum, (T*)Vsum, c0, Pk);
      else
        err = launch_pdl(summarize_reg_kernel<T, D, 16>, grid, dim3(128), 0, s, cfg, (const T*)K, (const T*)V, eps, (T*)Ksum, (T*)Vsum, c0, Pk);
      if (err != cudaSuccess) return err;
    } else if (Pk != nullptr) {
      return cudaErrorNotSupported;  // the projection lives in the register summariser only
    } else if (sm <= kSummSmemMax) {
      err = set_smem_attr((const void*)summarize_cta_kernel<T, D>, sm);
      if (err != cudaSuccess) return err;
      summarize_cta_kernel<T, D><<<dim3(nC, cfg.bh_count), SUMM_THREADS, sm, s>>>(
          cfg, (const T*)K, (const T*)V, eps, (T*)Ksum, (T*)Vsum, c0);
    } else {
      summarize_kernel<T, D><<<dim3((nC + 3) / 4, cfg.bh_count), 128, 0, s>>>(
          cfg, (const T*)K, (const T*)V, eps, (T*)Ksum, (T*)Vsum, c0);
    }
  }));
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_rope_summarize(const eva_config& cfg, const eva_rope_params& rp, const void* Q, const void* K,
                                  const void* V, const float* eps, void* Qr, void* Kr, void* Ksum, void* Vsum,
                                  cudaStream_t s) {
  const int nC = cfg.T / cfg.chunk;
  const int n_cta = nC + (cfg.T % cfg.chunk ? 1 : 0);
  if (n_cta == 0 || cfg.bh_count == 0) return cudaSuccess;
  const RopeSpec rs = make_rope_spec((double)rp.base, rp.rotary_dim ? rp.rotary_dim : cfg.d_head, rp.style, 1.f);
  cudaError_t err = cudaSuccess;
  EVA_DISPATCH_T(cfg.dtype, EVA_DISPATCH_D(cfg.d_head, {
    const int ni = summ_reg_ni<T, D>(cfg.chunk);
    if (ni > 16) return cudaErrorNotSupported;
    auto k = ni <= 2 ? rope_summarize_kernel<T, D, 2>
                     : ni <= 4 ? rope_summarize_kernel<T, D, 4>
                               : ni <= 8 ? rope_summarize_kernel<T, D, 8> : rope_summarize_kernel<T, D, 16>;
    err = launch_pdl(k, dim3(n_cta, cfg.bh_count), dim3(128), 0, s, cfg, rs, (const T*)Q, (const T*)K,
                     (const T*)V, eps, (T*)Qr, (T*)Kr, (T*)Ksum, (T*)Vsum);
    if (err != cudaSuccess) return err;
  }));
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_rope(const eva_config& cfg, const eva_rope_params& rp, const void* X, void* Y, int64_t pos0,
                        const int64_t* pos, bool inverse, cudaStream_t s) {
  const int64_t rows = (int64_t)cfg.bh_count * cfg.T;
  if (rows == 0) return cudaSuccess;
  const int rd = rp.rotary_dim ? rp.rotary_dim : cfg.d_head;
  const RopeSpec rs = make_rope_spec((double)rp.base, rd, rp.style, inverse ? -1.f : 1.f);
  cudaError_t err = cudaSuccess;
  EVA_DISPATCH_T(cfg.dtype, EVA_DISPATCH_D(cfg.d_head, {
    constexpr int VEC = 16 / (int)sizeof(T);
    const int per = (rs.style == EVA_ROPE_NEOX ? rd / (2 * VEC) : rd / VEC) + (D - rd) / VEC;
    const int64_t n = (rows + ROPE_RB - 1) / ROPE_RB * per;
    err = launch_pdl(rope_walk_kernel<T, D>, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, (const T*)X,
                     (T*)Y, rows, cfg.T, pos0, pos, rs);
    if (err != cudaSuccess) return err;
  }));
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_summarize_bcast(const eva_config& cfg, int c0, const void* K, const void* V,
                                   const float* eps, const unsigned long long* dst_k,
                                   const unsigned long long* dst_v, int n_dst, int dst_rows, cudaStream_t s) {
  const int nC = cfg.T / cfg.chunk;
  if (nC == 0 || cfg.bh_count == 0 || n_dst == 0) return cudaSuccess;
  cudaError_t err = cudaErrorNotSupported;
  EVA_DISPATCH_T(cfg.dtype, EVA_DISPATCH_D(cfg.d_head, {
    const int ni = summ_reg_ni<T, D>(cfg.chunk);
    if (ni <= 16) {
      const dim3 grid(nC, cfg.bh_count);
      if (ni <= 2)
        err = launch_pdl(summarize_bcast_kernel<T, D, 2>, grid, dim3(128), 0, s, cfg, (const T*)K, (const T*)V, eps,
                         dst_k, dst_v, n_dst, dst_rows, c0);
      else if (ni <= 4)
        err = launch_pdl(summarize_bcast_kernel<T, D, 4>, grid, dim3(128), 0, s, cfg, (const T*)K, (const T*)V, eps,
                         dst_k, dst_v, n_dst, dst_rows, c0);
      else if (ni <= 8)
        err = launch_pdl(summarize_bcast_kernel<T, D, 8>, grid, dim3(128), 0, s, cfg, (const T*)K, (const T*)V, eps,
                         dst_k, dst_v, n_dst, dst_rows, c0);
      else
        err = launch_pdl(summarize_bcast_kernel<T, D, 16>, grid, dim3(128), 0, s, cfg, (const T*)K, (const T*)V, eps,
                         dst_k, dst_v, n_dst, dst_rows, c0);
      if (err == cudaSuccess) note_launch();
    }
  }));
  if (err != cudaSuccess) return err;
  return cudaGetLastError();
}

cudaError_t launch_prefill_simt(const eva_config& cfg, const PrefillRange& rg, const void* Q,
                                const void* K, const void* V, const void* Ksum, const void* Vsum,
                                void* O, float* lse, cudaStream_t s) {
  if (cfg.bh_count == 0 || rg.nq == 0) return cudaSuccess;
  EVA_DISPATCH_T(cfg.dtype, EVA_DISPATCH_D(cfg.d_head, {
    constexpr int G = D >= 32 ? D / 32 : 1;
    constexpr int QT = 128 / G;
    dim3 grid((rg.nq + QT - 1) / QT, cfg.bh_count);
    prefill_simt_kernel<T, D><<<grid, 128, 0, s>>>(cfg, rg, (const T*)Q, (const T*)K, (const T*)V,
                                                   (const T*)Ksum, (const T*)Vsum, (T*)O, lse);
  }));
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_cache_append(const eva_cache& c, const void* Kn, const void* Vn, int n_new,
                                const float* eps, cudaStream_t s) {
  const int C = c.cfg.chunk, W = c.cfg.window;
  if (c.cfg.bh_count == 0) return cudaSuccess;
  const int64_t chunk0 = c.pos / C;                      // first chunk not yet summarised
  const int64_t chunk_end = (c.pos + n_new) / C;         // chunks complete after the append
  const int n_chunks = (int)std::max<int64_t>(0, chunk_end - chunk0);
  // Writing the ring can overwrite old positions still needed by a straddling
  // chunk only if n_new > W - C + 1; then summaries go first.
  const bool hazard = n_new > W - C + 1 && n_chunks > 0;
  cudaError_t err = cudaSuccess;
  EVA_DISPATCH_T(c.cfg.dtype, EVA_DISPATCH_D(c.cfg.d_head, {
    const size_t sm = summ_smem_bytes(C, D, sizeof(T));
    const int ni = summ_reg_ni<T, D>(C);
    const bool cta = ni <= 16 || sm <= kSummSmemMax;
    auto fn = ni <= 2 ? append_kernel<T, D, 2> : ni <= 4 ? append_kernel<T, D, 4> : ni <= 8 ? append_kernel<T, D, 8>
            : ni <= 16 ? append_kernel<T, D, 16>
            : sm <= kSummSmemMax ? append_kernel<T, D, 1> : append_kernel<T, D, 0>;
    const size_t smem = (ni > 16 && sm <= kSummSmemMax) ? sm : 0;
    if (smem) {
      err = set_smem_attr((const void*)append_kernel<T, D, 1>, sm);
      if (err != cudaSuccess) return err;
    }
    constexpr int VEC = 16 / sizeof(T);
    const int64_t pieces = (int64_t)std::min(n_new, W) * (D / VEC) * c.cfg.bh_count;
    const int n_copy = (int)((pieces + 127) / 128);
    const int n_sum = n_chunks == 0 ? 0 : c.cfg.bh_count * (cta ? n_chunks : (n_chunks + 3) / 4);
    const T* kn = (const T*)Kn;
    const T* vn = (const T*)Vn;
    if (!hazard) {
      fn<<<n_copy + n_sum, 128, smem, s>>>(c, kn, vn, eps, n_new, n_copy, 1, chunk0, n_chunks);
      note_launch();
    } else {  // summaries first, then the ring write
      fn<<<n_sum, 128, smem, s>>>(c, kn, vn, eps, n_new, 0, 1, chunk0, n_chunks);
      fn<<<n_copy, 128, smem, s>>>(c, kn, vn, eps, n_new, n_copy, 0, chunk0, 0);
      note_launch(2);
    }
    err = cudaGetLastError();
  }));
  return err;
}

int decode_splits(const eva_cache& c) {
  const int64_t n = c.pos - 1;
  const Range r = mask_range(n, c.cfg.chunk, c.cfg.window, c.cfg.mode);
  const int64_t E = r.nsum + (n - r.lo + 1);
  const int64_t target = (int64_t)num_sms() * 8;  // CTAs for ~full occupancy
  int64_t S = (target + c.cfg.bh_count - 1) / std::max(1, c.cfg.bh_count);
  S = std::min<int64_t>(S, std::max<int64_t>(1, E / 64));
  S = std::max<int64_t>(1, std::min<int64_t>(S, 64));
  return (int)S;
}

cudaError_t launch_decode(const eva_cache& c, const void* Q, void* O, float* lse, float* ws,
                          int splits, cudaStream_t s) {
  if (c.cfg.bh_count == 0) return cudaSuccess;
  EVA_DISPATCH_T(c.cfg.dtype, EVA_DISPATCH_D(c.cfg.d_head, {
    dim3 grid(c.cfg.bh_count, splits);
    cudaError_t e = launch_pdl(decode_kernel<T, D, false>, grid, dim3(128), 0, s, c, (const T*)Q, (T*)O, lse, ws,
                               splits, (const T*)nullptr, (const T*)nullptr, (int64_t*)nullptr, (const float*)nullptr, RopeSpec{});
    if (e != cudaSuccess) return e;
    note_launch();
  }));
  return cudaGetLastError();
}

cudaError_t launch_cache_load(const eva_cache& c, const void* K, const void* V, const void* Ksum,
                              const void* Vsum, int n, cudaStream_t s, bool copy_summaries) {
  if (c.cfg.bh_count == 0) return cudaSuccess;
  const int nC = copy_summaries ? n / c.cfg.chunk : 0;
  EVA_DISPATCH_T(c.cfg.dtype, EVA_DISPATCH_D(c.cfg.d_head, {
    constexpr int PPR = D * (int)sizeof(T) / 16;
    const int64_t pieces = (int64_t)c.cfg.bh_count * (std::min(n, c.cfg.window) + nC) * PPR;
    cudaError_t e = launch_pdl(cache_load_kernel<T, D>, dim3((unsigned)((pieces + 255) / 256)), dim3(256), 0, s,
                               c, (const T*)K, (const T*)V, (const T*)Ksum, (const T*)Vsum, n, nC);
    if (e != cudaSuccess) return e;
    note_launch();
  }));
  return cudaGetLastError();
}

cudaError_t launch_decode_step(const eva_cache& c_after, const void* Q, const void* Kn, const void* Vn,
                               void* O, float* lse, float* ws, int splits, cudaStream_t s) {
  if (c_after.cfg.bh_count == 0) return cudaSuccess;
  EVA_DISPATCH_T(c_after.cfg.dtype, EVA_DISPATCH_D(c_after.cfg.d_head, {
    dim3 grid(c_after.cfg.bh_count, splits);
    cudaError_t e = launch_pdl(decode_kernel<T, D, true>, grid, dim3(128), 0, s, c_after, (const T*)Q, (T*)O, lse,
                               ws, splits, (const T*)Kn, (const T*)Vn, (int64_t*)nullptr, (const float*)nullptr, RopeSpec{});
    if (e != cudaSuccess) return e;
    note_launch();
  }));
  return cudaGetLastError();
}

bool ragged_supported(const eva_config& cfg) {
  bool ok = false;
  auto probe = [&]() -> cudaError_t {
    EVA_DISPATCH_T(cfg.dtype, EVA_DISPATCH_D(cfg.d_head, { ok = summ_reg_ni<T, D>(cfg.chunk) <= 16; }));
    return cudaSuccess;
  };
  return probe() == cudaSuccess && ok;
}

cudaError_t launch_decode_step_ragged(const eva_cache& c, int64_t* pos, const void* Q, const void* Kn,
                                      const void* Vn, const float* eps, void* O, float* lse, float* ws,
                                      int splits, cudaStream_t s) {
  if (c.cfg.bh_count == 0) return cudaSuccess;
  EVA_DISPATCH_T(c.cfg.dtype, EVA_DISPATCH_D(c.cfg.d_head, {
    const int ni = summ_reg_ni<T, D>(c.cfg.chunk);
    auto ak = ni <= 2 ? ragged_append_kernel<T, D, 2>
                      : ni <= 4 ? ragged_append_kernel<T, D, 4>
                                : ni <= 8 ? ragged_append_kernel<T, D, 8> : ragged_append_kernel<T, D, 16>;
    cudaError_t e = launch_pdl(ak, dim3(c.cfg.bh_count), dim3(128), 0, s, c, pos, (const T*)Kn, (const T*)Vn, eps);
    if (e != cudaSuccess) return e;
    e = launch_pdl(decode_kernel<T, D, false, true>, dim3(c.cfg.bh_count, splits), dim3(128), 0, s, c, (const T*)Q,
                   (T*)O, lse, ws, splits, (const T*)nullptr, (const T*)nullptr, pos, (const float*)nullptr, RopeSpec{});
    if (e != cudaSuccess) return e;
    note_launch(2);
  }));
  return cudaGetLastError();
}

cudaError_t launch_decode_step_ragged_fused(const eva_cache& c, int64_t* pos, const void* Q, const void* Kn,
                                            const void* Vn, const float* eps, void* O, float* lse, float* ws,
                                            int splits, cudaStream_t s, const eva_rope_params* rp) {
  if (c.cfg.bh_count == 0) return cudaSuccess;
  EVA_DISPATCH_T(c.cfg.dtype, EVA_DISPATCH_D(c.cfg.d_head, {
    cudaError_t e;
    if (rp) {
      const RopeSpec rs = make_rope_spec((double)rp->base, rp->rotary_dim ? rp->rotary_dim : c.cfg.d_head,
                                         rp->style, 1.f);
      e = launch_pdl(decode_kernel<T, D, true, true, true>, dim3(c.cfg.bh_count, splits), dim3(128), 0, s, c,
                     (const T*)Q, (T*)O, lse, ws, splits, (const T*)Kn, (const T*)Vn, pos, eps, rs);
    } else {
      e = launch_pdl(decode_kernel<T, D, true, true>, dim3(c.cfg.bh_count, splits), dim3(128), 0, s, c,
                     (const T*)Q, (T*)O, lse, ws, splits, (const T*)Kn, (const T*)Vn, pos, eps, RopeSpec{});
    }
    if (e != cudaSuccess) return e;
    note_launch();
  }));
  return cudaGetLastError();
}

cudaError_t launch_mask_ranges(const eva_config& cfg, int64_t n0, int64_t count, int64_t* lo,
                               int64_t* nsum, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  mask_ranges_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(cfg.chunk, cfg.window, cfg.mode,
                                                                    n0, count, lo, nsum);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_philox(const uint32_t* in, uint32_t* out, int n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  philox_kernel<<<(n + 255) / 256, 256, 0, s>>>(in, out, n);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_draw_eps(const eva_config& cfg, float* eps, cudaStream_t s) {
  const int nC = cfg.T / cfg.chunk;
  const int64_t total = (int64_t)cfg.bh_count * nC * ((cfg.d_head + 3) / 4);
  if (total == 0) return cudaSuccess;
  draw_eps_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(cfg, nC, eps);
  note_launch();
  return cudaGetLastError();
}

}  // namespace eva
