// prefill_sm100.cu -- bf16 FlashEVA chunk-causal prefill on the sm_100a tensor cores.
//
// Computes, for every query n of a 128-query tile (Eq.12-14, mask P:124):
//   o_n = softmax over { s q_n.k~_c : c < nsum(n) }  U  { s q_n.k_m : lo(n) <= m <= n }
// with the summary prefix and the local span walked as 64-key tiles.
//
// CTA = one (unit, 128-query tile); 6 warps, warp-specialised:
//   warp 0      TMA producer: Q tile once, then K/V (or Ksum/Vsum) 64-row tiles into an
//               NSTAGE-deep shared-memory ring (SWIZZLE_128B, mbarrier complete_tx)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_j  = Q K_j^T      (SS, M=128 N=64 K=d)  -> TMEM S buffer j%2
//                 O   += P_j V_j      (TS, M=128 N=d K=64)   P_j read from TMEM
//               issue order S_0, S_1, PV_0, S_2, PV_1, ... so S_{j+1} overlaps softmax j
//   warps 2..5  softmax: thread <-> TMEM lane <-> query row.  tcgen05.ld S, apply the
//               per-row chunk-causal mask, online max (lazy rescale: O in TMEM is only
//               corrected when the running max grows by > 2^8), P = exp2(...) packed to
//               bf16 and tcgen05.st back into the S buffer, arrive p_full.
//               Epilogue: O / l -> bf16 -> swizzled smem -> TMA store; LSE.
// TMEM (256 columns): [0,64) S/P buffer 0, [64,128) S/P buffer 1, [128,128+d) O.
// Two CTAs fit on one SM (smem <= ~97 KB, 256 TMEM columns each).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "launch.h"
#include "prefill_common.cuh"
#include "sm100.cuh"

namespace eva {
namespace {

using namespace sm100;
using namespace pfx;
constexpr int BM = 128;       // queries per tile
constexpr int BN = 64;        // keys per KV tile
constexpr int NTHREADS = 192;
// EVA_SUMMARIES_FUSED: two more warps (6, 7) compute the chunk summaries in-kernel
constexpr int NTHREADS_F = 256;
constexpr int SUMM_THREADS_F = 64;
// in-kernel RoPE: ROPE_WARPS warps (6 ..) rotate the local K tiles
constexpr int ROPE_WARPS = 4;
constexpr int NTHREADS_R = NTHREADS + 32 * ROPE_WARPS;
constexpr uint32_t TMEM_COLS = 256;
constexpr uint32_t TM_O = 128;

// Exchange buffers of the fused summaries (fused_summaries below).
template <int D>
struct alignas(16) SummScratch {
  float eps[8][D];   // draws of the owned chunks (at most 128 / 16)
  float red[2][4][D];// per-warp partial column sums / weighted value sums, per chunk of the tile
  float om[4][D];    // omega per chunk of the tile
  float p[64];       // softmax weight of each tile row
  float l[4];        // softmax denominator per chunk
  float st[2][2];    // C = 64: per-warp max / sum
};

// NSTAGE < 10: NSTAGE K and NSTAGE V slots.  NSTAGE = 10*NSK + NSV: separate ring depths
// (a deeper K ring lets the next K tiles stream in earlier; K is consumed one softmax period
// before V).  Deep-ring layouts are sized to fill the SM with two CTAs, so they are used
// without the 1 KB alignment pad (the dynamic window is 1 KB aligned; checked in-kernel).
struct NoSumm {};
template <int D, int NSTAGE, bool FS = false>
struct __align__(1024) Smem {
  static constexpr int NSK = NSTAGE >= 10 ? NSTAGE / 10 : NSTAGE;
  static constexpr int NSV = NSTAGE >= 10 ? NSTAGE % 10 : NSTAGE;
  static constexpr size_t PAD = NSTAGE >= 10 ? 0 : 1024;
  __nv_bfloat16 q[BM * D];               // D/64 sub-tiles [128][64], 16 KB each
  __nv_bfloat16 k[NSK][BN * D];          // D/64 sub-tiles [64][64], 8 KB each
  __nv_bfloat16 v[NSV][BN * D];
  uint64_t q_full;
  // K and V slots are released separately: a K slot as soon as its S MMA completed, a V
  // slot after its PV MMA, so the next K tiles stream in one softmax period earlier.
  uint64_t k_full[NSK], v_full[NSV], k_empty[NSK], v_empty[NSV];
  uint64_t s_full[2], p_full[2], o_done, o_final;
  uint64_t q_rot, k_rot[NSK];  // RoPE in-kernel: Q rotated (warps 2-7), K tile rotated (warps 6, 7)
  uint32_t tmem_base;
  std::conditional_t<FS, SummScratch<D>, NoSumm> summ;  // fused summaries' exchange buffers (FS only)
  int ticket;           // fused: the CTA's query tile ticket and the launch epoch
  uint32_t epoch;
};

// Arguments of the in-kernel summaries (EVA_SUMMARIES_FUSED).  ws: [ticket, done, epoch, pad,
// flags[units * n_qt]] (fused_workspace); Ksum/Vsum are written with generic stores and read
// back by other CTAs through TMA once the owning tile's flag holds epoch + 1.
struct FusedArgs {
  eva_config cfg;
  const __nv_bfloat16* K;  // [units, T, D]: the summaries read their rows from global memory
  const __nv_bfloat16* V;
  int64_t T;
  __nv_bfloat16* ks;
  __nv_bfloat16* vs;
  const float* eps;
  uint32_t* ws;
  int nC, n_qt, units, total, order;
};

// RoPE applied inside the kernel (eva_attn_prefill_rope; reading R18/R19): Q and K come
// in un-rotated, the Q tile and every LOCAL K tile are rotated in shared memory after TMA lands
// them and before the MMA reads them, so RoPE(Q), RoPE(K) are never written to HBM.  The summary
// tiles are summaries of the rotated keys already (eva_rope_summarize_ex, summaries-only).
struct RopeArgs {
  double th[64];  // theta_j = base^(-2j/rd), j < rd/2, in double (computed on the host)
  int rd;         // rotary channels (a power of two, 16..D)
  int pad;
};

// RoPE of a landed tile by nthr threads.  A row's rotated channels form NI items --
// interleaved (STYLE 1): the 16-byte piece `item` (pairs j = 4 item + i, channels 2j, 2j+1);
// half-split (STYLE 2): pieces item and item + rd/16 (pairs j = 8 item + i, channels j, j + rd/2).
// NI divides nthr: thread t takes item t % NI of rows t / NI + k * rstep (rstep = nthr / NI) and
// walks them with a rotation recurrence -- the first row's angle comes from double precision
// (pos * theta_j mod 2 pi), each next row multiplies by e^{i rstep theta_j}.  Arithmetic on
// packed fp32x2 (two pairs per FFMA2); two rows per iteration for load/store overlap.
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t neg2(uint64_t a) { return a ^ 0x8000000080000000ull; }
__device__ __forceinline__ void rope_angle(double a, float& c, float& s) {
  a -= 6.283185307179586 * rint(a * 0.15915494309189535);
  __sincosf((float)a, &s, &c);
}
// bf16x2 word -> (low, high) channel as packed fp32x2 pieces of two words
__device__ __forceinline__ uint64_t lo2(uint32_t w0, uint32_t w1) {
  return (uint64_t)(w0 << 16) | ((uint64_t)(w1 << 16) << 32);
}
__device__ __forceinline__ uint64_t hi2(uint32_t w0, uint32_t w1) {
  return (uint64_t)(w0 & 0xffff0000u) | ((uint64_t)(w1 & 0xffff0000u) << 32);
}

template <int STYLE>
struct RopeWalker {
  static constexpr int NP = STYLE == 2 ? 8 : 4;  // pairs per item
  static constexpr int NQ = NP / 2;               // packed pair groups
  uint64_t c[NQ], s[NQ], sc[NQ], ss[NQ];          // angle of the next row; one row-step rotation
  const double* th;
  int item, g, rstep, off_b;
  int64_t at = -1;                                // position whose angle c / s hold (-1: none)
  __device__ __forceinline__ void init(const RopeArgs& ra, int t, int nthr) {
    const int NI = STYLE == 2 ? ra.rd / 16 : ra.rd / 8;
    item = t % NI;
    g = t / NI;
    rstep = nthr / NI;
    off_b = ra.rd / 2;
    th = ra.th + NP * item;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float a0, b0, a1, b1;
      rope_angle((double)rstep * th[2 * q], a0, b0);
      rope_angle((double)rstep * th[2 * q + 1], a1, b1);
      sc[q] = f2pack(a0, a1);
      ss[q] = f2pack(b0, b1);
    }
  }
  // Rotate rows g, g + rstep, ... < nrows of a swizzled tile (D/64 sub-tiles of nrows x 128 B)
  // holding positions pos0 + r.  A tile that continues the previous one (pos0 + g == at: the
  // local K tiles are consecutive) keeps the recurrence going; otherwise the first angle is
  // computed in double.
  __device__ __forceinline__ void run(uint8_t* base, int nrows, int64_t pos0) {
    if (g >= rstep) return;
    if (pos0 + g != at) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        float c0, s0, c1, s1;
        rope_angle((double)(pos0 + g) * th[2 * q], c0, s0);
        rope_angle((double)(pos0 + g) * th[2 * q + 1], c1, s1);
        c[q] = f2pack(c0, c1);
        s[q] = f2pack(s0, s1);
      }
    }
    const int ch_a = 8 * item, ch_b = ch_a + off_b;
    const uint32_t off_a = (uint32_t)(ch_a >> 6) * (uint32_t)nrows * 128u, c16_a = (uint32_t)((ch_a & 63) >> 3);
    const uint32_t offb = (uint32_t)(ch_b >> 6) * (uint32_t)nrows * 128u, c16_b = (uint32_t)((ch_b & 63) >> 3);
    int r = g;
#pragma unroll 2
    for (; r < nrows; r += rstep) {
      uint4* pa = reinterpret_cast<uint4*>(base + off_a + (uint32_t)r * 128u + ((c16_a ^ (uint32_t)(r & 7)) << 4));
      if constexpr (STYLE == 2) {
        uint4* pb = reinterpret_cast<uint4*>(base + offb + (uint32_t)r * 128u + ((c16_b ^ (uint32_t)(r & 7)) << 4));
        const uint4 xa = *pa, xb = *pb;
        const uint32_t wa[4] = {xa.x, xa.y, xa.z, xa.w}, wb[4] = {xb.x, xb.y, xb.z, xb.w};
        uint32_t oa[4], ob[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // pairs 2q, 2q+1: x0 from piece a, x1 from piece b
          const uint64_t x0 = lo2(wa[q], 0) | ((uint64_t)(wa[q] & 0xffff0000u) << 32);
          const uint64_t x1 = lo2(wb[q], 0) | ((uint64_t)(wb[q] & 0xffff0000u) << 32);
          const uint64_t y0 = ffma2(x1, neg2(s[q]), fmul2(x0, c[q]));
          const uint64_t y1 = ffma2(x1, c[q], fmul2(x0, s[q]));
          oa[q] = pack_bf16(f2lo(y0), f2hi(y0));
          ob[q] = pack_bf16(f2lo(y1), f2hi(y1));
        }
        *pa = make_uint4(oa[0], oa[1], oa[2], oa[3]);
        *pb = make_uint4(ob[0], ob[1], ob[2], ob[3]);
      } else {
        const uint4 xa = *pa;
        // pairs (0, 1) in words x, y; pairs (2, 3) in words z, w: even channels in the low halves
        const uint64_t e01 = lo2(xa.x, xa.y), o01 = hi2(xa.x, xa.y);
        const uint64_t e23 = lo2(xa.z, xa.w), o23 = hi2(xa.z, xa.w);
        const uint64_t ye01 = ffma2(o01, neg2(s[0]), fmul2(e01, c[0])), yo01 = ffma2(o01, c[0], fmul2(e01, s[0]));
        const uint64_t ye23 = ffma2(o23, neg2(s[1]), fmul2(e23, c[1])), yo23 = ffma2(o23, c[1], fmul2(e23, s[1]));
        *pa = make_uint4(pack_bf16(f2lo(ye01), f2lo(yo01)), pack_bf16(f2hi(ye01), f2hi(yo01)),
                         pack_bf16(f2lo(ye23), f2lo(yo23)), pack_bf16(f2hi(ye23), f2hi(yo23)));
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {  // next row: multiply by e^{i rstep theta}
        const uint64_t cn = ffma2(s[q], neg2(ss[q]), fmul2(c[q], sc[q]));
        s[q] = ffma2(c[q], ss[q], fmul2(s[q], sc[q]));
        c[q] = cn;
      }
    }
    at = pos0 + r;
  }
};

// Columns outside [vlo, vhi) or inside [xlo, xhi) of a 64-column S tile set to -inf.  A 64-bit
// valid mask is built once; each column then costs a shift pair (sign-extend its bit) and one
// LOP3 select -- the per-column range compares cost ~6 instructions per column (ncu: the masked
// tiles ran 383 extra instructions per warp, ~46 % of the tiles at configs[2]).
__device__ __forceinline__ void mask_columns(uint32_t (&sr)[64], int vlo, int vhi, int xlo, int xhi) {
  const uint64_t m = range_bits(vlo, vhi) & ~range_bits(xlo, xhi);
  const uint32_t mw[2] = {(uint32_t)m, (uint32_t)(m >> 32)};
#pragma unroll
  for (int c = 0; c < 64; ++c) {
    const uint32_t keep = (uint32_t)((int32_t)(mw[c >> 5] << (31 - (c & 31))) >> 31);  // all ones if valid
    sr[c] = (sr[c] & keep) | (0xff800000u & ~keep);
  }
}

// One softmax step of a 64-key tile for this thread's query row (thread <-> TMEM lane).
// S (fp32, raw q.k) is read from TMEM, columns outside [vlo, vhi) are masked, the running
// max m_ref (log2 units) is raised lazily (O and l are only rescaled when the tile max
// exceeds m_ref by more than 8, i.e. p <= 2^8), and P = exp2(s*scale_log2 - m_ref) is
// written back to the same TMEM columns as packed bf16 (the A operand of the PV MMA).
// wait_o() must make the previous PV of this Q tile complete before O is rescaled.
// Requires scale_log2 > 0 (validated by the C ABI), so max and scaling commute.
// Columns [xlo, xhi) are masked too (the non-causal mode's own-block summaries, R15), and
// bias2 (log2 units) is added to every logit of the tile (summary_bias on summary tiles, R16).
template <int D, typename WaitO>
__device__ __forceinline__ void softmax_tile_mx(uint32_t s_addr, uint32_t o_addr, int vlo, int vhi,
                                                int xlo, int xhi, float bias2, float scale_log2,
                                                float& m_ref, float& l, const WaitO& wait_o) {
  uint32_t sr[64];
  tmem_ld32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
  tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
  tmem_wait_ld();
  const bool full = vlo <= 0 && vhi >= 64 && (xhi <= 0 || xlo >= 64 || xlo >= xhi);
  if (!__all_sync(0xffffffffu, full)) mask_columns(sr, vlo, vhi, xlo, xhi);
  // tree max (8 independent chains) -- a 63-deep serial chain is latency-bound with only
  // two softmax warps per scheduler
  float pm[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) pm[i] = __uint_as_float(sr[i]);
#pragma unroll
  for (int c = 8; c < 64; ++c) pm[c & 7] = fmaxf(pm[c & 7], __uint_as_float(sr[c]));
  float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
  mx = mx * scale_log2 + bias2;
  const bool grow = mx > m_ref + 8.0f;
  if (__any_sync(0xffffffffu, grow && m_ref != -INFINITY)) {
    const float f = (grow && m_ref != -INFINITY) ? ex2(m_ref - mx) : 1.0f;
    wait_o();
    tc_fence_after();
    // 8 columns at a time: S (64 registers) stays live across the rescale
#pragma unroll 1
    for (int cc = 0; cc < D / 8; ++cc) {
      uint32_t o[8];
      tmem_ld8(o_addr + cc * 8, o);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
      tmem_st8(o_addr + cc * 8, o);
    }
    tmem_wait_st();
    l *= f;
  }
  if (grow) m_ref = mx;
  const float neg = (m_ref == -INFINITY ? 0.f : -m_ref) + bias2;
  float ls[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) ls[i] = 0.f;
  // P packed in place: pair c lands in sr[c] after sr[2c], sr[2c+1] are read (no second array,
  // so S, P and O's rescale fit the fused kernel's 128-register budget without spilling)
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const float p0 = ex2(fmaf(__uint_as_float(sr[2 * c]), scale_log2, neg));
    const float p1 = ex2(fmaf(__uint_as_float(sr[2 * c + 1]), scale_log2, neg));
    ls[(2 * c) & 7] += p0;
    ls[(2 * c + 1) & 7] += p1;
    sr[c] = pack_bf16(p0, p1);
  }
  l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
  tmem_st32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
  tmem_wait_st();
  tc_fence_before();
}

template <int D, typename WaitO>
__device__ __forceinline__ void softmax_tile(uint32_t s_addr, uint32_t o_addr, int vlo, int vhi,
                                             float scale_log2, float& m_ref, float& l,
                                             const WaitO& wait_o) {
  softmax_tile_mx<D>(s_addr, o_addr, vlo, vhi, 0, 0, 0.f, scale_log2, m_ref, l, wait_o);
}

// softmax_tile with packed fp32x2 arithmetic and EMU of every 8 column pairs exponentiated by
// exp2_poly2 instead of MUFU.EX2 (FA4-style split of the exponentials between the MUFU and
// FMA pipes).  Same contract and results up to the exp2 approximation (both are far below
// the bf16 rounding of P).
template <int D, int EMU, typename WaitO>
__device__ __forceinline__ void softmax_tile2(uint32_t s_addr, uint32_t o_addr, int vlo, int vhi,
                                              int xlo, int xhi, float bias2, float scale_log2,
                                              float& m_ref, float& l, const WaitO& wait_o) {
  uint32_t sr[64];
  tmem_ld32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
  tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
  tmem_wait_ld();
  const bool full = vlo <= 0 && vhi >= 64 && (xhi <= 0 || xlo >= 64 || xlo >= xhi);
  if (!__all_sync(0xffffffffu, full)) mask_columns(sr, vlo, vhi, xlo, xhi);
  float pm[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) pm[i] = __uint_as_float(sr[i]);
#pragma unroll
  for (int c = 8; c < 64; ++c) pm[c & 7] = fmaxf(pm[c & 7], __uint_as_float(sr[c]));
  float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
  mx = mx * scale_log2 + bias2;
  const bool grow = mx > m_ref + 8.0f;
  if (__any_sync(0xffffffffu, grow && m_ref != -INFINITY)) {
    const float f = (grow && m_ref != -INFINITY) ? ex2(m_ref - mx) : 1.0f;
    wait_o();
    tc_fence_after();
    const uint64_t f2 = f2pack(f, f);
#pragma unroll 1
    for (int cc = 0; cc < D / 8; ++cc) {
      uint32_t o[8];
      tmem_ld8(o_addr + cc * 8, o);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const uint64_t v = ffma2(f2pack(__uint_as_float(o[i]), __uint_as_float(o[i + 1])), f2, 0ull);
        o[i] = (uint32_t)v;
        o[i + 1] = (uint32_t)(v >> 32);
      }
      tmem_st8(o_addr + cc * 8, o);
    }
    tmem_wait_st();
    l *= f;
  }
  if (grow) m_ref = mx;
  const float neg = (m_ref == -INFINITY ? 0.f : -m_ref) + bias2;
  const uint64_t sc2 = f2pack(scale_log2, scale_log2), ng2 = f2pack(neg, neg);
  uint64_t ls[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const uint64_t x = ffma2(f2pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sc2, ng2);
    uint64_t p;
    if ((c & 7) < EMU) {
      p = exp2_poly2(x);
    } else {
      p = f2pack(ex2(f2lo(x)), ex2(f2hi(x)));
    }
    ls[c & 3] = fadd2(ls[c & 3], p);
    sr[c] = pack_bf16(f2lo(p), f2hi(p));
  }
  const uint64_t s2 = fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3]));
  l += f2lo(s2) + f2hi(s2);
  tmem_st32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
  tmem_wait_st();
  tc_fence_before();
}

// Tile plan of a query-range call (eva_attn_prefill_range): query tile qt covers absolute
// positions [q0 + qt*BM, ...), local key tiles start at lo(n0) (absolute); row() maps a
// tile base to the TMA row of its tensor (key rows are stored from position k0).
struct RangePlan {
  int64_t n0, nlast, lo0, k0;
  int n_st, n_lt;
  __device__ RangePlan(int qt, const PrefillRange& rg, int C, int W, int mode, bool fused = false) {
    const int64_t qend = rg.q0 + rg.nq;
    n0 = rg.q0 + (int64_t)qt * BM;
    nlast = min(n0 + BM - 1, qend - 1);
    const Vis vf = visible_set(n0, C, W, mode, qend), vl = visible_set(nlast, C, W, mode, qend);
    // causal: summary prefix [0, nsum(n_last)); non-causal: every summary (rows mask their
    // own block's chunks)
    n_st = (int)(((mode == EVA_NONCAUSAL ? (int64_t)rg.nsl : vl.s1) + BN - 1) / BN);
    lo0 = vf.lo;
    k0 = rg.k0;
    n_lt = (int)((vl.hi - lo0 + BN - 1) / BN);
    if (fused) {
      order = 2;
      rot = (int)((n0 - lo0) / BN);
      s_end = vl.s1;
    }
  }
  // Tile order: local tiles first, then the summary tiles (order 0) -- the local span
  // depends only on the inputs, so with EVA_PREFILL_OVERLAP it runs while the summarize
  // kernel is still finishing -- or summaries first (order 1).  Order 2 (fused summaries):
  // the local tiles rotated to start at the tile holding n0 (the tiles whose chunks this CTA
  // summarises come first), then the summary tiles aligned to END at nsum(n_last) -- the
  // first may start at a negative chunk (TMA zero-fills it; masked) -- so no row of a summary
  // tile is a chunk that is not complete and published yet.
  int order = 0, rot = 0;
  int64_t s_end = 0;
  __device__ int count() const { return n_st + n_lt; }
  __device__ bool summary(int j) const { return order == 1 ? j < n_st : j >= n_lt; }
  __device__ int local_index(int j) const {  // local tile (0..n_lt-1) walked at step j
    if (order == 1) return j - n_st;
    if (order == 2) return (j + rot) % n_lt;
    return j;
  }
  __device__ int64_t base(int j) const {
    if (summary(j)) {
      if (order == 1) return (int64_t)j * BN;
      if (order == 2) return s_end - (int64_t)(n_st - (j - n_lt)) * BN;
      return (int64_t)(j - n_lt) * BN;
    }
    return lo0 + (int64_t)local_index(j) * BN;
  }
  __device__ int row(int j) const {
    const int64_t b = base(j);
    return summary(j) ? (int)b : (int)(b - k0);
  }
};


// Debug timeline of the tile kernel (eva_debug_trace_prefill with variant 1): CTAs with
// linear id in {0, 1, 150, 151} log (globaltimer-free) clock64 events per role in shared
// memory and flush them to g_trace2 at exit.  Roles: 0 producer, 1 MMA, 2 softmax (warp 2
// lane 0).  kinds: 1 start, 2 Q arrived (MMA), 3 k_full(j) (MMA), 4 S(j) issued, 5 P(j)
// received (MMA), 6 PV(j) issued, 7 softmax got S(j), 8 softmax P(j) done, 9 o_final
// (epilogue start), 10 epilogue done, 11 producer slot free (j), 12 producer issued (j);
// fused: 16 producer starts waiting for the summary flags, 17 flags ready; role 3 (summary
// warps): 13 owned tile j landed, 14 tile j summarised and released, 15 flag published.
__device__ unsigned long long* g_trace2 = nullptr;
__device__ int g_trace_mid = 150;  // slots 2, 3 trace CTAs g_trace_mid, +1 (EVA_TRACE_MID)
constexpr int TT_ROLES = 4, TT_PER_ROLE = 48, TT_SLOTS = 4, TT_MAX_CTAS = 4096;
struct TileTrace {
  unsigned long long ev[TT_ROLES][TT_PER_ROLE];
  int n[TT_ROLES];
  int slot;  // tt_slot() read once at entry (it loads g_trace_mid from global memory)
};
__device__ __forceinline__ int tt_slot() {
  const int id = blockIdx.y * gridDim.x + blockIdx.x;
  return id == 0 ? 0 : id == 1 ? 1 : id == g_trace_mid ? 2 : id == g_trace_mid + 1 ? 3 : -1;
}
template <bool TRACE>
__device__ __forceinline__ void tt(TileTrace* tl, int role, int kind, int j) {
  if constexpr (TRACE) {
    if (tl->slot >= 0) {
      const int i = tl->n[role];
      if (i < TT_PER_ROLE) tl->ev[role][i] = ((unsigned long long)clock64() << 24) | ((unsigned)kind << 16) | (unsigned)(j & 0xffff);
      tl->n[role] = i + 1;
    }
  }
}

// ---- in-kernel chunk summaries (EVA_SUMMARIES_FUSED), run by warps 6 and 7 of the tile kernel.
// The CTA of query tile qt owns the complete chunks inside its own query rows [n0, n_last]
// (C in {16, 32, 64}; each lies inside one 64-key tile of the local span, which starts on a
// chunk boundary).  Per chunk c (formulas of summarize.cuh / eva.h eva_summarize):
//   k~_c    = (1/C) sum_i k_{cC+i}                      P:99 Eq.10 (reading R1)
//   omega_c = lambda * clip(k~_c + eps_c)                P:311-314 Eq.15 (R2, R3)
//   a_i     = omega_c . k_i - |k_i|^2 / 2                log xi
//   beta^_c = sum_i softmax(a)_i v_i                     P:92 Eq.9, S = 1
// The owned rows are read from the K/V tiles the producer lands in shared memory for the
// attention anyway (the walk starts with them, order 2); the summary side releases a slot as
// soon as it is done with it.  The code is kept small and rolled on purpose: it runs a few
// times per CTA next to the softmax loop, and unrolled it would stream from the instruction
// cache (measured: the unrolled form spent most of its time waiting for instructions).
//   0. at start: the random draws of every owned chunk (data-independent) into shared memory;
//   1. column sums: thread t sums the 16-byte piece pc = t % TPR of rows g, g + RPP, ...
//      (g = t / TPR, RPP = 64 / TPR) straight from bf16 (FHADD.BF16), reduced over g by
//      shuffles and across the two warps through shared memory -> k~, omega per chunk;
//   2. logits: thread t takes tile row t against its chunk's omega; max / sum over the chunk
//      by shuffles (C <= 32) or across the warps (C = 64) -> softmax weights in shared memory;
//   3. beta^: thread t accumulates weight x value piece over its rows, reduced like pass 1.
// After the last owned chunk the tile's ready flag is set to epoch + 1 (release, after a proxy
// fence: the readers load the rows by TMA).

// fp32 += bf16 (low / high half of a packed pair): FHADD.BF16, no unpacking
__device__ __forceinline__ float add_bf16lo(float acc, uint32_t w) {
  asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"((unsigned short)(w & 0xffffu)));
  return acc;
}
__device__ __forceinline__ float add_bf16hi(float acc, uint32_t w) {
  asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"((unsigned short)(w >> 16)));
  return acc;
}

template <int D, int CC, bool TRACE, typename SM, typename Plan>
__device__ __noinline__ void fused_summaries(SM* sm, const Plan& plan, const FusedArgs& fa, int u, int qt,
                                             uint32_t epoch, TileTrace* tl) {
  constexpr int NSK = SM::NSK, NSV = SM::NSV;
  constexpr int TPR = D / 8, RPP = SUMM_THREADS_F / TPR;  // pieces per row, rows per pass
  constexpr int NRC = CC / RPP, NCH = BN / CC;            // rows per thread per chunk, chunks per tile
  static_assert(CC % RPP == 0 && NCH <= 4, "chunk size outside the fused envelope");
  SummScratch<D>& sc = sm->summ;
  const int t = threadIdx.x - (NTHREADS_F - SUMM_THREADS_F), w = t >> 5, lane = t & 31;
  const int pc = t % TPR, g = t / TPR;
  const int64_t c_lo = plan.n0 / CC, c_hi = min((int64_t)fa.nC, (plan.nlast + 1) / CC);
  const uint32_t bh = (uint32_t)(fa.cfg.bh_begin + u);
  const uint32_t poff = (uint32_t)((pc >> 3) * (BN * 128)), c16 = (uint32_t)(pc & 7);
  if (t == 0) tt<TRACE>(tl, 3, 13, 0);
  // 0. the draws of the owned chunks: thread t does 4 channels per step
#pragma unroll 1
  for (int i = t; i < (int)(c_hi - c_lo) * (D / 4); i += SUMM_THREADS_F) {
    const int64_t c = c_lo + i / (D / 4);
    const int q = i % (D / 4);
    float4 z;
    if (fa.eps) z = __ldg(reinterpret_cast<const float4*>(fa.eps + ((size_t)u * fa.nC + (size_t)c) * D) + q);
    else z = philox_normal4(fa.cfg.seed, fa.cfg.layer, bh, (uint32_t)c, (uint32_t)q);
    *reinterpret_cast<float4*>(&sc.eps[c - c_lo][4 * q]) = z;
  }
  named_bar_sync(2, SUMM_THREADS_F);
  for (int j = 0; j < plan.n_lt; ++j) {
    const int64_t b = plan.base(j);  // a multiple of CC
    const int64_t ca = max(c_lo, b / CC), cb = min(c_hi, (b + BN) / CC);
    if (ca >= cb) break;  // the owned tiles are a prefix of the walk (order 2)
    const int sk = j % NSK, sv = j % NSV;
    const int64_t c0 = b / CC;
    mbar_wait(&sm->k_full[sk], (j / NSK) & 1);
    const uint8_t* kt = reinterpret_cast<const uint8_t*>(sm->k[sk]);
    // 1. column sums of every chunk of the tile
#pragma unroll 1
    for (int q = 0; q < NCH; ++q) {
      float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
      for (int k = 0; k < NRC; ++k) {
        const int r = q * CC + g + k * RPP;
        const uint4 x = *reinterpret_cast<const uint4*>(kt + poff + r * 128 + ((c16 ^ (uint32_t)(r & 7)) << 4));
        cs[0] = add_bf16lo(cs[0], x.x); cs[1] = add_bf16hi(cs[1], x.x);
        cs[2] = add_bf16lo(cs[2], x.y); cs[3] = add_bf16hi(cs[3], x.y);
        cs[4] = add_bf16lo(cs[4], x.z); cs[5] = add_bf16hi(cs[5], x.z);
        cs[6] = add_bf16lo(cs[6], x.w); cs[7] = add_bf16hi(cs[7], x.w);
      }
#pragma unroll
      for (int o = TPR; o < 32; o <<= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i) cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], o);
      if (lane < TPR) {
        float4* dst = reinterpret_cast<float4*>(&sc.red[w][q][pc * 8]);
        dst[0] = make_float4(cs[0], cs[1], cs[2], cs[3]);
        dst[1] = make_float4(cs[4], cs[5], cs[6], cs[7]);
      }
    }
    named_bar_sync(2, SUMM_THREADS_F);
    // k~ and omega: thread t does channel pairs of chunk q
#pragma unroll 1
    for (int i = t; i < NCH * (D / 2); i += SUMM_THREADS_F) {
      const int q = i / (D / 2), ch = 2 * (i % (D / 2));
      const int64_t c = c0 + q;
      const bool own = c >= ca && c < cb;
      float k2[2], o2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        k2[h] = (sc.red[0][q][ch + h] + sc.red[1][q][ch + h]) * (1.0f / (float)CC);
        const float e = own ? sc.eps[c - c_lo][ch + h] : 0.f;
        o2[h] = omega_of(k2[h], e, fa.cfg);
      }
      sc.om[q][ch] = o2[0];
      sc.om[q][ch + 1] = o2[1];
      if (own) *reinterpret_cast<uint32_t*>(fa.ks + ((size_t)u * fa.nC + (size_t)c) * D + ch) = pack_bf16(k2[0], k2[1]);
    }
    named_bar_sync(2, SUMM_THREADS_F);
    // 2. the logit of tile row t; softmax over its chunk
    {
      const int q = t / CC;
      float a4[4] = {0.f, 0.f, 0.f, 0.f};
      const uint8_t* rowp = kt + t * 128;
#pragma unroll 4
      for (int pp = 0; pp < TPR; ++pp) {
        const uint4 x = *reinterpret_cast<const uint4*>(rowp + (pp >> 3) * (BN * 128) + ((((uint32_t)pp & 7u) ^ (uint32_t)(t & 7)) << 4));
        const float4 o0 = *reinterpret_cast<const float4*>(&sc.om[q][pp * 8]);
        const float4 o1 = *reinterpret_cast<const float4*>(&sc.om[q][pp * 8 + 4]);
        float f[8];
        unpack16<__nv_bfloat16>(x, f);
        float& a = a4[pp & 3];
        a = fmaf(f[0], o0.x - 0.5f * f[0], a); a = fmaf(f[1], o0.y - 0.5f * f[1], a);
        a = fmaf(f[2], o0.z - 0.5f * f[2], a); a = fmaf(f[3], o0.w - 0.5f * f[3], a);
        a = fmaf(f[4], o1.x - 0.5f * f[4], a); a = fmaf(f[5], o1.y - 0.5f * f[5], a);
        a = fmaf(f[6], o1.z - 0.5f * f[6], a); a = fmaf(f[7], o1.w - 0.5f * f[7], a);
      }
      const float a = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      float m = a;
      constexpr int WR = CC < 32 ? CC : 32;
#pragma unroll
      for (int o = 1; o < WR; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if constexpr (CC == 64) {
        if (lane == 0) sc.st[0][w] = m;
        named_bar_sync(2, SUMM_THREADS_F);
        m = fmaxf(sc.st[0][0], sc.st[0][1]);
      }
      const float pr = __expf(a - m);
      sc.p[t] = pr;
      float l = pr;
#pragma unroll
      for (int o = 1; o < WR; o <<= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      if constexpr (CC == 64) {
        if (lane == 0) sc.st[1][w] = l;
      } else {
        if ((t & (CC - 1)) == 0) sc.l[q] = l;
      }
    }
    named_bar_sync(2, SUMM_THREADS_F);
    if (t == 0) {
      mbar_arrive(&sm->k_empty[sk]);
      tt<TRACE>(tl, 3, 20, j);
    }
    mbar_wait(&sm->v_full[sv], (j / NSV) & 1);
    const uint8_t* vt = reinterpret_cast<const uint8_t*>(sm->v[sv]);
    // 3. beta^ partial sums of every chunk
#pragma unroll 1
    for (int q = 0; q < NCH; ++q) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
      for (int k = 0; k < NRC; ++k) {
        const int r = q * CC + g + k * RPP;
        const uint4 x = *reinterpret_cast<const uint4*>(vt + poff + r * 128 + ((c16 ^ (uint32_t)(r & 7)) << 4));
        const float pr = sc.p[r];
        float f[8];
        unpack16<__nv_bfloat16>(x, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(pr, f[i], acc[i]);
      }
#pragma unroll
      for (int o = TPR; o < 32; o <<= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
      if (lane < TPR) {
        float4* dst = reinterpret_cast<float4*>(&sc.red[w][q][pc * 8]);
        dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      }
    }
    named_bar_sync(2, SUMM_THREADS_F);
    if (t == 0) mbar_arrive(&sm->v_empty[sv]);
#pragma unroll 1
    for (int i = t; i < NCH * (D / 2); i += SUMM_THREADS_F) {
      const int q = i / (D / 2), ch = 2 * (i % (D / 2));
      const int64_t c = c0 + q;
      if (c >= ca && c < cb) {
        const float il = 1.0f / (CC == 64 ? sc.st[1][0] + sc.st[1][1] : sc.l[q]);
        const float y0 = (sc.red[0][q][ch] + sc.red[1][q][ch]) * il;
        const float y1 = (sc.red[0][q][ch + 1] + sc.red[1][q][ch + 1]) * il;
        *reinterpret_cast<uint32_t*>(fa.vs + ((size_t)u * fa.nC + (size_t)c) * D + ch) = pack_bf16(y0, y1);
      }
    }
    named_bar_sync(2, SUMM_THREADS_F);  // the exchange buffers are reused by the next tile
    if (t == 0) tt<TRACE>(tl, 3, 14, j);
  }
  // publish: the owned summaries are complete
  fence_proxy_async_global();
  named_bar_sync(2, SUMM_THREADS_F);
  if (t == 0) {
    __threadfence();
    st_release_gpu(fa.ws + 4 + (size_t)u * fa.n_qt + qt, epoch + 1u);
    tt<TRACE>(tl, 3, 15, 0);
  }
}

// Does walk step j (a local tile) hold a chunk the CTA summarises?  (order 2)
template <typename Plan>
__device__ __forceinline__ bool owns_chunks(const Plan& plan, int j, int C, int nC) {
  if (plan.summary(j)) return false;
  const int64_t b = plan.base(j);
  const int64_t c_lo = plan.n0 / C, c_hi = min((int64_t)nC, (plan.nlast + 1) / C);
  return max(c_lo, b / C) < min(c_hi, (b + BN) / C);
}

// FC = 0: summaries provided (or computed by a separate launch); FC = C in {16, 32, 64}: the
// chunk summaries are computed in-kernel (one instantiation per chunk size keeps the code that
// the instruction cache has to hold small)
// RP: in-kernel RoPE -- 0 none; 1 / 2 Q and the local K tiles (interleaved / half-split pairs);
// 3 / 4 Q only, the keys (and their summaries) come in rotated (EVA_ROPE_K_ROTATED).
constexpr int rope_style(int rp) { return rp == 0 ? 0 : (rp - 1) % 2 + 1; }
constexpr bool rope_k(int rp) { return rp == 1 || rp == 2; }
constexpr int prefill_threads(int fc, int rp) { return rope_k(rp) ? NTHREADS_R : fc ? NTHREADS_F : NTHREADS; }

template <int D, int NSTAGE, bool TRACE = false, int SMX = -1, int FC = 0, int RP = 0>
__global__ void __launch_bounds__(prefill_threads(FC, RP), 2)
prefill_sm100_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                     const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mKs,
                     const __grid_constant__ CUtensorMap mVs, const __grid_constant__ CUtensorMap mO,
                     const PrefillRange rg, int C, int W, int mode, float scale_log2,
                     float bias_log2, float* __restrict__ lse, int overlap, int overlap_order_sum_first,
                     const __grid_constant__ FusedArgs fa, const __grid_constant__ RopeArgs ra) {
  constexpr bool FUSED = FC != 0;
  static_assert(!(FC && RP), "in-kernel summaries and in-kernel RoPE are separate variants");
  constexpr int RSTY = rope_style(RP);  // RopeWalker style
  constexpr bool RK = rope_k(RP);       // the local K tiles are rotated here too
  extern __shared__ uint8_t smem_raw[];
  using SM = Smem<D, NSTAGE, FC != 0>;
  constexpr int NSK = SM::NSK, NSV = SM::NSV;
  if constexpr (SM::PAD == 0) {
    if ((reinterpret_cast<uintptr_t>(smem_raw) & 1023) != 0) __trap();
  }
  // 1 KB aligned by an offset from smem_raw (not an integer round trip), so the compiler keeps
  // every access through sm in the shared window (LDS/STS, not generic loads)
  SM* sm = reinterpret_cast<SM*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TileTrace* tl = nullptr;
  if constexpr (TRACE) {
    __shared__ TileTrace tlog_s;
    tl = &tlog_s;
    if (threadIdx.x < TT_ROLES) tl->n[threadIdx.x] = 0;
    if (threadIdx.x == 0) tl->slot = tt_slot();
    // per-CTA entry / exit (globaltimer ns, comparable across SMs) after the 4 slot logs
    const int id = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0 && g_trace2 && id < TT_MAX_CTAS)
      g_trace2[TT_SLOTS * TT_ROLES * TT_PER_ROLE + 2 * id] = globaltimer_ns();
  }
  if constexpr (FUSED) {
    // Fused: query tiles are handed out by a monotone ticket, so every tile whose summaries a
    // CTA waits for (the same unit's tiles <= its own) belongs to a CTA that is already
    // resident -- and that CTA publishes them after its own local tiles, which wait on nobody.
    pdl_wait();  // the workspace counters of the previous launch on this stream are final
    if (threadIdx.x == 0) {
      sm->ticket = (int)atomicAdd(fa.ws, 1u);
      sm->epoch = *reinterpret_cast<volatile uint32_t*>(fa.ws + 2);
    }
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV);
    tma_prefetch(&mKs); tma_prefetch(&mVs); tma_prefetch(&mO);
    mbar_init(&sm->q_full, 1);
    for (int s = 0; s < NSK; ++s) {
      mbar_init(&sm->k_full[s], 1);
      // fused: + the summary side's release (by the summary warps for a tile with owned
      // chunks, by the producer at issue otherwise)
      mbar_init(&sm->k_empty[s], FUSED ? 2 : 1);
    }
    for (int s = 0; s < NSV; ++s) {
      mbar_init(&sm->v_full[s], 1);
      mbar_init(&sm->v_empty[s], FUSED ? 2 : 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->s_full[b], 1);
      mbar_init(&sm->p_full[b], 128);
    }
    mbar_init(&sm->o_done, 1);
    mbar_init(&sm->o_final, 1);
    if constexpr (RP != 0) {
      mbar_init(&sm->q_rot, prefill_threads(FC, RP) - 64);
      for (int s = 0; s < NSK; ++s) mbar_init(&sm->k_rot[s], 32 * ROPE_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(&sm->tmem_base, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm->tmem_base;
  int qt = blockIdx.x, u = blockIdx.y;
  uint32_t epoch = 0;
  if constexpr (FUSED) {
    // fa.order 1 (default): tile-major -- the tiles whose summaries a tile reads were
    // dispatched a row of units earlier (measured 1.20 ms at configs[2], though the K/V reuse
    // distance grows to a wave: +0.8 GB of DRAM reads); 0: unit-major -- a unit's tiles run
    // close together and share its K/V and summaries in L2 (1.61 GB), but a tile then waits
    // for its neighbours' summaries (1.65 ms)
    if (fa.order) {
      qt = sm->ticket / fa.units;
      u = sm->ticket % fa.units;
    } else {
      qt = sm->ticket % fa.n_qt;
      u = sm->ticket / fa.n_qt;
    }
    epoch = sm->epoch;
  }
  RangePlan plan(qt, rg, C, W, mode, FUSED);
  if constexpr (!FUSED) plan.order = overlap ? 0 : (overlap_order_sum_first ? 1 : 0);
  const int qrow = qt * BM;  // TMA row of this query tile in Q / O
  const int NT = plan.count();
  // PDL: by default every thread waits for the previous grid here.  With `overlap` (the
  // previous grid is the eva_summarize producing Ksum/Vsum and Q, K, V were complete before
  // it) only the producer waits, right before its first summary-tile access, so the local
  // tiles (processed first) overlap the summarize kernel's tail.
  if (!FUSED && !overlap) pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) tt<TRACE>(tl, 0, 1, 0);

  if constexpr (RP != 0) {
    // in-kernel RoPE of the Q tile by the softmax and rope warps (idle until S(0) anyway)
    if (warp >= 2) {
      mbar_wait(&sm->q_full, 0);
      RopeWalker<RSTY> rw;
      rw.init(ra, (int)threadIdx.x - 64, prefill_threads(FC, RP) - 64);
      rw.run(reinterpret_cast<uint8_t*>(sm->q), BM, plan.n0);
      fence_proxy_async_smem();  // generic-proxy writes -> the MMA's async-proxy reads
      mbar_arrive(&sm->q_rot);
    }
  }
  // Producer and MMA roles run on whole warps (warp-uniform control flow keeps every
  // descriptor and coordinate in uniform registers); one elected lane issues.
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(&sm->q_full, BM * D * 2);
      for (int kb = 0; kb < D / 64; ++kb)
        tma_load_3d(sm->q + kb * BM * 64, &mQ, &sm->q_full, kb * 64, qrow, u);
    }
    __syncwarp();
    bool waited = !overlap && !FUSED;
    auto wait_summaries = [&](int j) {
      if (!waited && plan.summary(j)) {
        if constexpr (FUSED) {
          // chunks [0, nsum(n_last)) are read: wait for the flags of their owner tiles
          // (tile of chunk c = ((c+1)C - 1) / 128 <= qt), all lanes polling in parallel
          if (lane == 0) tt<TRACE>(tl, 0, 16, j);
          if (plan.s_end > 0) {
            const int last = (int)((plan.s_end * C - 1) / BM);
            const uint32_t* fl = fa.ws + 4 + (size_t)u * fa.n_qt;
            for (int i = lane; i <= last; i += 32) {
              const uint64_t t0 = globaltimer_ns();
              while (ld_relaxed_gpu(fl + i) != epoch + 1u) {
                __nanosleep(32);
                // watchdog: a flag that never comes is a bug -- fail the launch, never hang the GPU
                if (globaltimer_ns() - t0 > 2000000000ull) __trap();
              }
            }
          }
          __syncwarp();
          __threadfence();  // acquire: order the summary reads after the flags seen above
          fence_proxy_async_global();
          if (lane == 0) tt<TRACE>(tl, 0, 17, j);
        } else {
          pdl_wait();
        }
        waited = true;
      }
    };
    auto prefetch_rest = [&] {
      // The ring holds only NSTAGE tiles; pull every later K/V tile of this CTA into L2 now
      // so its TMA load later on is an L2 hit instead of a full DRAM round trip (summary
      // tiles only once they are known to be complete).
      if (elect_one()) {
      for (int j = NSV < NSK ? NSV : NSK; j < NT; ++j) {
        if (!waited && plan.summary(j)) break;
        const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
        const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
        for (int kb = 0; kb < D / 64; ++kb) {
          tma_prefetch_l2_3d(mk, kb * 64, plan.row(j), u);
          tma_prefetch_l2_3d(mv, kb * 64, plan.row(j), u);
        }
      }
      }
      __syncwarp();
    };
    // Issue order K(0), K(1), V(0), K(2), V(1), ...: K(j+1) waits only for S(j+1-NSTAGE)
    // to finish reading its slot, V(j) for PV(j-NSTAGE).
    auto load_k = [&](int j) {
      const int s = j % NSK;
      if (j >= NSK) mbar_wait(&sm->k_empty[s], ((j / NSK) - 1) & 1);
      if (lane == 0) tt<TRACE>(tl, 0, 11, j);
      wait_summaries(j);
      const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm->k_full[s], BN * D * 2);
        for (int kb = 0; kb < D / 64; ++kb)
          tma_load_3d(sm->k[s] + kb * BN * 64, mk, &sm->k_full[s], kb * 64, plan.row(j), u);
        if (FUSED && !owns_chunks(plan, j, C, fa.nC)) mbar_arrive(&sm->k_empty[s]);  // summary side
      }
      __syncwarp();
      if (lane == 0) tt<TRACE>(tl, 0, 12, j);
    };
    auto load_v = [&](int j) {
      const int s = j % NSV;
      if (j >= NSV) mbar_wait(&sm->v_empty[s], ((j / NSV) - 1) & 1);
      wait_summaries(j);
      const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm->v_full[s], BN * D * 2);
        for (int kb = 0; kb < D / 64; ++kb)
          tma_load_3d(sm->v[s] + kb * BN * 64, mv, &sm->v_full[s], kb * 64, plan.row(j), u);
        if (FUSED && !owns_chunks(plan, j, C, fa.nC)) mbar_arrive(&sm->v_empty[s]);
      }
      __syncwarp();
    };
    // Fused: every local tile's K AND V are issued before the first summary-tile load waits for
    // the ready flags -- that wait may be on this CTA's own summaries (W = C), which need them.
    auto sum_next = [&](int j) { return FUSED && j + 1 < NT && plan.summary(j + 1) && !plan.summary(j); };
    load_k(0);
    if (sum_next(0)) {
      load_v(0);
      load_k(1);
    } else {
      if (NT > 1) load_k(1);
      load_v(0);
    }
    prefetch_rest();  // after the first tiles: they are on the critical path
    for (int j = 1; j < NT; ++j) {
      if (sum_next(j)) {
        load_v(j);
        load_k(j + 1);
      } else {
        if (j + 1 < NT) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(BM, BN, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BM, D, true);
    const uint32_t q_addr = smem_u32(sm->q);
    mbar_wait(RP ? &sm->q_rot : &sm->q_full, 0);
    if (lane == 0) tt<TRACE>(tl, 1, 2, 0);
    for (int j = 0; j <= NT; ++j) {
      if (j < NT) {
        const int s = j % NSK;
        mbar_wait(RK ? &sm->k_rot[s] : &sm->k_full[s], (j / NSK) & 1);
        if (lane == 0) tt<TRACE>(tl, 1, 3, j);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sm->k[s]);
        const uint32_t d_tmem = tmem + (uint32_t)(j & 1) * BN;
        if (elect_one()) {
          tt<TRACE>(tl, 1, 22, j);
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
            const uint64_t a = smem_desc_sw128(q_addr + kb * (BM * 128) + off, 16, 1024);
            const uint64_t b = smem_desc_sw128(k_addr + kb * (BN * 128) + off, 16, 1024);
            mma_ss(d_tmem, a, b, idesc_s, ks > 0 ? 1u : 0u);
          }
          tt<TRACE>(tl, 1, 23, j);
          mma_commit(&sm->s_full[j & 1]);
          mma_commit(&sm->k_empty[s]);
        }
        __syncwarp();
        if (lane == 0) tt<TRACE>(tl, 1, 4, j);
      }
      if (j >= 1) {
        const int jj = j - 1, s = jj % NSV;
        mbar_wait(&sm->p_full[jj & 1], (jj >> 1) & 1);
        if (lane == 0) tt<TRACE>(tl, 1, 5, jj);
        mbar_wait(&sm->v_full[s], (jj / NSV) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sm->v[s]);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < BN / 16; ++ks) {
            const uint32_t a_tmem = tmem + (uint32_t)(jj & 1) * BN + ks * 8;
            const uint64_t b = smem_desc_sw128(v_addr + ks * 16 * 128, BN * 128, 1024);
            mma_ts(tmem + TM_O, a_tmem, b, idesc_o, (jj > 0 || ks > 0) ? 1u : 0u);
          }
          mma_commit(&sm->v_empty[s]);
          mma_commit(&sm->o_done);
          if (jj == NT - 1) mma_commit(&sm->o_final);
        }
        __syncwarp();
        if (lane == 0) tt<TRACE>(tl, 1, 6, jj);
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ softmax warps
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int64_t n = plan.n0 + r;
    const bool valid = n < rg.q0 + rg.nq;
    const Vis rr = visible_set(valid ? n : plan.nlast, C, W, mode, rg.q0 + rg.nq);
    const uint32_t t_lane = tmem + ((uint32_t)(quad * 32) << 16);
    float m_ref = -INFINITY, l = 0.f;
    const bool tw = warp == 2 && lane == 0;
    for (int j = 0; j < NT; ++j) {
      mbar_wait(&sm->s_full[j & 1], (j >> 1) & 1);
      if (tw) tt<TRACE>(tl, 2, 7, j);
      tc_fence_after();
      const int64_t base = plan.base(j);
      int vlo, vhi, xlo = 0, xhi = 0;
      float bias2 = 0.f;
      if (plan.summary(j)) {
        vlo = (int)max((int64_t)0, -base);  // order 2: rows before chunk 0 are zero-filled
        if (mode == EVA_NONCAUSAL) {  // every summary except those of the row's own block
          vhi = (int)min((int64_t)BN, (int64_t)rg.nsl - base);
          xlo = (int)max((int64_t)-1, min((int64_t)BN, rr.s1 - base));
          xhi = (int)max((int64_t)-1, min((int64_t)BN, rr.s2 - base));
        } else {
          vhi = (int)min((int64_t)BN, rr.s1 - base);
        }
        bias2 = bias_log2;
      } else {
        vlo = (int)max((int64_t)0, rr.lo - base);
        vhi = (int)min((int64_t)BN, rr.hi - base);
      }
      if (!valid) vhi = vlo;
      if constexpr (SMX < 0)
        softmax_tile_mx<D>(t_lane + (uint32_t)(j & 1) * BN, t_lane + TM_O, vlo, vhi, xlo, xhi, bias2,
                           scale_log2, m_ref, l, [&] { mbar_wait(&sm->o_done, (j - 1) & 1); });
      else
        softmax_tile2<D, SMX>(t_lane + (uint32_t)(j & 1) * BN, t_lane + TM_O, vlo, vhi, xlo, xhi, bias2,
                              scale_log2, m_ref, l, [&] { mbar_wait(&sm->o_done, (j - 1) & 1); });
      mbar_arrive(&sm->p_full[j & 1]);
      if (tw) tt<TRACE>(tl, 2, 8, j);
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(&sm->o_final, 0);
    if (tw) tt<TRACE>(tl, 2, 9, 0);
    tc_fence_after();
    const float inv_l = l > 0.f ? 1.0f / l : 0.f;
    uint8_t* qs = reinterpret_cast<uint8_t*>(sm->q);
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t o[32];
      tmem_ld32(t_lane + TM_O + cc * 32, o);
      tmem_wait_ld();
      const int kb = (cc * 32) / 64, c16_0 = ((cc * 32) % 64) / 8;
      uint8_t* rowp = qs + kb * (BM * 128) + r * 128;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint4 w;
        w.x = pack_bf16(__uint_as_float(o[8 * g + 0]) * inv_l, __uint_as_float(o[8 * g + 1]) * inv_l);
        w.y = pack_bf16(__uint_as_float(o[8 * g + 2]) * inv_l, __uint_as_float(o[8 * g + 3]) * inv_l);
        w.z = pack_bf16(__uint_as_float(o[8 * g + 4]) * inv_l, __uint_as_float(o[8 * g + 5]) * inv_l);
        w.w = pack_bf16(__uint_as_float(o[8 * g + 6]) * inv_l, __uint_as_float(o[8 * g + 7]) * inv_l);
        *reinterpret_cast<uint4*>(rowp + (((c16_0 + g) ^ (r & 7)) * 16)) = w;
      }
    }
    if (valid && lse) lse[(size_t)u * rg.nq + (size_t)(n - rg.q0)] = (m_ref + __log2f(l)) * 0.69314718055994531f;
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (warp == 2 && lane == 0) {
      for (int kb = 0; kb < D / 64; ++kb) tma_store_3d(&mO, sm->q + kb * BM * 64, kb * 64, qrow, u);
      tma_store_commit();
      tma_store_wait_read();
      tt<TRACE>(tl, 2, 10, 0);
    }
  } else {
    // ------------------------------------------------------------ summary warps (fused)
    if constexpr (FUSED) fused_summaries<D, FC, TRACE>(sm, plan, fa, u, qt, epoch, tl);
    // ------------------------------------------------------------ rope warps (in-kernel RoPE)
    if constexpr (RK) {
      RopeWalker<RSTY> rw;
      rw.init(ra, (int)threadIdx.x - NTHREADS, 32 * ROPE_WARPS);
      for (int j = 0; j < NT; ++j) {
        const int s = j % NSK;
        mbar_wait(&sm->k_full[s], (j / NSK) & 1);
        if (!plan.summary(j)) {  // summary tiles hold summaries of rotated keys already
          rw.run(reinterpret_cast<uint8_t*>(sm->k[s]), BN, plan.base(j));
          fence_proxy_async_smem();
        }
        mbar_arrive(&sm->k_rot[s]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (TRACE) {
    const int slot = tl->slot;
    if (slot >= 0 && g_trace2) {
      for (int i = threadIdx.x; i < TT_ROLES * TT_PER_ROLE; i += blockDim.x) {
        const int r = i / TT_PER_ROLE, k = i % TT_PER_ROLE;
        g_trace2[(size_t)slot * TT_ROLES * TT_PER_ROLE + i] = k < tl->n[r] ? tl->ev[r][k] : 0ull;
      }
    }
    const int id = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0 && g_trace2 && id < TT_MAX_CTAS)
      g_trace2[TT_SLOTS * TT_ROLES * TT_PER_ROLE + 2 * id + 1] = globaltimer_ns();
  }
  if constexpr (FUSED) {
    // the last CTA to finish resets the ticket and done counters and advances the epoch
    if (threadIdx.x == 0) {
      __threadfence();
      const uint32_t d = atomicAdd(fa.ws + 1, 1u);
      if (d == (uint32_t)fa.total - 1u) {
        fa.ws[0] = 0u;
        fa.ws[1] = 0u;
        __threadfence();
        fa.ws[2] = epoch + 1u;
      }
    }
  }
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 3-D bf16 map over [units, rows, D] with a {64, box_rows, 1} box, 128-byte swizzle.
bool make_map(CUtensorMap* m, const void* base, int units, int rows, int D, int box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)rows, (cuuint64_t)units};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)rows * D * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tile order when not overlapping the summarize kernel: summary tiles first (measured 613 vs
// 629 us at configs[2]); EVA_PREFILL_SUMFIRST=0 selects local-first for measurements.
int tile_sum_first() {
  static const int v = [] {
    const char* e = getenv("EVA_PREFILL_SUMFIRST");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// ---- workspace of the fused launch: [ticket, done, epoch, pad] + one ready flag per
// (unit, query tile), zero-initialised once; the kernel leaves ticket/done at 0 and advances
// the epoch, so one buffer serves every later launch on the same stream (graph replays too).
struct FusedWs {
  uint32_t* p = nullptr;
  size_t flags = 0;
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, FusedWs> g_ws;

cudaError_t fused_workspace(size_t nflags, cudaStream_t s, uint32_t** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_ws_mu);
  FusedWs& w = g_ws[{dev, s}];
  if (w.flags < nflags) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    e = cudaStreamIsCapturing(s, &cs);
    if (e != cudaSuccess) return e;
    if (cs != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;
    if (w.p) {  // the previous buffer may still be read by work on this stream
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      cudaFree(w.p);
      w.p = nullptr;
      w.flags = 0;
    }
    const size_t n = std::max<size_t>(nflags, 4096);
    if ((e = cudaMalloc(&w.p, (n + 4) * sizeof(uint32_t))) != cudaSuccess) return e;
    if ((e = cudaMemset(w.p, 0, (n + 4) * sizeof(uint32_t))) != cudaSuccess) return e;
    w.flags = n;
  }
  *out = w.p;
  return cudaSuccess;
}

template <int D, int NSTAGE, bool TRACE = false, int SMX = -1, int FC = 0, int RP = 0>
cudaError_t launch_t(const eva_config& cfg, const PrefillRange& rg, const void* Q, const void* K,
                     const void* V, const void* Ksum, const void* Vsum, void* O, float* lse,
                     cudaStream_t s, bool overlap = false, const float* eps = nullptr,
                     const RopeArgs* rap = nullptr) {
  constexpr bool FUSED = FC != 0;
  if constexpr (!TRACE && SMX == -1 && !FUSED && RP == 0) {  // the packed softmax (softmax_tile2)
    return launch_t<D, NSTAGE, false, 0, 0>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap, eps);
  }
  const int BH = cfg.bh_count, nC = rg.nsl;
  if (rg.nq == 0) return cudaSuccess;
  CUtensorMap mQ, mK, mV, mKs, mVs, mO;
  bool ok = make_map(&mQ, Q, BH, rg.nq, D, BM) && make_map(&mK, K, BH, rg.nkv, D, BN) &&
            make_map(&mV, V, BH, rg.nkv, D, BN) && make_map(&mO, O, BH, rg.nq, D, BM);
  if (nC > 0) {
    ok = ok && make_map(&mKs, Ksum, BH, nC, D, BN) && make_map(&mVs, Vsum, BH, nC, D, BN);
  } else {  // never read (no summary tiles); any valid map will do
    mKs = mK;
    mVs = mV;
  }
  if (!ok) return cudaErrorInvalidValue;
  using K_t = decltype(&prefill_sm100_kernel<D, NSTAGE, TRACE, SMX, FC, RP>);
  K_t kern = prefill_sm100_kernel<D, NSTAGE, TRACE, SMX, FC, RP>;
  const size_t smem = sizeof(Smem<D, NSTAGE, FUSED>) + Smem<D, NSTAGE, FUSED>::PAD;
  {
    cudaError_t e = set_smem_attr((const void*)kern, smem);
    if (e != cudaSuccess) return e;
  }
  const int n_qt = (rg.nq + BM - 1) / BM;
  FusedArgs fa = {};
  dim3 grid(n_qt, BH);
  if constexpr (FUSED) {
    uint32_t* ws = nullptr;
    cudaError_t e = fused_workspace((size_t)BH * n_qt, s, &ws);
    if (e != cudaSuccess) return e;
    fa.cfg = cfg;
    fa.K = (const __nv_bfloat16*)K;
    fa.V = (const __nv_bfloat16*)V;
    fa.T = rg.nkv;
    fa.ks = (__nv_bfloat16*)Ksum;
    fa.vs = (__nv_bfloat16*)Vsum;
    fa.eps = eps;
    fa.ws = ws;
    fa.nC = nC;
    fa.n_qt = n_qt;
    fa.units = BH;
    fa.total = n_qt * BH;
    static const int order = [] {
      const char* e = getenv("EVA_FUSED_ORDER");
      return e ? atoi(e) : 1;
    }();
    fa.order = order;
    grid = dim3(n_qt * BH, 1);
  }
  const float scale_log2 = cfg.scale * 1.4426950408889634f;
  const RopeArgs ra = rap ? *rap : RopeArgs{};
  cudaError_t e = launch_pdl(kern, grid, dim3(prefill_threads(FC, RP)), smem, s, mQ, mK, mV,
                             mKs, mVs, mO, rg, cfg.chunk, cfg.window, cfg.mode, scale_log2,
                             cfg.summary_bias * 1.4426950408889634f, lse, overlap ? 1 : 0, tile_sum_first(), fa,
                             ra);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t debug_set_summ_trace(unsigned long long* p, cudaStream_t s);  // summarize_bulk.cu

bool make_tma_map_bf16(CUtensorMap* m, const void* base, int units, int rows, int D, int box_rows) {
  return make_map(m, base, units, rows, D, box_rows);
}

cudaError_t debug_trace_tile(const eva_config& cfg, const void* Q, const void* K, const void* V,
                             const void* Ksum, const void* Vsum, void* O, float* lse,
                             unsigned long long* trace_dev, bool fused, cudaStream_t s) {
  // Under stream capture the symbols keep the values an eager call set (a captured copy from a
  // host stack variable would read a dead address at replay).
  cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(s, &cap_st);
  if (e != cudaSuccess) return e;
  const bool capturing = cap_st != cudaStreamCaptureStatusNone;
  if (!capturing) e = cudaMemcpyToSymbolAsync(g_trace2, &trace_dev, sizeof(trace_dev), 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  static const int mid = [] {
    const char* v = getenv("EVA_TRACE_MID");
    return v ? atoi(v) : 150;
  }();
  if (!capturing) e = cudaMemcpyToSymbolAsync(g_trace_mid, &mid, sizeof(mid), 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  const PrefillRange rg = full_range(cfg);
  if (fused) {  // traced for C = 64 (the configs' chunk size)
    if (!prefill_fused_supported(cfg) || cfg.chunk != 64) return cudaErrorNotSupported;
    if (cfg.d_head == 128)
      return launch_t<128, 2, true, -1, 64>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, false, nullptr);
    return launch_t<64, 3, true, -1, 64>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, false, nullptr);
  }
  // EVA_TRACE_OVERLAP=1: the traced summarize kernel (CTA spans at trace[8960 + 2 i]) and then the
  // traced prefill in EVA_PREFILL_OVERLAP mode, as the step launches them
  // (EVA_TRACE_OVERLAP=2: the same pair with the prefill NOT in overlap mode)
  static const int ovl_mode = [] {
    const char* v = getenv("EVA_TRACE_OVERLAP");
    return v ? atoi(v) : 0;
  }();
  const bool ovl = ovl_mode == 1;
  if (ovl_mode) {
    if (!capturing) e = debug_set_summ_trace(trace_dev + TT_SLOTS * TT_ROLES * TT_PER_ROLE + 2 * TT_MAX_CTAS, s);
    if (e != cudaSuccess) return e;
    e = launch_summarize_bulk(cfg, K, V, nullptr, const_cast<void*>(Ksum), const_cast<void*>(Vsum), 0, s);
    if (e != cudaSuccess) return e;
  }
  if (cfg.d_head == 128) return launch_t<128, 2, true>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, ovl);
  if (cfg.d_head == 64) return launch_t<64, 3, true>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, ovl);
  return cudaErrorNotSupported;
}

bool prefill_sm100_supported(const eva_config& cfg) {
  return cfg.dtype == EVA_BF16 && (cfg.d_head == 64 || cfg.d_head == 128) && encode_fn() != nullptr;
}

// The in-kernel summaries (EVA_SUMMARIES_FUSED): causal modes, whole-sequence call, chunks of
// 16, 32 or 64 rows (whole chunks per 64-key tile, at most 4 of them).
bool prefill_fused_supported(const eva_config& cfg) {
  if (!prefill_sm100_supported(cfg) || cfg.mode == EVA_NONCAUSAL) return false;
  return cfg.chunk == 16 || cfg.chunk == 32 || cfg.chunk == 64;
}

cudaError_t launch_prefill_sm100(const eva_config& cfg, const PrefillRange& rg, const void* Q,
                                 const void* K, const void* V, const void* Ksum, const void* Vsum,
                                 void* O, float* lse, uint32_t variant, cudaStream_t s) {
  if (cfg.bh_count == 0) return cudaSuccess;
  const bool overlap = (variant & 0x100u) != 0;  // EVA_PREFILL_OVERLAP
  if (cfg.d_head == 128) return launch_t<128, 2>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
  if (cfg.d_head == 64) return launch_t<64, 3>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
  return cudaErrorNotSupported;
}

cudaError_t launch_prefill_sm100_fused(const eva_config& cfg, const void* Q, const void* K, const void* V,
                                       const float* eps, void* Ksum, void* Vsum, void* O, float* lse,
                                       cudaStream_t s) {
  if (cfg.bh_count == 0) return cudaSuccess;
  if (!prefill_fused_supported(cfg)) return cudaErrorNotSupported;
  const PrefillRange rg = full_range(cfg);
#define EVA_FUSED_LAUNCH(D_, NS_)                                                                     \
  switch (cfg.chunk) {                                                                                \
    case 16: return launch_t<D_, NS_, false, -1, 16>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, false, eps); \
    case 32: return launch_t<D_, NS_, false, -1, 32>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, false, eps); \
    default: return launch_t<D_, NS_, false, -1, 64>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, false, eps); \
  }
  if (cfg.d_head == 128) EVA_FUSED_LAUNCH(128, 2)
  if (cfg.d_head == 64) EVA_FUSED_LAUNCH(64, 3)
#undef EVA_FUSED_LAUNCH
  return cudaErrorNotSupported;
}

// In-kernel RoPE (eva_attn_prefill_rope): bf16, d in {64, 128}, whole-sequence call, rotary
// channels a power of two (>= 8 interleaved, >= 16 half-split) -- the rope warps' item split.
bool prefill_rope_supported(const eva_config& cfg, int rotary_dim, int style) {
  if (!prefill_sm100_supported(cfg)) return false;
  const int rd = rotary_dim ? rotary_dim : cfg.d_head;
  if (rd > cfg.d_head || (rd & (rd - 1)) != 0) return false;
  return style == EVA_ROPE_NEOX ? rd >= 16 : rd >= 8;
}

cudaError_t launch_prefill_sm100_rope(const eva_config& cfg, double log2_base, int rotary_dim, int style,
                                      const void* Q, const void* K, const void* V, const void* Ksum,
                                      const void* Vsum, void* O, float* lse, cudaStream_t s, bool k_rotated) {
  if (cfg.bh_count == 0) return cudaSuccess;
  if (!prefill_rope_supported(cfg, rotary_dim, style)) return cudaErrorNotSupported;
  const PrefillRange rg = full_range(cfg);
  RopeArgs ra{};
  ra.rd = rotary_dim ? rotary_dim : cfg.d_head;
  for (int j = 0; j < ra.rd / 2; ++j) ra.th[j] = std::exp2(log2_base * (-2.0 * (double)j / (double)ra.rd));
  const bool neox = style == EVA_ROPE_NEOX;
#define EVA_ROPE_LAUNCH(D_, NS_, RP_) \
  return launch_t<D_, NS_, false, 0, 0, RP_>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, false, nullptr, &ra)
  if (cfg.d_head == 128) {
    if (k_rotated) { if (neox) EVA_ROPE_LAUNCH(128, 2, 4); EVA_ROPE_LAUNCH(128, 2, 3); }
    if (neox) EVA_ROPE_LAUNCH(128, 2, 2);
    EVA_ROPE_LAUNCH(128, 2, 1);
  }
  if (k_rotated) { if (neox) EVA_ROPE_LAUNCH(64, 3, 4); EVA_ROPE_LAUNCH(64, 3, 3); }
  if (neox) EVA_ROPE_LAUNCH(64, 3, 2);
  EVA_ROPE_LAUNCH(64, 3, 1);
#undef EVA_ROPE_LAUNCH
}

cudaError_t prefill_fused_reserve(const eva_config& cfg, cudaStream_t s) {
  uint32_t* ws = nullptr;
  return fused_workspace((size_t)cfg.bh_count * ((cfg.T + BM - 1) / BM), s, &ws);
}

}  // namespace eva
