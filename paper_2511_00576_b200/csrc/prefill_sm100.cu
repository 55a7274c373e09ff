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
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "launch.h"
#include "sm100.cuh"

namespace eva {
namespace {

using namespace sm100;
constexpr int BM = 128;       // queries per tile
constexpr int BN = 64;        // keys per KV tile
constexpr int NTHREADS = 192;
constexpr uint32_t TMEM_COLS = 256;
constexpr uint32_t TM_O = 128;

// NSTAGE < 10: NSTAGE K and NSTAGE V slots.  NSTAGE = 10*NSK + NSV: separate ring depths
// (a deeper K ring lets the next K tiles stream in earlier; K is consumed one softmax period
// before V).  Deep-ring layouts are sized to fill the SM with two CTAs, so they are used
// without the 1 KB alignment pad (the dynamic window is 1 KB aligned; checked in-kernel).
template <int D, int NSTAGE>
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
  uint32_t tmem_base;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
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
  if (!__all_sync(0xffffffffu, full)) {
#pragma unroll
    for (int c = 0; c < 64; ++c)
      if (c < vlo || c >= vhi || (c >= xlo && c < xhi)) sr[c] = 0xff800000u;  // -inf
  }
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
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t o[32];
      tmem_ld32(o_addr + cc * 32, o);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
      tmem_st32(o_addr + cc * 32, o);
    }
    tmem_wait_st();
    l *= f;
  }
  if (grow) m_ref = mx;
  const float neg = (m_ref == -INFINITY ? 0.f : -m_ref) + bias2;
  uint32_t pk[32];
  float ls[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) ls[i] = 0.f;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const float p0 = ex2(fmaf(__uint_as_float(sr[2 * c]), scale_log2, neg));
    const float p1 = ex2(fmaf(__uint_as_float(sr[2 * c + 1]), scale_log2, neg));
    ls[(2 * c) & 7] += p0;
    ls[(2 * c + 1) & 7] += p1;
    pk[c] = pack_bf16(p0, p1);
  }
  l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
  tmem_st32(s_addr, pk);
  tmem_wait_st();
  tc_fence_before();
}

template <int D, typename WaitO>
__device__ __forceinline__ void softmax_tile(uint32_t s_addr, uint32_t o_addr, int vlo, int vhi,
                                             float scale_log2, float& m_ref, float& l,
                                             const WaitO& wait_o) {
  softmax_tile_mx<D>(s_addr, o_addr, vlo, vhi, 0, 0, 0.f, scale_log2, m_ref, l, wait_o);
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
  if (!__all_sync(0xffffffffu, full)) {
#pragma unroll
    for (int c = 0; c < 64; ++c)
      if (c < vlo || c >= vhi || (c >= xlo && c < xhi)) sr[c] = 0xff800000u;  // -inf
  }
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
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t o[32];
      tmem_ld32(o_addr + cc * 32, o);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const uint64_t v = ffma2(f2pack(__uint_as_float(o[i]), __uint_as_float(o[i + 1])), f2, 0ull);
        o[i] = (uint32_t)v;
        o[i + 1] = (uint32_t)(v >> 32);
      }
      tmem_st32(o_addr + cc * 32, o);
    }
    tmem_wait_st();
    l *= f;
  }
  if (grow) m_ref = mx;
  const float neg = (m_ref == -INFINITY ? 0.f : -m_ref) + bias2;
  const uint64_t sc2 = f2pack(scale_log2, scale_log2), ng2 = f2pack(neg, neg);
  uint32_t pk[32];
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
    pk[c] = pack_bf16(f2lo(p), f2hi(p));
  }
  const uint64_t s2 = fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3]));
  l += f2lo(s2) + f2hi(s2);
  tmem_st32(s_addr, pk);
  tmem_wait_st();
  tc_fence_before();
}

struct TilePlan {
  int n0, nlast, n_st, n_lt, lo0;
  __device__ TilePlan(int qt, int T, int C, int W, int mode) {
    n0 = qt * BM;
    nlast = min(n0 + BM - 1, T - 1);
    const Range rf = mask_range(n0, C, W, mode), rl = mask_range(nlast, C, W, mode);
    n_st = (int)((rl.nsum + BN - 1) / BN);
    lo0 = (int)rf.lo;
    n_lt = (nlast - lo0 + 1 + BN - 1) / BN;
  }
  __device__ int count() const { return n_st + n_lt; }
  __device__ bool summary(int j) const { return j < n_st; }
  __device__ int base(int j) const { return j < n_st ? j * BN : lo0 + (j - n_st) * BN; }
};

// TilePlan of a query-range call (eva_attn_prefill_range): query tile qt covers absolute
// positions [q0 + qt*BM, ...), local key tiles start at lo(n0) (absolute); row() maps a
// tile base to the TMA row of its tensor (key rows are stored from position k0).
struct RangePlan {
  int64_t n0, nlast, lo0, k0;
  int n_st, n_lt;
  __device__ RangePlan(int qt, const PrefillRange& rg, int C, int W, int mode) {
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
  }
  // Tile order: local tiles first, then the summary tiles (sum_first = 0) -- the local span
  // depends only on the inputs, so with EVA_PREFILL_OVERLAP it runs while the summarize
  // kernel is still finishing -- or summaries first (sum_first = 1).
  int sum_first = 0;
  __device__ int count() const { return n_st + n_lt; }
  __device__ bool summary(int j) const { return sum_first ? j < n_st : j >= n_lt; }
  __device__ int64_t base(int j) const {
    if (sum_first) return j < n_st ? (int64_t)j * BN : lo0 + (int64_t)(j - n_st) * BN;
    return j >= n_lt ? (int64_t)(j - n_lt) * BN : lo0 + (int64_t)j * BN;
  }
  __device__ int row(int j) const {
    if (sum_first) return j < n_st ? j * BN : (int)(lo0 - k0) + (j - n_st) * BN;
    return j >= n_lt ? (j - n_lt) * BN : (int)(lo0 - k0) + j * BN;
  }
};


// Debug timeline of the tile kernel (eva_debug_trace_prefill with variant 1): CTAs with
// linear id in {0, 1, 150, 151} log (globaltimer-free) clock64 events per role in shared
// memory and flush them to g_trace2 at exit.  Roles: 0 producer, 1 MMA, 2 softmax (warp 2
// lane 0).  kinds: 1 start, 2 Q arrived (MMA), 3 k_full(j) (MMA), 4 S(j) issued, 5 P(j)
// received (MMA), 6 PV(j) issued, 7 softmax got S(j), 8 softmax P(j) done, 9 o_final
// (epilogue start), 10 epilogue done, 11 producer slot free (j), 12 producer issued (j).
__device__ unsigned long long* g_trace2 = nullptr;
constexpr int TT_ROLES = 3, TT_PER_ROLE = 48, TT_SLOTS = 4;
struct TileTrace {
  unsigned long long ev[TT_ROLES][TT_PER_ROLE];
  int n[TT_ROLES];
};
__device__ __forceinline__ int tt_slot() {
  const int id = blockIdx.y * gridDim.x + blockIdx.x;
  return id == 0 ? 0 : id == 1 ? 1 : id == 150 ? 2 : id == 151 ? 3 : -1;
}
template <bool TRACE>
__device__ __forceinline__ void tt(TileTrace* tl, int role, int kind, int j) {
  if constexpr (TRACE) {
    if (tt_slot() >= 0) {
      const int i = tl->n[role];
      if (i < TT_PER_ROLE) tl->ev[role][i] = ((unsigned long long)clock64() << 24) | ((unsigned)kind << 16) | (unsigned)(j & 0xffff);
      tl->n[role] = i + 1;
    }
  }
}

template <int D, int NSTAGE, bool TRACE = false, int SMX = -1>
__global__ void __launch_bounds__(NTHREADS, 2)
prefill_sm100_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                     const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mKs,
                     const __grid_constant__ CUtensorMap mVs, const __grid_constant__ CUtensorMap mO,
                     const PrefillRange rg, int C, int W, int mode, float scale_log2,
                     float bias_log2, float* __restrict__ lse, int overlap, int overlap_order_sum_first) {
  extern __shared__ uint8_t smem_raw[];
  using SM = Smem<D, NSTAGE>;
  constexpr int NSK = SM::NSK, NSV = SM::NSV;
  if constexpr (SM::PAD == 0) {
    if ((reinterpret_cast<uintptr_t>(smem_raw) & 1023) != 0) __trap();
  }
  SM* sm = reinterpret_cast<SM*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.y;
  RangePlan plan(blockIdx.x, rg, C, W, mode);
  plan.sum_first = overlap ? 0 : (overlap_order_sum_first ? 1 : 0);
  const int qrow = blockIdx.x * BM;  // TMA row of this query tile in Q / O
  const int NT = plan.count();
  TileTrace* tl = nullptr;
  if constexpr (TRACE) {
    __shared__ TileTrace tlog_s;
    tl = &tlog_s;
    if (threadIdx.x < TT_ROLES) tl->n[threadIdx.x] = 0;
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV);
    tma_prefetch(&mKs); tma_prefetch(&mVs); tma_prefetch(&mO);
    mbar_init(&sm->q_full, 1);
    for (int s = 0; s < NSK; ++s) {
      mbar_init(&sm->k_full[s], 1);
      mbar_init(&sm->k_empty[s], 1);
    }
    for (int s = 0; s < NSV; ++s) {
      mbar_init(&sm->v_full[s], 1);
      mbar_init(&sm->v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->s_full[b], 1);
      mbar_init(&sm->p_full[b], 128);
    }
    mbar_init(&sm->o_done, 1);
    mbar_init(&sm->o_final, 1);
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
  // PDL: by default every thread waits for the previous grid here.  With `overlap` (the
  // previous grid is the eva_summarize producing Ksum/Vsum and Q, K, V were complete before
  // it) only the producer waits, right before its first summary-tile access, so the local
  // tiles (processed first) overlap the summarize kernel's tail.
  if (!overlap) pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) tt<TRACE>(tl, 0, 1, 0);

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
    bool waited = !overlap;
    auto wait_summaries = [&](int j) {
      if (!waited && plan.summary(j)) {
        pdl_wait();
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
      }
      __syncwarp();
    };
    load_k(0);
    if (NT > 1) load_k(1);
    load_v(0);
    prefetch_rest();  // after the first tiles: they are on the critical path
    for (int j = 1; j < NT; ++j) {
      if (j + 1 < NT) load_k(j + 1);
      load_v(j);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(BM, BN, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BM, D, true);
    const uint32_t q_addr = smem_u32(sm->q);
    mbar_wait(&sm->q_full, 0);
    if (lane == 0) tt<TRACE>(tl, 1, 2, 0);
    for (int j = 0; j <= NT; ++j) {
      if (j < NT) {
        const int s = j % NSK;
        mbar_wait(&sm->k_full[s], (j / NSK) & 1);
        if (lane == 0) tt<TRACE>(tl, 1, 3, j);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sm->k[s]);
        const uint32_t d_tmem = tmem + (uint32_t)(j & 1) * BN;
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
            const uint64_t a = smem_desc_sw128(q_addr + kb * (BM * 128) + off, 16, 1024);
            const uint64_t b = smem_desc_sw128(k_addr + kb * (BN * 128) + off, 16, 1024);
            mma_ss(d_tmem, a, b, idesc_s, ks > 0 ? 1u : 0u);
          }
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
  } else {
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
        vlo = 0;
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
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (TRACE) {
    const int slot = tt_slot();
    if (slot >= 0 && g_trace2) {
      for (int i = threadIdx.x; i < TT_ROLES * TT_PER_ROLE; i += blockDim.x) {
        const int r = i / TT_PER_ROLE, k = i % TT_PER_ROLE;
        g_trace2[(size_t)slot * TT_ROLES * TT_PER_ROLE + i] = k < tl->n[r] ? tl->ev[r][k] : 0ull;
      }
    }
  }
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ========================================================================== persistent tile kernel
// The one-tile-per-CTA kernel made persistent: two CTAs per SM walk the (unit, query tile)
// items w = blockIdx.x, + gridDim.x, ...  Ring indices and barrier phases run on global
// counters across items, so the next item's Q (released by the last S MMA of the current
// item), K/V tiles and first S MMAs stream in while the current item finishes; O is drained
// from TMEM by the softmax warps (o_free releases it for the next item's first PV) and
// written straight from registers (no smem staging, so Q's buffer is never shared).
template <int D, int NSTAGE>
struct __align__(1024) SmemP {
  static constexpr int NSK = NSTAGE >= 10 ? NSTAGE / 10 : NSTAGE;
  static constexpr int NSV = NSTAGE >= 10 ? NSTAGE % 10 : NSTAGE;
  __nv_bfloat16 q[BM * D];
  __nv_bfloat16 k[NSK][BN * D];
  __nv_bfloat16 v[NSV][BN * D];
  uint64_t q_full, q_empty;
  uint64_t k_full[NSK], v_full[NSV], k_empty[NSK], v_empty[NSV];
  uint64_t s_full[2], p_full[2], o_done, o_final, o_free;
  uint32_t tmem_base;
};

template <int D, int NSTAGE>
__global__ void __launch_bounds__(NTHREADS, 2)
prefill_persist_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                       const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mKs,
                       const __grid_constant__ CUtensorMap mVs, const PrefillRange rg, int C, int W, int mode,
                       float scale_log2, float bias_log2, float* __restrict__ lse, __nv_bfloat16* __restrict__ O,
                       int n_qt, int n_items) {
  extern __shared__ uint8_t smem_raw[];
  using SM = SmemP<D, NSTAGE>;
  constexpr int NSK = SM::NSK, NSV = SM::NSV;
  SM* sm = reinterpret_cast<SM*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto plan_of = [&](int w) {
    RangePlan p(w % n_qt, rg, C, W, mode);
    p.sum_first = 1;
    return p;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV);
    tma_prefetch(&mKs); tma_prefetch(&mVs);
    mbar_init(&sm->q_full, 1);
    mbar_init(&sm->q_empty, 1);
    for (int s = 0; s < NSK; ++s) {
      mbar_init(&sm->k_full[s], 1);
      mbar_init(&sm->k_empty[s], 1);
    }
    for (int s = 0; s < NSV; ++s) {
      mbar_init(&sm->v_full[s], 1);
      mbar_init(&sm->v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->s_full[b], 1);
      mbar_init(&sm->p_full[b], 128);
    }
    mbar_init(&sm->o_done, 1);
    mbar_init(&sm->o_final, 1);
    mbar_init(&sm->o_free, 128);
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
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    int tk = 0, tv = 0, ic = 0;  // global K tile, V tile and item counters
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++ic) {
      const RangePlan plan = plan_of(w);
      const int u = w / n_qt, qrow = (w % n_qt) * BM, NT = plan.count();
      if (ic > 0) mbar_wait(&sm->q_empty, (ic - 1) & 1);  // the last item's S MMAs are done
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm->q_full, BM * D * 2);
        for (int kb = 0; kb < D / 64; ++kb) tma_load_3d(sm->q + kb * BM * 64, &mQ, &sm->q_full, kb * 64, qrow, u);
        for (int j = 2; j < NT; ++j) {
          const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
          const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
          for (int kb = 0; kb < D / 64; ++kb) {
            tma_prefetch_l2_3d(mk, kb * 64, plan.row(j), u);
            tma_prefetch_l2_3d(mv, kb * 64, plan.row(j), u);
          }
        }
      }
      __syncwarp();
      auto load_k = [&](int j) {
        const int t = tk + j, s = t % NSK;
        if (t >= NSK) mbar_wait(&sm->k_empty[s], ((t / NSK) - 1) & 1);
        const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm->k_full[s], BN * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->k[s] + kb * BN * 64, mk, &sm->k_full[s], kb * 64, plan.row(j), u);
        }
        __syncwarp();
      };
      auto load_v = [&](int j) {
        const int t = tv + j, s = t % NSV;
        if (t >= NSV) mbar_wait(&sm->v_empty[s], ((t / NSV) - 1) & 1);
        const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm->v_full[s], BN * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->v[s] + kb * BN * 64, mv, &sm->v_full[s], kb * 64, plan.row(j), u);
        }
        __syncwarp();
      };
      load_k(0);
      for (int j = 0; j < NT; ++j) {
        if (j + 1 < NT) load_k(j + 1);
        load_v(j);
      }
      tk += NT;
      tv += NT;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(BM, BN, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BM, D, true);
    const uint32_t q_addr = smem_u32(sm->q);
    int t0 = 0, ic = 0;  // global tile counter at the item start, item counter
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++ic) {
      const int NT = plan_of(w).count();
      mbar_wait(&sm->q_full, ic & 1);
      for (int j = 0; j <= NT; ++j) {
        if (j < NT) {
          const int t = t0 + j, s = t % NSK;
          mbar_wait(&sm->k_full[s], (t / NSK) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sm->k[s]);
          const uint32_t d_tmem = tmem + (uint32_t)(t & 1) * BN;
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
              const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
              mma_ss(d_tmem, smem_desc_sw128(q_addr + kb * (BM * 128) + off, 16, 1024),
                     smem_desc_sw128(k_addr + kb * (BN * 128) + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
            }
            mma_commit(&sm->s_full[t & 1]);
            mma_commit(&sm->k_empty[s]);
            if (j == NT - 1) mma_commit(&sm->q_empty);  // Q is read by the S MMAs only
          }
          __syncwarp();
        }
        if (j >= 1) {
          const int jj = j - 1, t = t0 + jj, s = t % NSV;
          mbar_wait(&sm->p_full[t & 1], (t >> 1) & 1);
          if (jj == 0 && ic > 0) mbar_wait(&sm->o_free, (ic - 1) & 1);  // last item's O drained
          mbar_wait(&sm->v_full[s], (t / NSV) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(sm->v[s]);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < BN / 16; ++ks) {
              const uint32_t a_tmem = tmem + (uint32_t)(t & 1) * BN + ks * 8;
              mma_ts(tmem + TM_O, a_tmem, smem_desc_sw128(v_addr + ks * 16 * 128, BN * 128, 1024), idesc_o,
                     (jj > 0 || ks > 0) ? 1u : 0u);
            }
            mma_commit(&sm->v_empty[s]);
            mma_commit(&sm->o_done);
            if (jj == NT - 1) mma_commit(&sm->o_final);
          }
          __syncwarp();
        }
      }
      t0 += NT;
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue warps
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t t_lane = tmem + ((uint32_t)(quad * 32) << 16);
    const int64_t qend = rg.q0 + rg.nq;
    int t0 = 0, ic = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++ic) {
      const RangePlan plan = plan_of(w);
      const int u = w / n_qt, NT = plan.count();
      const int64_t n = plan.n0 + r;
      const bool valid = n < qend;
      const Vis rr = visible_set(valid ? n : plan.nlast, C, W, mode, qend);
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < NT; ++j) {
        const int t = t0 + j;
        mbar_wait(&sm->s_full[t & 1], (t >> 1) & 1);
        tc_fence_after();
        const int64_t base = plan.base(j);
        int vlo, vhi, xlo = 0, xhi = 0;
        float bias2 = 0.f;
        if (plan.summary(j)) {
          vlo = 0;
          if (mode == EVA_NONCAUSAL) {
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
        softmax_tile_mx<D>(t_lane + (uint32_t)(t & 1) * BN, t_lane + TM_O, vlo, vhi, xlo, xhi, bias2, scale_log2,
                           m_ref, l, [&] { mbar_wait(&sm->o_done, (t - 1) & 1); });
        mbar_arrive(&sm->p_full[t & 1]);
      }
      // ---- epilogue: O / l straight from TMEM to global (this thread's row), lse
      mbar_wait(&sm->o_final, ic & 1);
      tc_fence_after();
      const float inv_l = l > 0.f ? 1.0f / l : 0.f;
      __nv_bfloat16* orow = O + ((size_t)u * rg.nq + (size_t)(valid ? n - rg.q0 : 0)) * D;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32(t_lane + TM_O + cc * 32, o);
        tmem_wait_ld();
        if (cc == D / 32 - 1) {
          tc_fence_before();
          mbar_arrive(&sm->o_free);
        }
        if (valid) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 w4;
            w4.x = pack_bf16(__uint_as_float(o[8 * g + 0]) * inv_l, __uint_as_float(o[8 * g + 1]) * inv_l);
            w4.y = pack_bf16(__uint_as_float(o[8 * g + 2]) * inv_l, __uint_as_float(o[8 * g + 3]) * inv_l);
            w4.z = pack_bf16(__uint_as_float(o[8 * g + 4]) * inv_l, __uint_as_float(o[8 * g + 5]) * inv_l);
            w4.w = pack_bf16(__uint_as_float(o[8 * g + 6]) * inv_l, __uint_as_float(o[8 * g + 7]) * inv_l);
            *reinterpret_cast<uint4*>(orow + cc * 32 + 8 * g) = w4;
          }
        }
      }
      if (valid && lse) lse[(size_t)u * rg.nq + (size_t)(n - rg.q0)] = (m_ref + __log2f(l)) * 0.69314718055994531f;
      t0 += NT;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ========================================================================== split-softmax kernel
// The tile kernel with 8 softmax warps: warps 2..5 own columns [0,32) of every 64-key S tile,
// warps 6..9 columns [32,64), of the same 128 rows (warp w and w+4 share TMEM lane quadrant
// w%4).  The two halves exchange their partial row max through shared memory (a 64-thread
// named barrier per quadrant, double-buffered), so per-warp softmax work and latency halve.
// Register budget: 2 CTAs x 320 threads per SM (<= 102 registers per thread).
constexpr int NTHREADS2 = 320;

template <int D, int NSTAGE>
struct __align__(1024) Smem2 {
  __nv_bfloat16 q[BM * D];
  __nv_bfloat16 k[NSTAGE][BN * D];
  __nv_bfloat16 v[NSTAGE][BN * D];
  float xmax[2][2][BM];  // [tile parity][half][row]
  float xsum[2][BM];
  uint64_t q_full;
  uint64_t k_full[NSTAGE], v_full[NSTAGE], k_empty[NSTAGE], v_empty[NSTAGE];
  uint64_t s_full[2], p_full[2], o_done, o_final;
  uint32_t tmem_base;
};

template <int D, int NSTAGE>
__global__ void __launch_bounds__(NTHREADS2, 2)
prefill_split_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                     const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mKs,
                     const __grid_constant__ CUtensorMap mVs, const __grid_constant__ CUtensorMap mO,
                     int T, int C, int W, int mode, float scale_log2, float* __restrict__ lse) {
  extern __shared__ uint8_t smem_raw[];
  Smem2<D, NSTAGE>* sm = reinterpret_cast<Smem2<D, NSTAGE>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.y;
  const TilePlan plan(blockIdx.x, T, C, W, mode);
  const int NT = plan.count();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV);
    tma_prefetch(&mKs); tma_prefetch(&mVs); tma_prefetch(&mO);
    mbar_init(&sm->q_full, 1);
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm->k_full[s], 1);
      mbar_init(&sm->v_full[s], 1);
      mbar_init(&sm->k_empty[s], 1);
      mbar_init(&sm->v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm->s_full[b], 1);
      mbar_init(&sm->p_full[b], 256);
    }
    mbar_init(&sm->o_done, 1);
    mbar_init(&sm->o_final, 1);
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

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(&sm->q_full, BM * D * 2);
      for (int kb = 0; kb < D / 64; ++kb)
        tma_load_3d(sm->q + kb * BM * 64, &mQ, &sm->q_full, kb * 64, plan.n0, u);
    }
    __syncwarp();
    auto prefetch_rest = [&] {
      if (elect_one()) {
      for (int j = NSTAGE; j < NT; ++j) {
        const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
        const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
        for (int kb = 0; kb < D / 64; ++kb) {
          tma_prefetch_l2_3d(mk, kb * 64, plan.base(j), u);
          tma_prefetch_l2_3d(mv, kb * 64, plan.base(j), u);
        }
      }
      }
      __syncwarp();
    };
    auto load_k = [&](int j) {
      const int s = j % NSTAGE;
      if (j >= NSTAGE) mbar_wait(&sm->k_empty[s], ((j / NSTAGE) - 1) & 1);
      const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm->k_full[s], BN * D * 2);
        for (int kb = 0; kb < D / 64; ++kb)
          tma_load_3d(sm->k[s] + kb * BN * 64, mk, &sm->k_full[s], kb * 64, plan.base(j), u);
      }
      __syncwarp();
    };
    auto load_v = [&](int j) {
      const int s = j % NSTAGE;
      if (j >= NSTAGE) mbar_wait(&sm->v_empty[s], ((j / NSTAGE) - 1) & 1);
      const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
      if (elect_one()) {
        mbar_arrive_expect_tx(&sm->v_full[s], BN * D * 2);
        for (int kb = 0; kb < D / 64; ++kb)
          tma_load_3d(sm->v[s] + kb * BN * 64, mv, &sm->v_full[s], kb * 64, plan.base(j), u);
      }
      __syncwarp();
    };
    load_k(0);
    if (NT > 1) load_k(1);
    load_v(0);
    prefetch_rest();  // after the first tiles: they are on the critical path
    for (int j = 1; j < NT; ++j) {
      if (j + 1 < NT) load_k(j + 1);
      load_v(j);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(BM, BN, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BM, D, true);
    const uint32_t q_addr = smem_u32(sm->q);
    mbar_wait(&sm->q_full, 0);
    for (int j = 0; j <= NT; ++j) {
      if (j < NT) {
        const int s = j % NSTAGE;
        mbar_wait(&sm->k_full[s], (j / NSTAGE) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sm->k[s]);
        const uint32_t d_tmem = tmem + (uint32_t)(j & 1) * BN;
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
            mma_ss(d_tmem, smem_desc_sw128(q_addr + kb * (BM * 128) + off, 16, 1024),
                   smem_desc_sw128(k_addr + kb * (BN * 128) + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
          }
          mma_commit(&sm->s_full[j & 1]);
          mma_commit(&sm->k_empty[s]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int jj = j - 1, s = jj % NSTAGE;
        mbar_wait(&sm->p_full[jj & 1], (jj >> 1) & 1);
        mbar_wait(&sm->v_full[s], (jj / NSTAGE) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sm->v[s]);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < BN / 16; ++ks)
            mma_ts(tmem + TM_O, tmem + (uint32_t)(jj & 1) * BN + ks * 8,
                   smem_desc_sw128(v_addr + ks * 16 * 128, BN * 128, 1024), idesc_o, (jj > 0 || ks > 0) ? 1u : 0u);
          mma_commit(&sm->v_empty[s]);
          mma_commit(&sm->o_done);
          if (jj == NT - 1) mma_commit(&sm->o_final);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ softmax halves + epilogue
    const int h = (warp - 2) >> 2;          // column half: 0 -> [0,32), 1 -> [32,64)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int n = plan.n0 + r;
    const bool valid = n < T;
    const Range rr = mask_range(valid ? n : plan.nlast, C, W, mode);
    const uint32_t t_lane = tmem + ((uint32_t)(quad * 32) << 16);
    constexpr int DH = D / 2;               // O columns owned by this half
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < NT; ++j) {
      const int b = j & 1;
      mbar_wait(&sm->s_full[b], (j >> 1) & 1);
      tc_fence_after();
      const int base = plan.base(j) + 32 * h;
      int vlo, vhi;
      if (plan.summary(j)) {
        vlo = 0;
        vhi = (int)min((int64_t)32, rr.nsum - base);
      } else {
        vlo = (int)max((int64_t)0, rr.lo - base);
        vhi = min(32, n - base + 1);
      }
      if (!valid) vhi = vlo;
      uint32_t sr[32];
      tmem_ld32(t_lane + (uint32_t)b * BN + 32 * h, sr);
      tmem_wait_ld();
      if (!__all_sync(0xffffffffu, vlo <= 0 && vhi >= 32)) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < vlo || c >= vhi) sr[c] = 0xff800000u;
      }
      float pm[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pm[i] = __uint_as_float(sr[i]);
#pragma unroll
      for (int c = 4; c < 32; ++c) pm[c & 3] = fmaxf(pm[c & 3], __uint_as_float(sr[c]));
      const float pmx = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3]));
      sm->xmax[b][h][r] = pmx;
      named_bar_sync(2 + quad, 64);
      const float mx = fmaxf(pmx, sm->xmax[b][1 - h][r]) * scale_log2;
      const bool grow = mx > m_ref + 8.0f;
      if (__any_sync(0xffffffffu, grow && m_ref != -INFINITY)) {
        const float f = (grow && m_ref != -INFINITY) ? ex2(m_ref - mx) : 1.0f;
        mbar_wait(&sm->o_done, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < DH / 32; ++cc) {
          uint32_t o[32];
          tmem_ld32(t_lane + TM_O + h * DH + cc * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
          tmem_st32(t_lane + TM_O + h * DH + cc * 32, o);
        }
        tmem_wait_st();
        l *= f;
      }
      if (grow) m_ref = mx;
      const float neg = m_ref == -INFINITY ? 0.f : -m_ref;
      uint32_t pk[16];
      float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float p0 = ex2(fmaf(__uint_as_float(sr[2 * c]), scale_log2, neg));
        const float p1 = ex2(fmaf(__uint_as_float(sr[2 * c + 1]), scale_log2, neg));
        ls[(2 * c) & 3] += p0;
        ls[(2 * c + 1) & 3] += p1;
        pk[c] = pack_bf16(p0, p1);
      }
      l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      tmem_st16(t_lane + (uint32_t)b * BN + 16 * h, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&sm->p_full[b]);
    }
    // ------------------------------------------------------------ epilogue
    sm->xsum[h][r] = l;
    mbar_wait(&sm->o_final, 0);
    tc_fence_after();
    named_bar_sync(2 + quad, 64);
    const float lt = sm->xsum[0][r] + sm->xsum[1][r];
    const float inv_l = lt > 0.f ? 1.0f / lt : 0.f;
    uint8_t* qs = reinterpret_cast<uint8_t*>(sm->q);
#pragma unroll
    for (int cc = 0; cc < DH / 32; ++cc) {
      uint32_t o[32];
      const int col = h * DH + cc * 32;
      tmem_ld32(t_lane + TM_O + col, o);
      tmem_wait_ld();
      const int kb = col / 64, c16_0 = (col % 64) / 8;
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
    if (h == 0 && valid && lse) lse[(size_t)u * T + n] = (m_ref + __log2f(lt)) * 0.69314718055994531f;
    fence_proxy_async_smem();
    named_bar_sync(1, 256);
    if (warp == 2 && lane == 0) {
      for (int kb = 0; kb < D / 64; ++kb) tma_store_3d(&mO, sm->q + kb * BM * 64, kb * 64, plan.n0, u);
      tma_store_commit();
      tma_store_wait_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ========================================================================== wide-tile kernel
// One 128-query tile per CTA (two CTAs per SM) walking 128-key tiles: the S MMA is
// M=128 x N=128 (full tensor rate; N=64 SS MMAs are shared-memory bound at 48 instead of
// 32 cycles per K-step).  TMEM (256 columns): S/P [0,128) single-buffered, O [128,128+d).
// Per tile the MMA warp issues PV(j-1) then S(j), so when softmax sees S(j) complete,
// PV(j-1) has completed too and O may be rescaled without another barrier.  K and V have
// separate slot rings (NSK, NSV) released by the S and the PV MMA respectively.
constexpr int BNW = 128;

struct WidePlan {
  int n0, nlast, n_st, n_lt, lo0;
  __device__ WidePlan(int qt, int T, int C, int W, int mode) {
    n0 = qt * BM;
    nlast = min(n0 + BM - 1, T - 1);
    const Range rf = mask_range(n0, C, W, mode), rl = mask_range(nlast, C, W, mode);
    n_st = (int)((rl.nsum + BNW - 1) / BNW);
    lo0 = (int)rf.lo;
    n_lt = (nlast - lo0 + 1 + BNW - 1) / BNW;
  }
  __device__ int count() const { return n_st + n_lt; }
  __device__ bool summary(int j) const { return j < n_st; }
  __device__ int base(int j) const { return j < n_st ? j * BNW : lo0 + (j - n_st) * BNW; }
};

template <int D, int NSK, int NSV>
struct __align__(1024) SmemWide {
  __nv_bfloat16 q[BM * D];           // D/64 sub-tiles [128][64]
  __nv_bfloat16 k[NSK][BNW * D];     // D/64 sub-tiles [128][64]
  __nv_bfloat16 v[NSV][BNW * D];
  uint64_t q_full, k_full[NSK], k_empty[NSK], v_full[NSV], v_empty[NSV];
  uint64_t s_full, p_full, o_final;
  uint32_t tmem_base;
};

// Softmax step on a 128-column S tile (see softmax_tile): pass 1 loads all 128 columns and
// finds the row max, pass 2 writes P (bf16 pairs) in place and stores it to TMEM [0,64).
// The previous PV has completed whenever this runs (issue order), so no wait is needed
// before rescaling O.
template <int D>
__device__ __forceinline__ void softmax_tile128(uint32_t s_addr, uint32_t o_addr, int vlo, int vhi,
                                                float scale_log2, float& m_ref, float& l) {
  // pass 1: row max over the 128 columns, 32 at a time (keeps register use low)
  const bool full = __all_sync(0xffffffffu, vlo <= 0 && vhi >= 128);
  float pm[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) pm[i] = -INFINITY;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t sr[32];
    tmem_ld32(s_addr + 32 * q, sr);
    tmem_wait_ld();
    if (!full) {
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (32 * q + c < vlo || 32 * q + c >= vhi) sr[c] = 0xff800000u;
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) pm[c & 7] = fmaxf(pm[c & 7], __uint_as_float(sr[c]));
  }
  float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
  mx *= scale_log2;
  const bool grow = mx > m_ref + 8.0f;
  if (__any_sync(0xffffffffu, grow && m_ref != -INFINITY)) {
    const float f = (grow && m_ref != -INFINITY) ? ex2(m_ref - mx) : 1.0f;
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t o[32];
      tmem_ld32(o_addr + cc * 32, o);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
      tmem_st32(o_addr + cc * 32, o);
    }
    tmem_wait_st();
    l *= f;
  }
  if (grow) m_ref = mx;
  const float neg = m_ref == -INFINITY ? 0.f : -m_ref;
  // pass 2: P = exp2(s*scale - m) as bf16 pairs; chunk q (S columns 32q..32q+31) lands in
  // P columns 16q..16q+15, which only overwrite S columns already consumed
  float ls[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) ls[i] = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t sr[32];
    tmem_ld32(s_addr + 32 * q, sr);
    tmem_wait_ld();
    if (!full) {
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (32 * q + c < vlo || 32 * q + c >= vhi) sr[c] = 0xff800000u;
    }
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float p0 = ex2(fmaf(__uint_as_float(sr[2 * c]), scale_log2, neg));
      const float p1 = ex2(fmaf(__uint_as_float(sr[2 * c + 1]), scale_log2, neg));
      ls[(2 * c) & 7] += p0;
      ls[(2 * c + 1) & 7] += p1;
      pk[c] = pack_bf16(p0, p1);
    }
    tmem_st16(s_addr + 16 * q, pk);
  }
  l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
  tmem_wait_st();
  tc_fence_before();
}

template <int D, int NSK, int NSV>
__global__ void __launch_bounds__(NTHREADS, 2)
prefill_wide_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                    const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mKs,
                    const __grid_constant__ CUtensorMap mVs, const __grid_constant__ CUtensorMap mO,
                    int T, int C, int W, int mode, float scale_log2, float* __restrict__ lse) {
  extern __shared__ uint8_t smem_raw[];
  SmemWide<D, NSK, NSV>* sm = reinterpret_cast<SmemWide<D, NSK, NSV>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.y;
  const WidePlan plan(blockIdx.x, T, C, W, mode);
  const int NT = plan.count();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV);
    tma_prefetch(&mKs); tma_prefetch(&mVs); tma_prefetch(&mO);
    mbar_init(&sm->q_full, 1);
    for (int s = 0; s < NSK; ++s) { mbar_init(&sm->k_full[s], 1); mbar_init(&sm->k_empty[s], 1); }
    for (int s = 0; s < NSV; ++s) { mbar_init(&sm->v_full[s], 1); mbar_init(&sm->v_empty[s], 1); }
    mbar_init(&sm->s_full, 1);
    mbar_init(&sm->p_full, 128);
    mbar_init(&sm->o_final, 1);
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

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(&sm->q_full, BM * D * 2);
      for (int kb = 0; kb < D / 64; ++kb)
        tma_load_3d(sm->q + kb * BM * 64, &mQ, &sm->q_full, kb * 64, plan.n0, u);
      for (int j = 1; j < NT; ++j) {  // later tiles: warm L2 (the rings hold only NSK/NSV)
        const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
        const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
        for (int kb = 0; kb < D / 64; ++kb) {
          tma_prefetch_l2_3d(mk, kb * 64, plan.base(j), u);
          tma_prefetch_l2_3d(mv, kb * 64, plan.base(j), u);
        }
      }
    }
    __syncwarp();
    auto load = [&](bool is_k, int j) {
      const int s = is_k ? j % NSK : j % NSV;
      const int ns = is_k ? NSK : NSV;
      uint64_t* empty = is_k ? &sm->k_empty[s] : &sm->v_empty[s];
      uint64_t* full = is_k ? &sm->k_full[s] : &sm->v_full[s];
      __nv_bfloat16* dst = is_k ? sm->k[s] : sm->v[s];
      if (j >= ns) mbar_wait(empty, ((j / ns) - 1) & 1);
      const CUtensorMap* m = plan.summary(j) ? (is_k ? &mKs : &mVs) : (is_k ? &mK : &mV);
      if (elect_one()) {
        mbar_arrive_expect_tx(full, BNW * D * 2);
        for (int kb = 0; kb < D / 64; ++kb) tma_load_3d(dst + kb * BNW * 64, m, full, kb * 64, plan.base(j), u);
      }
      __syncwarp();
    };
    // K(j) is consumed by S(j), V(j) by PV(j) one softmax later: K runs one tile ahead.
    load(true, 0);
    for (int j = 0; j < NT; ++j) {
      load(false, j);
      if (j + 1 < NT) load(true, j + 1);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(BM, BNW, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BM, D, true);
    const uint32_t q_addr = smem_u32(sm->q);
    mbar_wait(&sm->q_full, 0);
    for (int j = 0; j <= NT; ++j) {
      if (j >= 1) {  // PV(j-1)
        const int jj = j - 1, s = jj % NSV;
        mbar_wait(&sm->p_full, jj & 1);
        mbar_wait(&sm->v_full[s], (jj / NSV) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sm->v[s]);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < BNW / 16; ++ks)
            mma_ts(tmem + TM_O, tmem + ks * 8, smem_desc_sw128(v_addr + ks * 16 * 128, BNW * 128, 1024),
                   idesc_o, (jj > 0 || ks > 0) ? 1u : 0u);
          mma_commit(&sm->v_empty[s]);
          if (jj == NT - 1) mma_commit(&sm->o_final);
        }
        __syncwarp();
      }
      if (j < NT) {  // S(j)
        const int s = j % NSK;
        mbar_wait(&sm->k_full[s], (j / NSK) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sm->k[s]);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
            mma_ss(tmem, smem_desc_sw128(q_addr + kb * (BM * 128) + off, 16, 1024),
                   smem_desc_sw128(k_addr + kb * (BNW * 128) + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
          }
          mma_commit(&sm->s_full);
          mma_commit(&sm->k_empty[s]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps + epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int n = plan.n0 + r;
    const bool valid = n < T;
    const Range rr = mask_range(valid ? n : plan.nlast, C, W, mode);
    const uint32_t t_lane = tmem + ((uint32_t)(quad * 32) << 16);
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < NT; ++j) {
      mbar_wait(&sm->s_full, j & 1);
      tc_fence_after();
      const int base = plan.base(j);
      int vlo, vhi;
      if (plan.summary(j)) {
        vlo = 0;
        vhi = (int)min((int64_t)BNW, rr.nsum - base);
      } else {
        vlo = (int)max((int64_t)0, rr.lo - base);
        vhi = min(BNW, n - base + 1);
      }
      if (!valid) vhi = vlo;
      softmax_tile128<D>(t_lane, t_lane + TM_O, vlo, vhi, scale_log2, m_ref, l);
      mbar_arrive(&sm->p_full);
    }
    mbar_wait(&sm->o_final, 0);
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
    if (valid && lse) lse[(size_t)u * T + n] = (m_ref + __log2f(l)) * 0.69314718055994531f;
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (warp == 2 && lane == 0) {
      for (int kb = 0; kb < D / 64; ++kb) tma_store_3d(&mO, sm->q + kb * BM * 64, kb * 64, plan.n0, u);
      tma_store_commit();
      tma_store_wait_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ========================================================================== pair kernel
// Persistent variant for large problems: a CTA owns one SM and loops over work items
// (unit, pair of adjacent 128-query tiles).  The two Q tiles share one K/V stream (the
// union of their tile lists, loaded once through an NS-deep TMA ring), each Q tile has
// its own softmax warpgroup and its own TMEM half (S double buffer + O):
//   warp 0      TMA producer (Q tiles of the next item prefetched as soon as the last
//               S MMA of the current item has consumed the old ones)
//   warp 1      MMA issuer: per union tile j: S_t(j) for each Q tile t that needs j,
//               then PV_t(j-1); stage released after the last PV that reads it
//   warps 2-5   softmax + epilogue of Q tile 0;   warps 6-9   the same for Q tile 1
// Epilogue: O / l straight from registers to global (rows are contiguous 2d-byte runs).
constexpr int PAIR_THREADS = 352;  // + warp 10: Q-tile loader
constexpr uint32_t PAIR_TMEM_COLS = 512;

// Debug timeline (eva_debug_trace_prefill): CTA 0 records (clock64 << 24 | code) events in
// per-role shared-memory logs (no atomics: role r appends to its own slice), copied to
// global memory at exit.  code = kind << 20 | t << 16 | j.  kinds: 1 producer issued tile j,
// 2 MMA issued S_t(j), 3 MMA issued PV_t(j), 4 softmax t got S(j), 5 softmax t released
// P(j), 6 epilogue t done, 7 producer slot free for tile j, 8 MMA got k_full(j),
// 9 MMA got p_full_t(j).
__device__ unsigned long long* g_trace = nullptr;
__device__ int g_trace_n = 0;
__device__ int g_trace_cap = 0;
constexpr int TRACE_ROLES = 4, TRACE_PER_ROLE = 384;
struct TraceLog {
  unsigned long long ev[TRACE_ROLES][TRACE_PER_ROLE];
  int n[TRACE_ROLES];
};
template <bool TRACE>
__device__ __forceinline__ void trace(TraceLog* log, int role, int kind, int t, int j) {
  if constexpr (TRACE) {
    if (blockIdx.x == 0) {
      const int i = log->n[role];
      if (i < TRACE_PER_ROLE)
        log->ev[role][i] = ((unsigned long long)clock64() << 24) | ((unsigned)kind << 20) |
                           ((unsigned)t << 16) | ((unsigned)j & 0xffff);
      log->n[role] = i + 1;
    }
  }
}
template <bool TRACE>
__device__ __forceinline__ void trace_flush(TraceLog* log) {
  if constexpr (TRACE) {
    if (blockIdx.x == 0 && g_trace) {
      for (int r = 0; r < TRACE_ROLES; ++r) {
        const int n = min(log->n[r], TRACE_PER_ROLE);
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          const int k = r * TRACE_PER_ROLE + i;
          if (k < g_trace_cap) g_trace[k] = log->ev[r][i];
        }
      }
    }
  }
}

template <int D, int NS>
struct __align__(1024) SmemPair {
  __nv_bfloat16 q[2][BM * D];
  __nv_bfloat16 k[NS][BN * D];
  __nv_bfloat16 v[NS][BN * D];
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[NS], v_full[NS], kv_empty[NS];
  uint64_t s_full[2][2], p_full[2][2], o_done[2], o_final[2], o_empty[2];
  uint32_t tmem_base;
};

// Tile plan of one work item (two adjacent Q tiles).  Scalar fields only (selected with
// t ? x1 : x0) so that nothing is indexed dynamically and the plan stays in registers.
struct PairPlan {
  int n0, n_st, n_lt, lo0;
  int nlast0, nlast1, lof0, lof1, nsl0, nsl1;
  __device__ PairPlan(int pair, int T, int C, int W, int mode) {
    n0 = pair * 2 * BM;
    const int a1 = n0 + BM;
    nlast0 = min(n0 + BM - 1, T - 1);
    lof0 = (int)mask_range(n0, C, W, mode).lo;
    nsl0 = (int)mask_range(nlast0, C, W, mode).nsum;
    if (a1 < T) {
      nlast1 = min(a1 + BM - 1, T - 1);
      lof1 = (int)mask_range(a1, C, W, mode).lo;
      nsl1 = (int)mask_range(nlast1, C, W, mode).nsum;
    } else {
      nlast1 = -1;
      lof1 = 0;
      nsl1 = 0;
    }
    const int nl = nlast1 >= 0 ? nlast1 : nlast0;
    const int ns = nlast1 >= 0 ? nsl1 : nsl0;
    n_st = (ns + BN - 1) / BN;
    lo0 = lof0;
    n_lt = (nl - lo0 + 1 + BN - 1) / BN;
  }
  __device__ int nlast(int t) const { return t ? nlast1 : nlast0; }
  __device__ bool active(int t) const { return nlast(t) >= 0; }
  __device__ int count() const { return n_st + n_lt; }
  __device__ bool summary(int j) const { return j < n_st; }
  __device__ int base(int j) const { return j < n_st ? j * BN : lo0 + (j - n_st) * BN; }
  __device__ bool need(int t, int j) const {
    const int nl = t ? nlast1 : nlast0;
    if (nl < 0) return false;
    const int b = base(j);
    if (j < n_st) return b < (t ? nsl1 : nsl0);
    return b <= nl && b + BN - 1 >= (t ? lof1 : lof0);
  }
  __device__ int last_need(int t) const {
    // local tiles are needed on a contiguous range ending at the tile containing nlast(t);
    // if the Q tile has no local tile (impossible: n is in E(n)) fall back to a scan.
    const int nl = t ? nlast1 : nlast0;
    if (nl < 0) return -1;
    return n_st + (nl - lo0) / BN;
  }
};

template <int D, int NS, bool TRACE>
__global__ void __launch_bounds__(PAIR_THREADS, 1)
prefill_pair_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                    const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mKs,
                    const __grid_constant__ CUtensorMap mVs, int BH, int T, int C, int W, int mode,
                    float scale_log2, __nv_bfloat16* __restrict__ O, float* __restrict__ lse) {
  extern __shared__ uint8_t smem_raw[];
  SmemPair<D, NS>* sm = reinterpret_cast<SmemPair<D, NS>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  TraceLog* tlog = reinterpret_cast<TraceLog*>(sm + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ppu = (T + 2 * BM - 1) / (2 * BM);
  if (TRACE && threadIdx.x < TRACE_ROLES) tlog->n[threadIdx.x] = 0;
  const int n_items = BH * ppu;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV); tma_prefetch(&mKs); tma_prefetch(&mVs);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm->q_full[t], 1);
      mbar_init(&sm->q_empty[t], 1);
      mbar_init(&sm->o_done[t], 1);
      mbar_init(&sm->o_final[t], 1);
      mbar_init(&sm->o_empty[t], 128);
      for (int b = 0; b < 2; ++b) {
        mbar_init(&sm->s_full[t][b], 1);
        mbar_init(&sm->p_full[t][b], 128);
      }
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm->k_full[s], 1);
      mbar_init(&sm->v_full[s], 1);
      mbar_init(&sm->kv_empty[s], 2);  // one release per Q tile
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(&sm->tmem_base, PAIR_TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (whole warp)
    uint32_t kv = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const bool tr = TRACE && item >= (int)(blockIdx.x + 3 * gridDim.x);  // steady-state window
      const int u = item / ppu;
      const PairPlan plan(item % ppu, T, C, W, mode);
      const int NT = plan.count();
      for (int j = 0; j < NT; ++j, ++kv) {
        const int s = kv % NS;
        if (kv >= (uint32_t)NS) mbar_wait(&sm->kv_empty[s], ((kv / NS) - 1) & 1);
        if (tr && lane == 0) trace<TRACE>(tlog, 0, 7, 0, kv);
        const bool summ = plan.summary(j);
        const int row = plan.base(j);
        const CUtensorMap* mk = summ ? &mKs : &mK;
        const CUtensorMap* mv = summ ? &mVs : &mV;
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm->k_full[s], BN * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->k[s] + kb * BN * 64, mk, &sm->k_full[s], kb * 64, row, u);
          mbar_arrive_expect_tx(&sm->v_full[s], BN * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->v[s] + kb * BN * 64, mv, &sm->v_full[s], kb * 64, row, u);
        }
        __syncwarp();
        if (tr && lane == 0) trace<TRACE>(tlog, 0, 1, 0, kv);
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ Q-tile loader (whole warp)
    // Separate from the K/V producer so the ring keeps streaming the next item's tiles
    // while this warp waits for the current item's last S MMA to release a Q buffer.
    int qcnt0 = 0, qcnt1 = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int u = item / ppu;
      const PairPlan plan(item % ppu, T, C, W, mode);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (!plan.active(t)) continue;
        int& qc = t ? qcnt1 : qcnt0;
        if (qc > 0) mbar_wait(&sm->q_empty[t], (qc - 1) & 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm->q_full[t], BM * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->q[t] + kb * BM * 64, &mQ, &sm->q_full[t], kb * 64, plan.n0 + t * BM, u);
        }
        __syncwarp();
        ++qc;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (whole warp)
    // Ping-pong order per Q tile t (FA4-style): PV_t(i) is followed immediately by
    // S_t(next tile of t), so while softmax warpgroup 0 works the tensor core runs Q tile 1
    // and vice versa.  Each union tile's ring slot is released by two tcgen05.commit
    // arrivals (kv_empty count 2): one per Q tile, after its PV (or, if that Q tile skips
    // the tile, as soon as its cursor passes it).  All state stays in scalar registers.
    constexpr uint32_t idesc_s = idesc_bf16_f32(BM, BN, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BM, D, true);
    const uint32_t q0_addr = smem_u32(sm->q[0]), q1_addr = smem_u32(sm->q[1]);
    uint32_t kv = 0;  // ring index of the item's union tile 0
    uint32_t cS0 = 0, cS1 = 0, cP0 = 0, cP1 = 0, icnt0 = 0, icnt1 = 0;
#define EVA_ISSUE_S(T_, J_, CS_)                                                                        \
  do {                                                                                                 \
    const uint32_t kk = kv + (uint32_t)(J_);                                                           \
    mbar_wait(&sm->k_full[kk % NS], (kk / NS) & 1);                                                    \
    tc_fence_after();                                                                                  \
    const uint32_t k_addr = smem_u32(sm->k[kk % NS]);                                                  \
    if (elect_one()) {                                                                                 \
      const uint32_t d_tmem = tmem + (T_) * 256u + ((CS_) & 1) * BN;                                   \
      const uint32_t qa = (T_) ? q1_addr : q0_addr;                                                    \
      _Pragma("unroll") for (int ks = 0; ks < D / 16; ++ks) {                                          \
        const uint32_t kb = ks >> 2, off = (ks & 3) * 32;                                              \
        mma_ss(d_tmem, smem_desc_sw128(qa + kb * (BM * 128) + off, 16, 1024),                          \
               smem_desc_sw128(k_addr + kb * (BN * 128) + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);  \
      }                                                                                                \
      mma_commit(&sm->s_full[T_][(CS_) & 1]);                                                          \
      if ((J_) == ((T_) ? last1 : last0)) mma_commit(&sm->q_empty[T_]);                                \
    }                                                                                                  \
    __syncwarp();                                                                                      \
    ++(CS_);                                                                                           \
  } while (0)
#define EVA_ISSUE_PV(T_, J_, CP_, FIRST_, ICNT_)                                                       \
  do {                                                                                                 \
    const uint32_t kk = kv + (uint32_t)(J_);                                                           \
    mbar_wait(&sm->p_full[T_][(CP_) & 1], ((CP_) >> 1) & 1);                                           \
    if ((FIRST_) && (ICNT_) > 0) mbar_wait(&sm->o_empty[T_], ((ICNT_) - 1) & 1);                       \
    mbar_wait(&sm->v_full[kk % NS], (kk / NS) & 1);                                                    \
    tc_fence_after();                                                                                  \
    const uint32_t v_addr = smem_u32(sm->v[kk % NS]);                                                  \
    if (elect_one()) {                                                                                 \
      const uint32_t tb = tmem + (T_) * 256u;                                                          \
      _Pragma("unroll") for (int ks = 0; ks < BN / 16; ++ks)                                           \
        mma_ts(tb + TM_O, tb + ((CP_) & 1) * BN + ks * 8,                                              \
               smem_desc_sw128(v_addr + ks * 16 * 128, BN * 128, 1024), idesc_o,                       \
               (!(FIRST_) || ks > 0) ? 1u : 0u);                                                       \
      mma_commit(&sm->o_done[T_]);                                                                     \
      if ((J_) == ((T_) ? last1 : last0)) mma_commit(&sm->o_final[T_]);                                \
      mma_commit(&sm->kv_empty[kk % NS]);                                                              \
      if (!plan.need(1 - (T_), (J_))) mma_commit(&sm->kv_empty[kk % NS]); /* other tile's share */     \
    }                                                                                                  \
    __syncwarp();                                                                                      \
    (FIRST_) = false;                                                                                  \
    ++(CP_);                                                                                           \
  } while (0)
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const bool tr = TRACE && item >= (int)(blockIdx.x + 3 * gridDim.x);
      const PairPlan plan(item % ppu, T, C, W, mode);
      const int NT = plan.count();
      const bool act1 = plan.active(1);
      const int last0 = plan.last_need(0), last1 = plan.last_need(1);
      // next needed union tile of Q tile t at or after j (NT if none)
      auto next_need = [&](int t, int j) {
        while (j < NT && !plan.need(t, j)) ++j;
        return j;
      };
      bool first0 = true, first1 = true;
      mbar_wait(&sm->q_full[0], icnt0 & 1);
      if (act1) mbar_wait(&sm->q_full[1], icnt1 & 1);
      // Event loop: per Q tile, S runs at most one tile ahead of PV (double-buffered S/P);
      // whichever Q tile has its operands ready is served first (non-blocking probes), so
      // the two softmax warpgroups are never lock-stepped through this single issuer.
      int s0 = next_need(0, 0), s1 = act1 ? next_need(1, 0) : NT;   // next S tile
      int p0 = s0, p1 = s1;                                          // next PV tile
      int ahead0 = 0, ahead1 = 0;                                    // S issued - PV issued
      while (p0 < NT || p1 < NT) {
        bool progress = false;
        // ---- Q tile 0
        if (s0 < NT && ahead0 < 2) {
          const uint32_t kk = kv + (uint32_t)s0;
          if (mbar_test(&sm->k_full[kk % NS], (kk / NS) & 1)) {
            EVA_ISSUE_S(0, s0, cS0);
            s0 = next_need(0, s0 + 1);
            ++ahead0;
            progress = true;
          }
        }
        if (p0 < NT && ahead0 > 0 && mbar_test(&sm->p_full[0][cP0 & 1], (cP0 >> 1) & 1)) {
          EVA_ISSUE_PV(0, p0, cP0, first0, icnt0);
          if (tr && lane == 0) trace<TRACE>(tlog, 1, 3, 0, kv + p0);
          p0 = next_need(0, p0 + 1);
          --ahead0;
          progress = true;
        }
        // ---- Q tile 1
        if (s1 < NT && ahead1 < 2) {
          const uint32_t kk = kv + (uint32_t)s1;
          if (mbar_test(&sm->k_full[kk % NS], (kk / NS) & 1)) {
            EVA_ISSUE_S(1, s1, cS1);
            s1 = next_need(1, s1 + 1);
            ++ahead1;
            progress = true;
          }
        }
        if (p1 < NT && ahead1 > 0 && mbar_test(&sm->p_full[1][cP1 & 1], (cP1 >> 1) & 1)) {
          EVA_ISSUE_PV(1, p1, cP1, first1, icnt1);
          if (tr && lane == 0) trace<TRACE>(tlog, 1, 3, 1, kv + p1);
          p1 = next_need(1, p1 + 1);
          --ahead1;
          progress = true;
        }
        if (!progress) __nanosleep(32);
      }
      kv += (uint32_t)NT;
      ++icnt0;
      if (act1) ++icnt1;
    }
#undef EVA_ISSUE_S
#undef EVA_ISSUE_PV
  } else {
    // ------------------------------------------------------------ softmax warpgroups
    const int t = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t t_lane = tmem + (uint32_t)t * 256 + ((uint32_t)(quad * 32) << 16);
    int cS = 0, icnt = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const bool tr = TRACE && item >= (int)(blockIdx.x + 3 * gridDim.x);
      const int u = item / ppu;
      const PairPlan plan(item % ppu, T, C, W, mode);
      if (!plan.active(t)) continue;
      const int n = plan.n0 + t * BM + r;
      const bool valid = n <= plan.nlast(t);
      const Range rr = mask_range(valid ? n : plan.nlast(t), C, W, mode);
      const int NT = plan.count();
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < NT; ++j) {
        if (!plan.need(t, j)) continue;
        const int b = cS & 1;
        mbar_wait(&sm->s_full[t][b], (cS >> 1) & 1);
        if (tr && r == 0) trace<TRACE>(tlog, 2 + t, 4, t, cS);
        tc_fence_after();
        const int base = plan.base(j);
        int vlo, vhi;
        if (plan.summary(j)) {
          vlo = 0;
          vhi = (int)min((int64_t)BN, rr.nsum - base);
        } else {
          vlo = (int)max((int64_t)0, rr.lo - base);
          vhi = min(BN, n - base + 1);
        }
        if (!valid) vhi = vlo;
        softmax_tile<D>(t_lane + (uint32_t)b * BN, t_lane + TM_O, vlo, vhi, scale_log2, m_ref, l,
                        [&] { mbar_wait(&sm->o_done[t], (cS - 1) & 1); });
        mbar_arrive(&sm->p_full[t][b]);
        if (tr && r == 0) trace<TRACE>(tlog, 2 + t, 5, t, cS);
        ++cS;
      }
      // ---------------------------------------------------------- epilogue
      mbar_wait(&sm->o_final[t], icnt & 1);
      tc_fence_after();
      const float inv_l = l > 0.f ? 1.0f / l : 0.f;
      uint32_t ob[D / 2];
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32(t_lane + TM_O + cc * 32, o);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i)
          ob[cc * 16 + i] = pack_bf16(__uint_as_float(o[2 * i]) * inv_l, __uint_as_float(o[2 * i + 1]) * inv_l);
      }
      tc_fence_before();
      mbar_arrive(&sm->o_empty[t]);
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(O + ((size_t)u * T + n) * D);
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
          dst[i] = make_uint4(ob[4 * i], ob[4 * i + 1], ob[4 * i + 2], ob[4 * i + 3]);
        if (lse) lse[(size_t)u * T + n] = (m_ref + __log2f(l)) * 0.69314718055994531f;
      }
      if (tr && r == 0) trace<TRACE>(tlog, 2 + t, 6, t, icnt);
      ++icnt;
    }
  }
  tc_fence_before();
  __syncthreads();
  trace_flush<TRACE>(tlog);
  if (warp == 1) tmem_dealloc(tmem, PAIR_TMEM_COLS);
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

// Softmax exponential split of the tile kernel: -1 = all MUFU.EX2 (softmax_tile), k >= 0 =
// softmax_tile2 with k of every 8 column pairs on the FMA pipe.  EVA_SOFTMAX_EMU overrides
// the default (tuning knob, read once).
int softmax_emu() {
  static const int v = [] {
    const char* e = getenv("EVA_SOFTMAX_EMU");
    return e ? atoi(e) : -1;
  }();
  return v;
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

template <int D, int NSTAGE, bool TRACE = false, int SMX = -1>
cudaError_t launch_t(const eva_config& cfg, const PrefillRange& rg, const void* Q, const void* K,
                     const void* V, const void* Ksum, const void* Vsum, void* O, float* lse,
                     cudaStream_t s, bool overlap = false) {
  if constexpr (!TRACE && SMX == -1) {
    switch (softmax_emu()) {
      case 0: return launch_t<D, NSTAGE, false, 0>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
      case 1: return launch_t<D, NSTAGE, false, 1>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
      case 2: return launch_t<D, NSTAGE, false, 2>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
      case 3: return launch_t<D, NSTAGE, false, 3>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
      default: break;
    }
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
  const size_t smem = sizeof(Smem<D, NSTAGE>) + Smem<D, NSTAGE>::PAD;
  {
    cudaError_t e = set_smem_attr((const void*)prefill_sm100_kernel<D, NSTAGE, TRACE, SMX>, smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((rg.nq + BM - 1) / BM, BH);
  const float scale_log2 = cfg.scale * 1.4426950408889634f;
  cudaError_t e = launch_pdl(prefill_sm100_kernel<D, NSTAGE, TRACE, SMX>, grid, dim3(NTHREADS), smem, s, mQ, mK, mV,
                             mKs, mVs, mO, rg, cfg.chunk, cfg.window, cfg.mode, scale_log2,
                             cfg.summary_bias * 1.4426950408889634f, lse, overlap ? 1 : 0, tile_sum_first());
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

template <int D, int NSTAGE>
cudaError_t launch_persist(const eva_config& cfg, const PrefillRange& rg, const void* Q, const void* K,
                           const void* V, const void* Ksum, const void* Vsum, void* O, float* lse,
                           cudaStream_t s) {
  const int BH = cfg.bh_count, nC = rg.nsl;
  if (rg.nq == 0) return cudaSuccess;
  CUtensorMap mQ, mK, mV, mKs, mVs;
  bool ok = make_map(&mQ, Q, BH, rg.nq, D, BM) && make_map(&mK, K, BH, rg.nkv, D, BN) &&
            make_map(&mV, V, BH, rg.nkv, D, BN);
  if (nC > 0) {
    ok = ok && make_map(&mKs, Ksum, BH, nC, D, BN) && make_map(&mVs, Vsum, BH, nC, D, BN);
  } else {
    mKs = mK;
    mVs = mV;
  }
  if (!ok) return cudaErrorInvalidValue;
  const size_t smem = sizeof(SmemP<D, NSTAGE>) + 1024;
  {
    cudaError_t e = set_smem_attr((const void*)prefill_persist_kernel<D, NSTAGE>, smem);
    if (e != cudaSuccess) return e;
  }
  const int n_qt = (rg.nq + BM - 1) / BM;
  const int n_items = n_qt * BH;
  const int grid = std::max(1, std::min(n_items, 2 * num_sms()));
  const float scale_log2 = cfg.scale * 1.4426950408889634f;
  cudaError_t e = launch_pdl(prefill_persist_kernel<D, NSTAGE>, dim3(grid), dim3(NTHREADS), smem, s, mQ, mK, mV,
                             mKs, mVs, rg, cfg.chunk, cfg.window, cfg.mode, scale_log2,
                             cfg.summary_bias * 1.4426950408889634f, lse, (__nv_bfloat16*)O, n_qt, n_items);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

template <int D, int NSTAGE>
cudaError_t launch_split(const eva_config& cfg, const void* Q, const void* K, const void* V,
                         const void* Ksum, const void* Vsum, void* O, float* lse, cudaStream_t s) {
  const int BH = cfg.bh_count, T = cfg.T, nC = T / cfg.chunk;
  CUtensorMap mQ, mK, mV, mKs, mVs, mO;
  bool ok = make_map(&mQ, Q, BH, T, D, BM) && make_map(&mK, K, BH, T, D, BN) &&
            make_map(&mV, V, BH, T, D, BN) && make_map(&mO, O, BH, T, D, BM);
  if (nC > 0) {
    ok = ok && make_map(&mKs, Ksum, BH, nC, D, BN) && make_map(&mVs, Vsum, BH, nC, D, BN);
  } else {
    mKs = mK;
    mVs = mV;
  }
  if (!ok) return cudaErrorInvalidValue;
  const size_t smem = sizeof(Smem2<D, NSTAGE>) + 1024;
  {
    cudaError_t e = set_smem_attr((const void*)prefill_split_kernel<D, NSTAGE>, smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((T + BM - 1) / BM, BH);
  const float scale_log2 = cfg.scale * 1.4426950408889634f;
  prefill_split_kernel<D, NSTAGE><<<grid, NTHREADS2, smem, s>>>(mQ, mK, mV, mKs, mVs, mO, T, cfg.chunk,
                                                               cfg.window, cfg.mode, scale_log2, lse);
  note_launch();
  return cudaGetLastError();
}

template <int D, int NSK, int NSV>
cudaError_t launch_wide(const eva_config& cfg, const void* Q, const void* K, const void* V,
                        const void* Ksum, const void* Vsum, void* O, float* lse, cudaStream_t s) {
  const int BH = cfg.bh_count, T = cfg.T, nC = T / cfg.chunk;
  CUtensorMap mQ, mK, mV, mKs, mVs, mO;
  bool ok = make_map(&mQ, Q, BH, T, D, BM) && make_map(&mK, K, BH, T, D, BNW) &&
            make_map(&mV, V, BH, T, D, BNW) && make_map(&mO, O, BH, T, D, BM);
  if (nC > 0) {
    ok = ok && make_map(&mKs, Ksum, BH, nC, D, BNW) && make_map(&mVs, Vsum, BH, nC, D, BNW);
  } else {
    mKs = mK;
    mVs = mV;
  }
  if (!ok) return cudaErrorInvalidValue;
  const size_t smem = sizeof(SmemWide<D, NSK, NSV>) + 1024;
  {
    cudaError_t e = set_smem_attr((const void*)prefill_wide_kernel<D, NSK, NSV>, smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((T + BM - 1) / BM, BH);
  const float scale_log2 = cfg.scale * 1.4426950408889634f;
  prefill_wide_kernel<D, NSK, NSV><<<grid, NTHREADS, smem, s>>>(mQ, mK, mV, mKs, mVs, mO, T, cfg.chunk,
                                                               cfg.window, cfg.mode, scale_log2, lse);
  note_launch();
  return cudaGetLastError();
}

template <int D, int NS, bool TRACE = false>
cudaError_t launch_pair(const eva_config& cfg, const void* Q, const void* K, const void* V,
                        const void* Ksum, const void* Vsum, void* O, float* lse, cudaStream_t s) {
  const int BH = cfg.bh_count, T = cfg.T, nC = T / cfg.chunk;
  CUtensorMap mQ, mK, mV, mKs, mVs;
  bool ok = make_map(&mQ, Q, BH, T, D, BM) && make_map(&mK, K, BH, T, D, BN) &&
            make_map(&mV, V, BH, T, D, BN);
  if (nC > 0) {
    ok = ok && make_map(&mKs, Ksum, BH, nC, D, BN) && make_map(&mVs, Vsum, BH, nC, D, BN);
  } else {
    mKs = mK;
    mVs = mV;
  }
  if (!ok) return cudaErrorInvalidValue;
  const size_t smem = sizeof(SmemPair<D, NS>) + 1024 + (TRACE ? sizeof(TraceLog) : 0);
  {
    cudaError_t e = set_smem_attr((const void*)prefill_pair_kernel<D, NS, TRACE>, smem);
    if (e != cudaSuccess) return e;
  }
  const int ppu = (T + 2 * BM - 1) / (2 * BM);
  const int64_t items = (int64_t)BH * ppu;
  const int grid = (int)std::min<int64_t>(items, num_sms());  // 1 CTA/SM: all CTAs co-resident
  const float scale_log2 = cfg.scale * 1.4426950408889634f;
  prefill_pair_kernel<D, NS, TRACE><<<grid, PAIR_THREADS, smem, s>>>(mQ, mK, mV, mKs, mVs, BH, T, cfg.chunk,
                                                              cfg.window, cfg.mode, scale_log2,
                                                              (__nv_bfloat16*)O, lse);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

bool make_tma_map_bf16(CUtensorMap* m, const void* base, int units, int rows, int D, int box_rows) {
  return make_map(m, base, units, rows, D, box_rows);
}

cudaError_t debug_trace_prefill(const eva_config& cfg, const void* Q, const void* K, const void* V,
                                const void* Ksum, const void* Vsum, void* O, float* lse,
                                unsigned long long* trace_dev, int cap, cudaStream_t s) {
  cudaError_t e = cudaMemcpyToSymbolAsync(g_trace, &trace_dev, sizeof(trace_dev), 0, cudaMemcpyHostToDevice, s);
  const int zero = 0;
  if (e == cudaSuccess) e = cudaMemcpyToSymbolAsync(g_trace_n, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyToSymbolAsync(g_trace_cap, &cap, sizeof(int), 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  if (cfg.d_head == 128) return launch_pair<128, 4, true>(cfg, Q, K, V, Ksum, Vsum, O, lse, s);
  if (cfg.d_head == 64) return launch_pair<64, 8, true>(cfg, Q, K, V, Ksum, Vsum, O, lse, s);
  return cudaErrorNotSupported;
}

cudaError_t debug_trace_tile(const eva_config& cfg, const void* Q, const void* K, const void* V,
                             const void* Ksum, const void* Vsum, void* O, float* lse,
                             unsigned long long* trace_dev, cudaStream_t s) {
  cudaError_t e = cudaMemcpyToSymbolAsync(g_trace2, &trace_dev, sizeof(trace_dev), 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  const PrefillRange rg = full_range(cfg);
  if (cfg.d_head == 128) return launch_t<128, 2, true>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
  if (cfg.d_head == 64) return launch_t<64, 3, true>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
  return cudaErrorNotSupported;
}

bool prefill_sm100_supported(const eva_config& cfg) {
  return cfg.dtype == EVA_BF16 && (cfg.d_head == 64 || cfg.d_head == 128) && encode_fn() != nullptr;
}

cudaError_t launch_prefill_sm100(const eva_config& cfg, const PrefillRange& rg, const void* Q,
                                 const void* K, const void* V, const void* Ksum, const void* Vsum,
                                 void* O, float* lse, uint32_t variant, cudaStream_t s) {
  if (cfg.bh_count == 0) return cudaSuccess;
  const bool overlap = (variant & 0x100u) != 0;  // EVA_PREFILL_OVERLAP
  variant &= 0xffu;
  const PrefillRange full = full_range(cfg);
  if (rg.q0 != full.q0 || rg.nq != full.nq || rg.k0 != full.k0 || rg.nkv != full.nkv || rg.nsl != full.nsl)
    variant = 1;  // query-range calls: the one-tile-per-CTA kernel only
  if (cfg.mode == EVA_NONCAUSAL || cfg.summary_bias != 0.f) variant = 1;  // variants: tile kernel only
  // The one-tile-per-CTA kernel (two CTAs per SM) is the default: on B200 it beats the
  // persistent pair kernel at every measured size (configs[2]: 0.65 vs 0.90 ms); the pair
  // kernel stays selectable for experiments (EVA_PREFILL_TC_PAIR).
  bool pair = false;
  if (variant == 1) pair = false;
  if (variant == 2) pair = true;
  if (variant == 5) {
    if (cfg.d_head == 128) return launch_persist<128, 2>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
    if (cfg.d_head == 64) return launch_persist<64, 3>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
  }
  if (variant == 4) {
    if (cfg.d_head == 128) return launch_split<128, 2>(cfg, Q, K, V, Ksum, Vsum, O, lse, s);
    if (cfg.d_head == 64) return launch_split<64, 3>(cfg, Q, K, V, Ksum, Vsum, O, lse, s);
  }
  if (variant == 3) {
    if (cfg.d_head == 128) return launch_wide<128, 1, 1>(cfg, Q, K, V, Ksum, Vsum, O, lse, s);
    if (cfg.d_head == 64) return launch_wide<64, 2, 2>(cfg, Q, K, V, Ksum, Vsum, O, lse, s);
  }
  if (pair) {
    if (cfg.d_head == 128) return launch_pair<128, 5>(cfg, Q, K, V, Ksum, Vsum, O, lse, s);
    if (cfg.d_head == 64) return launch_pair<64, 8>(cfg, Q, K, V, Ksum, Vsum, O, lse, s);
  } else {
    // ring depths of the tile kernel (EVA_PREFILL_RING overrides: "2"/"32" at d=128, "3"/"54" at d=64)
    static const int ring = [] {
      const char* e = getenv("EVA_PREFILL_RING");
      return e ? atoi(e) : 0;
    }();
    if (cfg.d_head == 128) {
      if (ring == 32) return launch_t<128, 32>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
      return launch_t<128, 2>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
    }
    if (cfg.d_head == 64) {
      if (ring == 54) return launch_t<64, 54>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
      return launch_t<64, 3>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s, overlap);
    }
  }
  return cudaErrorNotSupported;
}

}  // namespace eva
