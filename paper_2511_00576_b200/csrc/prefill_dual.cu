// prefill_dual.cu -- the d = 128 bf16 FlashEVA prefill with 128-key tiles and two query tiles per
// CTA (opt-in, EVA_PREFILL_DUAL=1: measured slower than prefill_sm100.cu, see the end of this
// comment).
//
// Same result as prefill_sm100.cu (Eq.12-14, mask P:124): for every query n
//   o_n = softmax over { s q_n.k~_c : c < nsum(n) }  U  { s q_n.k_m : lo(n) <= m <= n }.
//
// Why a second kernel: on B200 an SS UMMA with N = 64 (the S tile of the 64-key kernel) takes 48
// cycles per K = 16 step where N = 128 takes 64 (scripts/umma_bench.cu: 2729 vs 4094 MAC/clk/SM),
// and the 64-key kernel at configs[2] spends 1260 cycles of one SM per 128x64 tile step, most
// of it in the tensor pipe (S 384 + PV 256 cycles per tile, two CTAs per SM).  128-key tiles need
// a 128-column S buffer per query tile: TMEM (512 columns) then holds one CTA per SM with two
// query tiles -- S0 [0,128) O0 [128,256) S1 [256,384) O1 [384,512) -- whose chains ping-pong on
// the tensor pipe: while softmax warpgroup 0 exponentiates S0(j), the pipe runs PV1(j-1) and
// S1(j), and the other way round.
//
// Persistent CTA (grid = SMs): items (unit, pair of 128-query tiles) i = blockIdx.x + k*gridDim.x,
// unit-major so that neighbouring CTAs share the unit's K/V and summaries in L2.  Roles:
//   warp 0      TMA producer: Q0/Q1 of each item (once their previous S MMAs completed), then
//               the item's 128-row K/V tiles through 2-deep K and V rings; the union of the two
//               query tiles' key tiles is walked once (summary tiles first, then local).
//   warp 1      TMEM allocator + MMA issuer: for every key tile j and query tile i that sees it,
//               PV_i(previous) then S_i(j) = Q_i K_j^T (SS, M=128 N=128 K=128); PV_i(j) =
//               P_i(j) V_j (TS, P read from TMEM, M=128 N=128 K=128) is issued when the next
//               S_i comes (or the stream ends), so a query tile's chain continues into the next
//               item while its epilogue still runs.
//   warps 4-7   softmax warpgroup of query tile 0, warps 8-11 of query tile 1: thread <-> TMEM
//               lane <-> query row; per 128-column tile: mask, online max with lazy rescale
//               (2^8), P = exp2 packed to bf16 in place; epilogue O / l straight from TMEM to
//               global memory (16-byte stores per row), LSE, then O's TMEM columns are released.
//
// Measured (configs[2] attention, B200): 0.877 ms (two-pass softmax; one-pass 0.977, with a
// quarter of the exponentials on the FMA pipe 0.887) against 0.579 ms for prefill_sm100.cu.
// The CTA-0 timeline (scripts/trace_dual.py) shows why: a 128-column softmax step takes 2.8-4k
// cycles (the exponentials alone are 1024 MUFU cycles per warp, and both warpgroups' warps share
// each sub-partition's MUFU), issuing 8 UMMAs takes ~800 cycles (issue blocks at the pipe's
// rate), and each query tile's chain S -> softmax -> PV -> next S is serial because its S buffer
// is also its P buffer; the two chains interleave only partly.  Kept for the record and as the
// starting point of an FA4-style schedule (exp2 emulation balanced against MUFU, a correction
// warpgroup, ready-first MMA issue).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "prefill_common.cuh"
#include "sm100.cuh"

namespace eva {
namespace {

using namespace sm100;
using namespace pfx;
constexpr int D = 128;
constexpr int BM = 128;   // queries per query tile (two per item)
constexpr int BN = 128;   // keys per key tile
constexpr int NK = 2, NV = 2;
// 12 warps = 3 warpgroups: warps 0 (producer) and 1 (MMA) of warpgroup 0 hand registers to the
// two softmax warpgroups (setmaxnreg), whose 128-column tiles need ~170 live registers
constexpr int NTHREADS = 384;
constexpr uint32_t REG_CTRL = 72, REG_SOFTMAX = 216;  // 128 * (56 + 2 * 224) = 384 * 168
constexpr uint32_t TMEM_COLS = 512;

template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

struct __align__(1024) DualSmem {
  __nv_bfloat16 q[2][BM * D];   // per query tile: 2 sub-tiles [128][64] (16 KB each)
  __nv_bfloat16 k[NK][BN * D];  // 2 sub-tiles [128][64]
  __nv_bfloat16 v[NV][BN * D];
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[NK], k_empty[NK], v_full[NV], v_empty[NV];
  uint64_t s_full[2], p_full[2], o_done[2], o_final[2], o_free[2];
  uint32_t tmem_base;
};

// The key tiles of one item: the summary prefix [0, max nsum) in 128-chunk tiles, then the
// local span [lo(n0 of tile 0), last row + 1) in 128-key tiles; need(i, j) says whether query
// tile i sees any key of tile j (its summary prefix / local span intersects it).
struct DualPlan {
  int u, qt0;
  bool valid[2];
  int64_t n0[2], nlast[2], lo[2], s1[2];
  int64_t lo0, k0;
  int n_st, n_lt;
  __device__ DualPlan(int item, int n_pairs, int n_qt, const PrefillRange& rg, int C, int W, int mode) {
    u = item / n_pairs;
    const int pair = item % n_pairs;
    qt0 = 2 * pair;
    const int64_t qend = rg.q0 + rg.nq;
    int64_t s1max = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      valid[i] = qt0 + i < n_qt;
      n0[i] = rg.q0 + (int64_t)(qt0 + i) * BM;
      nlast[i] = min(n0[i] + BM - 1, qend - 1);
      if (valid[i]) {
        const Vis vf = visible_set(n0[i], C, W, mode, qend), vl = visible_set(nlast[i], C, W, mode, qend);
        lo[i] = vf.lo;
        s1[i] = vl.s1;
        s1max = max(s1max, s1[i]);
        hi = max(hi, vl.hi);
      } else {
        lo[i] = INT64_MAX;
        s1[i] = 0;
      }
    }
    lo0 = lo[0];
    k0 = rg.k0;
    n_st = (int)((s1max + BN - 1) / BN);
    n_lt = (int)((hi - lo0 + BN - 1) / BN);
  }
  __device__ int count() const { return n_st + n_lt; }
  __device__ bool summary(int j) const { return j < n_st; }
  __device__ int64_t base(int j) const { return j < n_st ? (int64_t)j * BN : lo0 + (int64_t)(j - n_st) * BN; }
  __device__ int row(int j) const { return j < n_st ? (int)base(j) : (int)(base(j) - k0); }
  // (selects, not indexing: i is a runtime value and indexed member arrays would go to local memory)
  __device__ bool need(int i, int j) const {
    if (!(i ? valid[1] : valid[0])) return false;
    if (j < n_st) return (int64_t)j * BN < (i ? s1[1] : s1[0]);
    const int64_t b = base(j);
    return b <= (i ? nlast[1] : nlast[0]) && b + BN > (i ? lo[1] : lo[0]);
  }
  __device__ int last(int i) const {  // the last key tile query tile i sees
    for (int j = count() - 1; j >= 0; --j)
      if (need(i, j)) return j;
    return -1;
  }
};

// One softmax step of a 128-key tile for this thread's query row: the 64-key kernel's step
// (prefill_sm100.cu softmax_tile2) widened to 128 columns.  P (bf16 pairs) lands in the first 64
// TMEM columns of the S buffer, the A operand of the PV MMA.
// EMU: of every 8 column pairs, EMU are exponentiated by exp2_poly2 on the FMA pipe instead of
// MUFU.EX2 (two warpgroups exponentiate at once here: 32768 exponentials per 128-key step pair,
// 2048 cycles of the MUFU pipe alone).
template <int EMU, typename WaitO, typename Mark>
__device__ __forceinline__ void softmax128(uint32_t s_addr, uint32_t o_addr, int vlo, int vhi, float bias2,
                                           float scale_log2, float& m_ref, float& l, const WaitO& wait_o,
                                           const Mark& mark) {
  uint32_t sr[128];
#pragma unroll
  for (int q = 0; q < 4; ++q) tmem_ld32(s_addr + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * q]));
  tmem_wait_ld();
  mark(13);
  const bool full = vlo <= 0 && vhi >= 128;
  if (!__all_sync(0xffffffffu, full)) {
    const uint64_t m0 = range_bits(vlo, vhi), m1 = range_bits(vlo - 64, vhi - 64);
    const uint32_t mw[4] = {(uint32_t)m0, (uint32_t)(m0 >> 32), (uint32_t)m1, (uint32_t)(m1 >> 32)};
#pragma unroll
    for (int c = 0; c < 128; ++c) {
      const uint32_t keep = (uint32_t)((int32_t)(mw[c >> 5] << (31 - (c & 31))) >> 31);
      sr[c] = (sr[c] & keep) | (0xff800000u & ~keep);
    }
  }
  float pm[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) pm[i] = __uint_as_float(sr[i]);
#pragma unroll
  for (int c = 8; c < 128; ++c) pm[c & 7] = fmaxf(pm[c & 7], __uint_as_float(sr[c]));
  float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
  mx = mx * scale_log2 + bias2;
  const bool grow = mx > m_ref + 8.0f;
  mark(14);
  if (__any_sync(0xffffffffu, grow && m_ref != -INFINITY)) {
    const float f = (grow && m_ref != -INFINITY) ? ex2(m_ref - mx) : 1.0f;
    wait_o();
    mark(15);
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
  for (int c = 0; c < 64; ++c) {
    const uint64_t x = ffma2(f2pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sc2, ng2);
    uint64_t p;
    if ((c & 7) < EMU) p = exp2_poly2(x);
    else p = f2pack(ex2(f2lo(x)), ex2(f2hi(x)));
    ls[c & 3] = fadd2(ls[c & 3], p);
    sr[c] = pack_bf16(f2lo(p), f2hi(p));
  }
  const uint64_t s2 = fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3]));
  l += f2lo(s2) + f2hi(s2);
  mark(16);
  tmem_st32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
  tmem_st32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
  tmem_wait_st();
  tc_fence_before();
}

// Two-pass variant: the tile is read from TMEM twice in 64-column halves (rolled loops), the
// first pass for the row max, the second for P -- the code of one 64-column half instead of a
// fully unrolled 128-column step (instruction-cache footprint, ~64 fewer live registers).  P of
// half h lands in TMEM columns [32h, 32h + 32), which hold S values already re-read.
template <int EMU, typename WaitO, typename Mark>
__device__ __forceinline__ void softmax128_2p(uint32_t s_addr, uint32_t o_addr, int vlo, int vhi, float bias2,
                                              float scale_log2, float& m_ref, float& l, const WaitO& wait_o,
                                              const Mark& mark) {
  const bool full = __all_sync(0xffffffffu, vlo <= 0 && vhi >= 128);
  auto load_half = [&](int h, uint32_t (&sr)[64]) {
    tmem_ld32(s_addr + 64 * h, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
    tmem_ld32(s_addr + 64 * h + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
    tmem_wait_ld();
    if (!full) {
      const uint64_t m = range_bits(vlo - 64 * h, vhi - 64 * h);
      const uint32_t mw[2] = {(uint32_t)m, (uint32_t)(m >> 32)};
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        const uint32_t keep = (uint32_t)((int32_t)(mw[c >> 5] << (31 - (c & 31))) >> 31);
        sr[c] = (sr[c] & keep) | (0xff800000u & ~keep);
      }
    }
  };
  float pm[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) pm[i] = -INFINITY;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    uint32_t sr[64];
    load_half(h, sr);
#pragma unroll
    for (int c = 0; c < 64; ++c) pm[c & 7] = fmaxf(pm[c & 7], __uint_as_float(sr[c]));
  }
  mark(13);
  float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
  mx = mx * scale_log2 + bias2;
  const bool grow = mx > m_ref + 8.0f;
  mark(14);
  if (__any_sync(0xffffffffu, grow && m_ref != -INFINITY)) {
    const float f = (grow && m_ref != -INFINITY) ? ex2(m_ref - mx) : 1.0f;
    wait_o();
    mark(15);
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
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    uint32_t sr[64];
    load_half(h, sr);
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint64_t x = ffma2(f2pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sc2, ng2);
      uint64_t p;
      if ((c & 7) < EMU) p = exp2_poly2(x);
      else p = f2pack(ex2(f2lo(x)), ex2(f2hi(x)));
      ls[c & 3] = fadd2(ls[c & 3], p);
      sr[c] = pack_bf16(f2lo(p), f2hi(p));
    }
    tmem_st32(s_addr + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
  }
  const uint64_t s2 = fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3]));
  l += f2lo(s2) + f2hi(s2);
  mark(16);
  tmem_wait_st();
  tc_fence_before();
}

// Debug timeline (eva_debug_trace_prefill variant 3): CTA 0 logs clock64 events per role --
// 0 producer, 1 MMA, 2/3 softmax warpgroup 0/1 (first warp, lane 0) -- flushed to g_dual_trace.
// kinds: 1 Q(i) load issued, 2 K(j) issued, 3 V(j) issued, 4 K(j) seen by MMA, 5 S_i(j) issued,
// 6 P_i seen, 7 PV_i issued, 8 S_i(j) seen by softmax, 9 P_i(j) done, 10 O final seen,
// 11 epilogue done, 12 item start; j carries (i << 12) | j.
__device__ unsigned long long* g_dual_trace = nullptr;
constexpr int DT_PER_ROLE = 160;
struct DualTrace {
  unsigned long long ev[4][DT_PER_ROLE];
  int n[4];
};
template <bool TRACE>
__device__ __forceinline__ void dt(DualTrace* tl, int role, int kind, int j) {
  if constexpr (TRACE) {
    if (blockIdx.x == 0) {
      const int i = tl->n[role];
      if (i < DT_PER_ROLE) tl->ev[role][i] = ((unsigned long long)clock64() << 24) | ((unsigned)kind << 16) | (unsigned)(j & 0xffff);
      tl->n[role] = i + 1;
    }
  }
}

template <bool TRACE, int EMU, bool TWOPASS>
__global__ void __launch_bounds__(NTHREADS, 1)
prefill_dual_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                    const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mKs,
                    const __grid_constant__ CUtensorMap mVs, __nv_bfloat16* __restrict__ O,
                    const PrefillRange rg, int C, int W, int mode, float scale_log2, float bias_log2,
                    float* __restrict__ lse, int n_items, int n_pairs, int n_qt) {
  extern __shared__ uint8_t smem_raw[];
  DualSmem* sm = reinterpret_cast<DualSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DualTrace* tl = nullptr;
  if constexpr (TRACE) {
    __shared__ DualTrace tlog_s;
    tl = &tlog_s;
    if (threadIdx.x < 4) tl->n[threadIdx.x] = 0;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV);
    tma_prefetch(&mKs); tma_prefetch(&mVs);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm->q_full[i], 1);
      mbar_init(&sm->q_empty[i], 1);
      mbar_init(&sm->s_full[i], 1);
      mbar_init(&sm->p_full[i], 128);
      mbar_init(&sm->o_done[i], 1);
      mbar_init(&sm->o_final[i], 1);
      mbar_init(&sm->o_free[i], 128);
    }
    for (int s = 0; s < NK; ++s) {
      mbar_init(&sm->k_full[s], 1);
      mbar_init(&sm->k_empty[s], 1);
    }
    // a V slot is released by one arrival per query tile: the PV commit of a tile that reads
    // it, a plain arrive for a tile that does not
    for (int s = 0; s < NV; ++s) {
      mbar_init(&sm->v_full[s], 1);
      mbar_init(&sm->v_empty[s], 2);
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
  pdl_wait();
  pdl_trigger();
  // the two-pass softmax holds half the tile: more registers to the producer / MMA warps
  constexpr uint32_t RC = TWOPASS ? 152 : REG_CTRL, RS = TWOPASS ? 176 : REG_SOFTMAX;
  static_assert(RC + 2 * RS == 3 * 168, "register split");
  if (warp < 4) {
  setmaxnreg_dec<RC>();
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    int kc = 0, vc = 0, qc[2] = {0, 0};
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const DualPlan plan(item, n_pairs, n_qt, rg, C, W, mode);
      const int NT = plan.count();
      auto load_q = [&](int i) {
        if (!plan.valid[i]) return;
        if (qc[i] > 0) mbar_wait(&sm->q_empty[i], (qc[i] - 1) & 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm->q_full[i], BM * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->q[i] + kb * BM * 64, &mQ, &sm->q_full[i], kb * 64, (plan.qt0 + i) * BM, plan.u);
        }
        __syncwarp();
        if (lane == 0) dt<TRACE>(tl, 0, 1, i << 12);
        ++qc[i];
      };
      auto load_k = [&](int j) {
        const int s = kc % NK;
        if (kc >= NK) mbar_wait(&sm->k_empty[s], ((kc / NK) - 1) & 1);
        const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm->k_full[s], BN * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->k[s] + kb * BN * 64, mk, &sm->k_full[s], kb * 64, plan.row(j), plan.u);
        }
        __syncwarp();
        if (lane == 0) dt<TRACE>(tl, 0, 2, j);
        ++kc;
      };
      auto load_v = [&](int j) {
        const int s = vc % NV;
        if (vc >= NV) mbar_wait(&sm->v_empty[s], ((vc / NV) - 1) & 1);
        const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm->v_full[s], BN * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->v[s] + kb * BN * 64, mv, &sm->v_full[s], kb * 64, plan.row(j), plan.u);
        }
        __syncwarp();
        if (lane == 0) dt<TRACE>(tl, 0, 3, j);
        ++vc;
      };
      // the item's later tiles into L2 now (the rings hold two)
      if (elect_one()) {
        for (int j = 2; j < NT; ++j) {
          const CUtensorMap* mk = plan.summary(j) ? &mKs : &mK;
          const CUtensorMap* mv = plan.summary(j) ? &mVs : &mV;
          for (int kb = 0; kb < D / 64; ++kb) {
            tma_prefetch_l2_3d(mk, kb * 64, plan.row(j), plan.u);
            tma_prefetch_l2_3d(mv, kb * 64, plan.row(j), plan.u);
          }
        }
      }
      __syncwarp();
      load_q(0);
      load_k(0);
      load_q(1);
      if (NT > 1) load_k(1);
      load_v(0);
      for (int j = 1; j < NT; ++j) {
        if (j + 1 < NT) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(BM, BN, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(BM, D, true);
    int kc = 0, vc_base = 0;       // ring positions of the current item's tile 0
    int qc[2] = {0, 0};            // items seen per query tile (q_full / q_empty / o_free phases)
    int pc[2] = {0, 0};            // P tiles consumed per query tile (p_full phases)
    int pend[2] = {-1, -1};        // key tile (ring index) whose PV is pending, per query tile
    bool pend_last[2] = {false, false}, pend_first[2] = {false, false}, pend_other[2] = {false, false};
    // PV_i of the pending tile: P_i ready, V landed; accumulate unless it is the item's first
    // (then the previous item's epilogue must have read O_i); commit o_done (and o_final at the
    // item's end); release the V slot for this query tile (and for the other one if it skips it)
    auto issue_pv = [&](int i) {
      const int g = pend[i], s = g % NV;
      mbar_wait(&sm->p_full[i], pc[i] & 1);
      if (lane == 0) dt<TRACE>(tl, 1, 6, i << 12);
      ++pc[i];
      mbar_wait(&sm->v_full[s], (g / NV) & 1);
      if (pend_first[i] && qc[i] > 1) mbar_wait(&sm->o_free[i], (qc[i] - 2) & 1);
      tc_fence_after();
      const uint32_t v_addr = smem_u32(sm->v[s]);
      const uint32_t s_tm = tmem + (uint32_t)i * 256, o_tm = s_tm + 128;
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < BN / 16; ++ks) {
          const uint64_t b = smem_desc_sw128(v_addr + ks * 16 * 128, BN * 128, 1024);
          mma_ts(o_tm, s_tm + ks * 8, b, idesc_o, (!pend_first[i] || ks > 0) ? 1u : 0u);
        }
        mma_commit(&sm->o_done[i]);
        if (pend_last[i]) mma_commit(&sm->o_final[i]);
        mma_commit(&sm->v_empty[s]);
        if (!pend_other[i]) mbar_arrive(&sm->v_empty[s]);
      }
      __syncwarp();
      if (lane == 0) dt<TRACE>(tl, 1, 7, i << 12);
      pend[i] = -1;
    };
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const DualPlan plan(item, n_pairs, n_qt, rg, C, W, mode);
      const int NT = plan.count();
      const int lastj[2] = {plan.last(0), plan.last(1)};
      if (lane == 0) dt<TRACE>(tl, 1, 12, item);
      bool first[2] = {true, true};
      for (int j = 0; j < NT; ++j) {
        const int g = kc, s = g % NK;
        mbar_wait(&sm->k_full[s], (g / NK) & 1);
        if (lane == 0) dt<TRACE>(tl, 1, 4, j);
        const uint32_t k_addr = smem_u32(sm->k[s]);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (!plan.need(i, j)) {
            if (pend[i] >= 0 && pend_last[i]) issue_pv(i);  // finish the previous item's O_i now
            continue;
          }
          if (pend[i] >= 0) issue_pv(i);
          if (first[i]) {
            mbar_wait(&sm->q_full[i], qc[i] & 1);
            ++qc[i];
          }
          tc_fence_after();
          const uint32_t q_addr = smem_u32(sm->q[i]);
          const uint32_t s_tm = tmem + (uint32_t)i * 256;
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
              const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
              const uint64_t a = smem_desc_sw128(q_addr + kb * (BM * 128) + off, 16, 1024);
              const uint64_t b = smem_desc_sw128(k_addr + kb * (BN * 128) + off, 16, 1024);
              mma_ss(s_tm, a, b, idesc_s, ks > 0 ? 1u : 0u);
            }
            mma_commit(&sm->s_full[i]);
            if (j == lastj[i]) mma_commit(&sm->q_empty[i]);
          }
          __syncwarp();
          if (lane == 0) dt<TRACE>(tl, 1, 5, (i << 12) | j);
          pend[i] = vc_base + j;
          pend_first[i] = first[i];
          pend_last[i] = j == lastj[i];
          pend_other[i] = plan.need(1 - i, j);
          first[i] = false;
        }
        if (elect_one()) mma_commit(&sm->k_empty[s]);
        __syncwarp();
        ++kc;
      }
      vc_base += NT;
    }
    for (int i = 0; i < 2; ++i)
      if (pend[i] >= 0) issue_pv(i);
  }
  } else {
    setmaxnreg_inc<RS>();
    // ------------------------------------------------------------ softmax warpgroups
    const int i = (warp - 4) >> 2;  // query tile
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t t_lane = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)i * 256;
    const int64_t qend = rg.q0 + rg.nq;
    int sc = 0, ic = 0;  // S tiles and items processed by this query tile
    const bool tw = (warp & 3) == 0 && lane == 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const DualPlan plan(item, n_pairs, n_qt, rg, C, W, mode);
      if (!(i ? plan.valid[1] : plan.valid[0])) continue;
      const int NT = plan.count();
      const int64_t n = (i ? plan.n0[1] : plan.n0[0]) + r;
      const bool valid = n < qend;
      const Vis rr = visible_set(valid ? n : (i ? plan.nlast[1] : plan.nlast[0]), C, W, mode, qend);
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < NT; ++j) {
        if (!plan.need(i, j)) continue;
        mbar_wait(&sm->s_full[i], sc & 1);
        if (tw) dt<TRACE>(tl, 2 + i, 8, j);
        tc_fence_after();
        const int64_t base = plan.base(j);
        int vlo, vhi;
        float bias2 = 0.f;
        if (plan.summary(j)) {
          vlo = 0;
          vhi = (int)min((int64_t)BN, rr.s1 - base);
          bias2 = bias_log2;
        } else {
          vlo = (int)max((int64_t)0, rr.lo - base);
          vhi = (int)min((int64_t)BN, rr.hi - base);
        }
        if (!valid) vhi = vlo;
        const int sprev = sc;
        auto wait_fn = [&] { mbar_wait(&sm->o_done[i], (sprev - 1) & 1); };
        auto mark_fn = [&](int k) { if (tw) dt<TRACE>(tl, 2 + i, k, j); };
        if constexpr (TWOPASS)
          softmax128_2p<EMU>(t_lane, t_lane + 128, vlo, vhi, bias2, scale_log2, m_ref, l, wait_fn, mark_fn);
        else
          softmax128<EMU>(t_lane, t_lane + 128, vlo, vhi, bias2, scale_log2, m_ref, l, wait_fn, mark_fn);
        mbar_arrive(&sm->p_full[i]);
        if (tw) dt<TRACE>(tl, 2 + i, 9, j);
        ++sc;
      }
      // ---------------------------------------------------------- epilogue
      mbar_wait(&sm->o_final[i], ic & 1);
      if (tw) dt<TRACE>(tl, 2 + i, 10, 0);
      ++ic;
      tc_fence_after();
      const float inv_l = l > 0.f ? 1.0f / l : 0.f;
      __nv_bfloat16* orow = O + ((size_t)plan.u * rg.nq + (size_t)(valid ? n - rg.q0 : 0)) * D;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32(t_lane + 128 + cc * 32, o);
        tmem_wait_ld();
        if (cc == D / 32 - 1) {  // O's TMEM columns are free for the next item's first PV
          tc_fence_before();
          mbar_arrive(&sm->o_free[i]);
        }
        if (valid) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(o[8 * g + 0]) * inv_l, __uint_as_float(o[8 * g + 1]) * inv_l);
            w.y = pack_bf16(__uint_as_float(o[8 * g + 2]) * inv_l, __uint_as_float(o[8 * g + 3]) * inv_l);
            w.z = pack_bf16(__uint_as_float(o[8 * g + 4]) * inv_l, __uint_as_float(o[8 * g + 5]) * inv_l);
            w.w = pack_bf16(__uint_as_float(o[8 * g + 6]) * inv_l, __uint_as_float(o[8 * g + 7]) * inv_l);
            *reinterpret_cast<uint4*>(orow + cc * 32 + 8 * g) = w;
          }
        }
      }
      if (valid && lse) lse[(size_t)plan.u * rg.nq + (size_t)(n - rg.q0)] = (m_ref + __log2f(l)) * 0.69314718055994531f;
      if (tw) dt<TRACE>(tl, 2 + i, 11, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (TRACE) {
    if (blockIdx.x == 0 && g_dual_trace) {
      for (int k = threadIdx.x; k < 4 * DT_PER_ROLE; k += blockDim.x) {
        const int r = k / DT_PER_ROLE, e = k % DT_PER_ROLE;
        g_dual_trace[k] = e < tl->n[r] ? tl->ev[r][e] : 0ull;
      }
    }
  }
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace

bool prefill_dual_supported(const eva_config& cfg) {
  return cfg.dtype == EVA_BF16 && cfg.d_head == 128 && cfg.mode != EVA_NONCAUSAL;
}

namespace {
template <bool TRACE, int EMU, bool TWOPASS = true>
cudaError_t launch_dual_t(const eva_config& cfg, const PrefillRange& rg, const void* Q, const void* K,
                          const void* V, const void* Ksum, const void* Vsum, void* O, float* lse,
                          cudaStream_t s) {
  if (!prefill_dual_supported(cfg)) return cudaErrorNotSupported;
  const int BH = cfg.bh_count, nC = rg.nsl;
  if (BH == 0 || rg.nq == 0) return cudaSuccess;
  CUtensorMap mQ, mK, mV, mKs, mVs;
  bool ok = make_tma_map_bf16(&mQ, Q, BH, rg.nq, D, BM) && make_tma_map_bf16(&mK, K, BH, rg.nkv, D, BN) &&
            make_tma_map_bf16(&mV, V, BH, rg.nkv, D, BN);
  if (nC > 0) {
    ok = ok && make_tma_map_bf16(&mKs, Ksum, BH, nC, D, BN) && make_tma_map_bf16(&mVs, Vsum, BH, nC, D, BN);
  } else {  // never read (no summary tiles)
    mKs = mK;
    mVs = mV;
  }
  if (!ok) return cudaErrorInvalidValue;
  const size_t smem = sizeof(DualSmem) + 1024;
  auto kern = prefill_dual_kernel<TRACE, EMU, TWOPASS>;
  cudaError_t e = set_smem_attr((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  const int n_qt = (rg.nq + BM - 1) / BM, n_pairs = (n_qt + 1) / 2;
  const int n_items = n_pairs * BH;
  const int grid = std::min(n_items, num_sms());
  const float scale_log2 = cfg.scale * 1.4426950408889634f;
  e = launch_pdl(kern, dim3(grid), dim3(NTHREADS), smem, s, mQ, mK, mV, mKs, mVs,
                 (__nv_bfloat16*)O, rg, cfg.chunk, cfg.window, cfg.mode, scale_log2,
                 cfg.summary_bias * 1.4426950408889634f, lse, n_items, n_pairs, n_qt);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}
// Exponentials on the FMA pipe per 8 column pairs (EVA_DUAL_EMU, default 0; -1: the one-pass
// softmax).
int dual_emu() {
  static const int v = [] {
    const char* e = getenv("EVA_DUAL_EMU");
    return e ? atoi(e) : 0;
  }();
  return v;
}
}  // namespace

cudaError_t launch_prefill_dual(const eva_config& cfg, const PrefillRange& rg, const void* Q, const void* K,
                                const void* V, const void* Ksum, const void* Vsum, void* O, float* lse,
                                cudaStream_t s) {
  if (dual_emu() < 0) return launch_dual_t<false, 0, false>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
  switch (dual_emu()) {
    case 1: return launch_dual_t<false, 1>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
    case 2: return launch_dual_t<false, 2>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
    case 3: return launch_dual_t<false, 3>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
    case 4: return launch_dual_t<false, 4>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
    default: return launch_dual_t<false, 0>(cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
  }
}

cudaError_t debug_trace_dual(const eva_config& cfg, const void* Q, const void* K, const void* V, const void* Ksum,
                             const void* Vsum, void* O, float* lse, unsigned long long* trace_dev, cudaStream_t s) {
  cudaError_t e = cudaMemcpyToSymbolAsync(g_dual_trace, &trace_dev, sizeof(trace_dev), 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  return launch_dual_t<true, 0>(cfg, full_range(cfg), Q, K, V, Ksum, Vsum, O, lse, s);
}

}  // namespace eva
