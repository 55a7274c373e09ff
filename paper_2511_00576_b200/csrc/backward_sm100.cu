// backward_sm100.cu -- tensor-core (tcgen05/TMEM/TMA) main pass of the FlashEVA prefill
// backward (the paper trains with it), bf16, d = 128.
//
// It replaces bwd_main_kernel of backward_simt.cu for that case: the prep kernel has written
// D_n = dO_n . o_n and zeroed the fp32 accumulators.  Two schedules (launch_backward):
//   unfused: one launch over every work item, local dK/dV to the fp32 workspace, then the
//            finalize kernel applies the summary chain rule (k~ = chunk mean, Eq.15 omega,
//            log-xi softmax) and converts;
//   fused (default): the summary items, then bwd_coef (the chain-rule coefficients: w_i, da_i
//            per row, omega_c and d k~_c / C per chunk), then the local items, whose drain
//            applies the chain rule and stores bf16 dK/dV directly, then the dQ conversion --
//            no fp32 dK/dV round trip through HBM (4.3 GB less traffic at configs[2]).
//
// Work item = one unit x one tile of 128 keys (local keys, or 128 summaries k~_c / beta_c
// with a segment of the query tiles that see them); the CTA walks its 64-query tiles:
//     S^T  = K Q_i^T                (SS, M=128 keys, N=64 queries, K=d)     TMEM [0,64)
//     dP^T = V dO_i^T               (SS)                                    TMEM [64,128)
//     P^T  = exp2(s S^T log2e - lse2),  dS^T = P^T (dP^T - D)   (thread <-> key row; mask)
//            P^T, dS^T bf16 back into TMEM (A operands), dS^T also into smem (swizzled)
//     dV  += P^T dO_i               (TS, M=128, N=d, K=64)                   TMEM [256,384)
//     dK  += dS^T Q_i               (TS)                                    TMEM [384,512)
//     dQ_i^T = K^T dS^T             (SS, A = K tile MN-major, B = dS^T MN-major; M=d, N=64)
//            -> fp32 red.global.add into the dQ accumulator (thread <-> channel)
// Warps: 0 TMA producer (K/V once, Q_i/dO_i through a 2-stage ring), 1 TMEM allocator +
// single-thread MMA issuer, 2-5 softmax/dS + dQ epilogue + dK/dV write-out.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "sm100.cuh"

namespace eva {
namespace {

using namespace sm100;
constexpr int BK = 128;  // keys per work item (MMA M)
// query tiles per summary work item: chosen per launch (bwd_seg_for), 8 .. 32
constexpr int BWD_TC_THREADS = 320;

// Tiling per head dim.  d = 128: 64-query steps, dQ computed transposed (dQ^T = K^T dS^T,
// M = d = 128); d = 64: 128-query steps, dQ = dS K (M = 128 queries).  TMEM columns:
// S^T, dP^T (BQ each), dQ, dV, dK.
template <int D> struct BwdT;
// NK: K tile buffers -- 2 lets the next work item's K load run under the current item.
// Measured at configs[2] (fused schedule): d = 128 with NK = 2 has room only for a 2-slot
// Q/dO ring and is slower (3.42 vs 3.33 ms), so it keeps NSQ = 3, NK = 1; d = 64 takes
// NK = 2 (neutral at configs[1]).
template <> struct BwdT<128> {
  static constexpr int BQ = 64, NSQ = 3, PBUF = 1, NK = 1;
  static constexpr bool DQT = true;
  // P^T and dS^T go to shared memory (the dV/dK MMAs read them from there), so S^T/dP^T in
  // TMEM are free as soon as the softmax warps have loaded them: the next step's S/dP MMAs
  // run during this step's softmax.
  static constexpr bool PSMEM = true;
  static constexpr uint32_t TM_S = 0, TM_DP = 64, TM_DQ = 128, TM_DV = 256, TM_DK = 384;
  static constexpr int DQS_FLOATS = 32 * 128;  // staging [32 queries][128] (column writes),
                                               // the 64-query dQ tile in two halves
};
template <> struct BwdT<64> {
  static constexpr int BQ = 128, NSQ = 2, PBUF = 1, NK = 2;
  static constexpr bool DQT = false;
  static constexpr bool PSMEM = false;  // P^T, dS^T back into TMEM (TS MMAs)
  static constexpr uint32_t TM_S = 0, TM_DP = 128, TM_DQ = 256, TM_DV = 320, TM_DK = 384;
  static constexpr int DQS_FLOATS = BQ * 68;   // staging rows padded to 68 floats (row writes)
};

template <int D>
struct __align__(1024) BwdSm {
  static constexpr int BQ = BwdT<D>::BQ, NSQ = BwdT<D>::NSQ;
  __nv_bfloat16 k[BwdT<D>::NK][BK * D];  // D/64 sub-tiles [128 keys][64 ch], 16 KB each
  __nv_bfloat16 v[BK * D];
  __nv_bfloat16 q[NSQ][BQ * D];   // D/64 sub-tiles [BQ queries][64 ch]
  __nv_bfloat16 dO[NSQ][BQ * D];
  __nv_bfloat16 ds[2][BK * BQ];   // dS^T [128 keys][BQ queries]: BQ/64 sub-tiles of 128-byte
                                  // swizzled rows, double-buffered
  float dqs[BwdT<D>::DQS_FLOATS]; // dQ staging (fp32) for the bulk reduce-add
  __nv_bfloat16 p[BwdT<D>::PBUF][BwdT<D>::PSMEM ? BK * BQ : 8];  // P^T [128 keys][BQ] (PSMEM)
  float lse2[NSQ][BQ], Dq[NSQ][BQ];  // per Q/dO ring slot, loaded by the producer warp
  uint64_t k_full[BwdT<D>::NK], v_full, k_free[BwdT<D>::NK], v_free, q_full[NSQ], q_empty[NSQ], s_full, p_full, st_free, dq_full, dq_free,
      ds_free[2], acc_done, acc_free, s_free, p_free[BwdT<D>::PBUF];
  uint32_t tmem_base;
};

struct BwdWsT {
  float *D, *dQ, *dK, *dV, *dKs, *dVs;
};
// Fused summary chain rule for the local items (launch split: summary items, then
// bwd_coef_kernel, then the local items with this set).  For key row m of complete chunk
// c = m / C (the finalize's formulas, backward_simt.cu):
//     dK_m = s dK_local + da_m (omega_c - k_m) + dkt_c,   dV_m = dV_local + w_m dbeta_c
// with w, da per row and omega, dkt (= d k~ / C) per chunk from bwd_coef_kernel and dbeta_c
// the summary items' fp32 accumulator; written straight to the bf16 outputs (no fp32 dK / dV
// round trip).  dK == nullptr: the unfused path (fp32 workspace + finalize).
struct BwdFused {
  const float *w, *da, *om, *dkt;
  const __nv_bfloat16* K;
  __nv_bfloat16 *dK, *dV;
};

// Inverse maps of the mask (same formulas as backward_simt.cu): queries [qlo_of_key,
// qhi_of_key] see local key m; summary c is seen from qlo_of_summary on -- for the
// non-causal partition (R15) by every query outside the block of W holding chunk c.
__host__ __device__ __forceinline__ int64_t qlo_of_key(int64_t m, int W, int mode) {
  return mode == EVA_NONCAUSAL ? (m / W) * (int64_t)W : m;
}
__host__ __device__ __forceinline__ int64_t qhi_of_key(int64_t m, int C, int W, int mode) {
  if (mode == EVA_WINDOW_SLIDING) return (m / C + W / C) * (int64_t)C - 1;
  return (m / W + 1) * (int64_t)W - 1;
}
__host__ __device__ __forceinline__ int64_t qlo_of_summary(int64_t c, int C, int W, int mode) {
  if (mode == EVA_NONCAUSAL) return 0;
  if (mode == EVA_WINDOW_SLIDING) return (c + W / C) * (int64_t)C;
  return (c / (W / C) + 1) * (int64_t)W;
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
// Bits [a, b) of a 32-column group (empty when b <= a).
__device__ __forceinline__ uint32_t range_bits(int a, int b) {
  a = min(max(a, 0), 32);
  b = min(max(b, 0), 32);
  return (uint32_t)(((1ull << b) - 1ull) & ~((1ull << a) - 1ull));
}
template <int BQ> __host__ __device__ __forceinline__ int nqt(int T) { return (T + BQ - 1) / BQ; }
template <int BQ>
__host__ __device__ __forceinline__ int sum_qt0(int s, int T, int C, int W, int mode) {
  const int64_t q = qlo_of_summary((int64_t)s * BK, C, W, mode);
  return q >= T ? nqt<BQ>(T) : (int)(q / BQ);
}
template <int BQ>
__host__ __device__ __forceinline__ int sum_segs(int s, int T, int C, int W, int mode, int SEG) {
  return (nqt<BQ>(T) - sum_qt0<BQ>(s, T, C, W, mode) + SEG - 1) / SEG;
}

// Bulk (non-tensor) reduce-add of `bytes` contiguous fp32 from shared to global memory,
// performed by the TMA unit at L2 (one instruction per 64 x d tile instead of 64 x d REDs).
__device__ __forceinline__ void bulk_reduce_add_f32(float* gdst, const float* ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// 16-byte shared-memory load through the shared window (the arrays live in dynamic shared
// memory reached by a generic pointer, which the compiler would otherwise load with
// generic, serialised LD instructions)
__device__ __forceinline__ float4 lds4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

struct Item {
  bool is_sum;
  int u, k0, nk, qt_begin, nsteps;
};

// Work item w of the linearised (unit, item) list: items [0, n_sum_items) of a unit are
// summary tiles of 128 summaries x SEG query tiles, the rest local tiles of 128 keys.
template <int BQ>
__device__ __forceinline__ Item decode_item(int w, int items_per_unit, int item_base, int n_sum_items, int T,
                                            int C, int W, int mode, int SEG) {
  Item it;
  it.u = w / items_per_unit;
  int item = item_base + w % items_per_unit;
  const int nC = T / C;
  int qt_end;
  if (item < n_sum_items) {
    it.is_sum = true;
    int s = 0;
    for (;; ++s) {
      const int ns = sum_segs<BQ>(s, T, C, W, mode, SEG);
      if (item < ns) break;
      item -= ns;
    }
    it.k0 = s * BK;
    it.nk = min(BK, nC - it.k0);
    it.qt_begin = sum_qt0<BQ>(s, T, C, W, mode) + item * SEG;
    qt_end = min(nqt<BQ>(T), it.qt_begin + SEG);
  } else {
    it.is_sum = false;
    it.k0 = (item - n_sum_items) * BK;
    it.nk = min(BK, T - it.k0);
    it.qt_begin = (int)(qlo_of_key(it.k0, W, mode) / BQ);
    const int64_t qhi = min((int64_t)T - 1, qhi_of_key(it.k0 + it.nk - 1, C, W, mode));
    qt_end = (int)(qhi / BQ) + 1;
  }
  it.nsteps = max(0, qt_end - it.qt_begin);
  return it;
}

// Persistent: one CTA per SM walks work items w = blockIdx.x, + gridDim.x, ...  10 warps:
// 0 TMA producer, 1 TMEM allocator + MMA issuer, 2-5 softmax / dS (thread <-> key row) and
// the item's dK/dV write-out, 6-9 dQ epilogue (thread <-> channel).  Ring stages and barrier
// phases follow a step counter g that runs across items.  Per step the MMA warp issues S(g),
// dP(g), then dQ(g-1) (its dS buffer was written one step earlier), then -- after the
// softmax -- dV(g), dK(g); so the softmax of step g+1 overlaps dQ(g) and its epilogue, and
// the next item's K/V load and first MMAs overlap this item's dK/dV write-out.
__device__ long long g_bwd_trs[5][512];  // debug timeline (EVA_BWD_TRACE)
__device__ int g_bwd_trn[5];

template <int D, bool TRACE>
__global__ void __launch_bounds__(BWD_TC_THREADS, 1)
bwd_main_sm100_kernel(const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mV,
                      const __grid_constant__ CUtensorMap mKs, const __grid_constant__ CUtensorMap mVs,
                      const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mdO,
                      int T, int C, int W, int mode, float scale, float bias2, const float* __restrict__ lse,
                      BwdWsT ws, BwdFused fz, int n_sum_items, int items_per_unit, int item_base, int n_items,
                      int seg, int trace) {
  // debug timeline (EVA_BWD_TRACE=1): CTA 0 records clock64 per role and prints it at exit
  constexpr int TRN = 512;
  auto TR = [&](int role, int code) {
    if constexpr (TRACE) {
      if (trace && blockIdx.x == 0) {
        const int k = atomicAdd(&g_bwd_trn[role], 1);
        if (k < TRN) g_bwd_trs[role][k] = (clock64() << 8) | code;
      }
    }
  };
  using TT = BwdT<D>;
  constexpr int BQ = TT::BQ, NSQ = TT::NSQ;
  constexpr uint32_t TM_S = TT::TM_S, TM_DP = TT::TM_DP, TM_DQ = TT::TM_DQ, TM_DV = TT::TM_DV,
                     TM_DK = TT::TM_DK;
  extern __shared__ uint8_t smem_raw[];
  BwdSm<D>* sm = reinterpret_cast<BwdSm<D>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nC = T / C;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mK); tma_prefetch(&mV); tma_prefetch(&mKs); tma_prefetch(&mVs);
    tma_prefetch(&mQ); tma_prefetch(&mdO);
    for (int b = 0; b < TT::NK; ++b) {
      mbar_init(&sm->k_full[b], 1);
      mbar_init(&sm->k_free[b], 1);
    }
    mbar_init(&sm->v_full, 1);
    mbar_init(&sm->v_free, 1);
    for (int s = 0; s < NSQ; ++s) {
      mbar_init(&sm->q_full[s], 1 + 32);  // the TMA expect_tx + the producer lanes' lse/D stores
      mbar_init(&sm->q_empty[s], 1);
    }
    mbar_init(&sm->s_full, 1);
    mbar_init(&sm->p_full, 128);
    mbar_init(&sm->st_free, 1);
    mbar_init(&sm->dq_full, 1);
    mbar_init(&sm->dq_free, 128);
    mbar_init(&sm->ds_free[0], 1);
    mbar_init(&sm->ds_free[1], 1);
    mbar_init(&sm->acc_done, 1);
    mbar_init(&sm->acc_free, 128);
    mbar_init(&sm->s_free, 128);
    for (int k = 0; k < BwdT<D>::PBUF; ++k) mbar_init(&sm->p_free[k], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(&sm->tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm->tmem_base;
  auto item_of = [&](int w) {
    return decode_item<BQ>(w, items_per_unit, item_base, n_sum_items, T, C, W, mode, seg);
  };
  // dK, dV of a finished key tile: drain the TMEM accumulators, release them, write out.
  // Summary tiles reduce into the fp32 dk~ / dbeta accumulators; local tiles either store
  // fp32 partials (unfused) or apply the summary chain rule and store bf16 (fused).  Called by
  // 128 threads whose warp quarter `quad` owns TMEM lanes [32 quad, 32 quad + 32).
  auto drain = [&](const Item& it, int kcount, int quad) {
    const int r = quad * 32 + lane;
    const uint32_t t_lane = tmem + ((uint32_t)(quad * 32) << 16);
    const int64_t m = (int64_t)it.k0 + r;
    // fused path: the row's chain-rule scalars (w_m, da_m), loaded before the accumulators
    // are ready (the chunk coefficients are read per 8-channel piece below; the producer
    // pulled them into L2 at item start and the last step into L1)
    const bool fused = fz.dK != nullptr && !it.is_sum;
    float wm = 0.f, dam = 0.f;
    if (fused && r < it.nk && m < (int64_t)nC * C) {
      wm = __ldg(fz.w + (size_t)it.u * T + m);
      dam = __ldg(fz.da + (size_t)it.u * T + m);
    }
    mbar_wait(&sm->acc_done, kcount & 1);
    if (r == 0) TR(3, 11);
    tc_fence_after();
#pragma unroll 1
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t kv[32], vv[32];
      tmem_ld32(t_lane + TM_DK + cc * 32, kv);
      tmem_ld32(t_lane + TM_DV + cc * 32, vv);
      tmem_wait_ld();
      if (cc == D / 32 - 1) {
        tc_fence_before();
        mbar_arrive(&sm->acc_free);
      }
      if (fused) {
        // dK_m = s dK_local + da_m (omega_c - k_m) + dkt_c,  dV_m = dV_local + w_m dbeta_c
        const bool ok_row = r < it.nk;
        const bool inc = ok_row && m < (int64_t)nC * C;  // rows of a complete chunk get its terms
        const size_t row = (size_t)it.u * T + (ok_row ? m : 0);
        const size_t crow = ((size_t)it.u * nC + (inc ? m / C : 0)) * D + cc * 32;
        const uint4* kg = reinterpret_cast<const uint4*>(fz.K + row * D + cc * 32);
        uint4* okp = reinterpret_cast<uint4*>(fz.dK + row * D + cc * 32);
        uint4* ovp = reinterpret_cast<uint4*>(fz.dV + row * D + cc * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // 8 channels per 16-byte piece
          const uint4 kr = ok_row ? __ldg(kg + e) : make_uint4(0u, 0u, 0u, 0u);
          const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kr);
          float om[8], dk[8], db[8];
          if (inc) {
            *reinterpret_cast<float4*>(&om[0]) = __ldg(reinterpret_cast<const float4*>(fz.om + crow + 8 * e));
            *reinterpret_cast<float4*>(&om[4]) = __ldg(reinterpret_cast<const float4*>(fz.om + crow + 8 * e + 4));
            *reinterpret_cast<float4*>(&dk[0]) = __ldg(reinterpret_cast<const float4*>(fz.dkt + crow + 8 * e));
            *reinterpret_cast<float4*>(&dk[4]) = __ldg(reinterpret_cast<const float4*>(fz.dkt + crow + 8 * e + 4));
            *reinterpret_cast<float4*>(&db[0]) = __ldg(reinterpret_cast<const float4*>(ws.dVs + crow + 8 * e));
            *reinterpret_cast<float4*>(&db[4]) = __ldg(reinterpret_cast<const float4*>(ws.dVs + crow + 8 * e + 4));
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) om[j] = dk[j] = db[j] = 0.f;
          }
          uint32_t pk[4], pv[4];
#pragma unroll
          for (int j2 = 0; j2 < 4; ++j2) {
            const float2 kf = __bfloat1622float2(k2[j2]);
            const int j = 2 * j2, t = 8 * e + j;
            const float gk0 = scale * __uint_as_float(kv[t]) + dam * (om[j] - kf.x) + dk[j];
            const float gk1 = scale * __uint_as_float(kv[t + 1]) + dam * (om[j + 1] - kf.y) + dk[j + 1];
            pk[j2] = pack2(gk0, gk1);
            pv[j2] = pack2(__uint_as_float(vv[t]) + wm * db[j], __uint_as_float(vv[t + 1]) + wm * db[j + 1]);
          }
          if (ok_row) {
            okp[e] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            ovp[e] = make_uint4(pv[0], pv[1], pv[2], pv[3]);
          }
        }
      } else if (r < it.nk) {
        if (it.is_sum) {
          // summary tiles are split into query segments over several CTAs: vector
          // reductions (red.global.add.v4.f32) into the fp32 accumulators
          float4* dks = reinterpret_cast<float4*>(ws.dKs + ((size_t)it.u * nC + m) * D + cc * 32);
          float4* dvs = reinterpret_cast<float4*>(ws.dVs + ((size_t)it.u * nC + m) * D + cc * 32);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            atomicAdd(dks + e, make_float4(scale * __uint_as_float(kv[4 * e]), scale * __uint_as_float(kv[4 * e + 1]),
                                           scale * __uint_as_float(kv[4 * e + 2]),
                                           scale * __uint_as_float(kv[4 * e + 3])));
            atomicAdd(dvs + e, make_float4(__uint_as_float(vv[4 * e]), __uint_as_float(vv[4 * e + 1]),
                                           __uint_as_float(vv[4 * e + 2]), __uint_as_float(vv[4 * e + 3])));
          }
        } else {
          float4* dkl = reinterpret_cast<float4*>(ws.dK + ((size_t)it.u * T + m) * D + cc * 32);
          float4* dvl = reinterpret_cast<float4*>(ws.dV + ((size_t)it.u * T + m) * D + cc * 32);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            dkl[e] = make_float4(scale * __uint_as_float(kv[4 * e]), scale * __uint_as_float(kv[4 * e + 1]),
                                 scale * __uint_as_float(kv[4 * e + 2]), scale * __uint_as_float(kv[4 * e + 3]));
            dvl[e] = make_float4(__uint_as_float(vv[4 * e]), __uint_as_float(vv[4 * e + 1]),
                                 __uint_as_float(vv[4 * e + 2]), __uint_as_float(vv[4 * e + 3]));
          }
        }
      }
    }
  };


  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    int g = 0, kcount = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const Item it = item_of(w);
      if (it.nsteps == 0) continue;
      const CUtensorMap* mk = it.is_sum ? &mKs : &mK;
      const CUtensorMap* mv = it.is_sum ? &mVs : &mV;
      auto issue_q = [&](int i) {  // Q / dO tiles and lse / D of step i into its ring slot
        const int s = g % NSQ;
        // lse (log2 units) and D of the step's queries: loaded into registers first, so their
        // latency overlaps the wait for the ring slot
        float lv[BQ / 32], dvv[BQ / 32];
        const int n0 = (it.qt_begin + i) * BQ;
#pragma unroll
        for (int k = 0; k < BQ / 32; ++k) {
          const int n = n0 + lane + 32 * k;
          // summary keys carry the logit bias (R16), folded into the row constant
          lv[k] = n < T ? lse[(size_t)it.u * T + n] * 1.4426950408889634f - (it.is_sum ? bias2 : 0.f) : 0.f;
          dvv[k] = n < T ? ws.D[(size_t)it.u * T + n] : 0.f;
        }
        if (g >= NSQ) mbar_wait(&sm->q_empty[s], ((g / NSQ) - 1) & 1);
        if (elect_one()) {
          TR(0, 1);
          mbar_arrive_expect_tx(&sm->q_full[s], 2 * BQ * D * 2);
          for (int kb = 0; kb < D / 64; ++kb) {
            tma_load_3d(sm->q[s] + kb * BQ * 64, &mQ, &sm->q_full[s], kb * 64, n0, it.u);
            tma_load_3d(sm->dO[s] + kb * BQ * 64, &mdO, &sm->q_full[s], kb * 64, n0, it.u);
          }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < BQ / 32; ++k) {  // lse / D into the slot, then arrive
          sm->lse2[s][lane + 32 * k] = lv[k];
          sm->Dq[s][lane + 32 * k] = dvv[k];
        }
        mbar_arrive(&sm->q_full[s]);
        ++g;
      };
      if (fz.dK != nullptr && !it.is_sum && it.k0 < nC * C && elect_one()) {
        // the fused drain's chunk coefficients (omega, dkt, dbeta of the tile's chunks): back
        // into L2 while the item runs
        const int c0 = it.k0 / C, c1 = min(nC - 1, (it.k0 + it.nk - 1) / C);
        const size_t off = ((size_t)it.u * nC + c0) * D;
        const uint32_t bytes = (uint32_t)((c1 - c0 + 1) * D * 4);
        bulk_prefetch_l2(fz.om + off, bytes);
        bulk_prefetch_l2(fz.dkt + off, bytes);
        bulk_prefetch_l2(ws.dVs + off, bytes);
      }
      // V is free once the last item's last dP MMA is done, K only after its last dQ MMA:
      // K of this item (slot kcount % NK); with NK = 2 its slot was freed an item ago, so it
      // goes first and loads under the current item's tail
      constexpr int NK = TT::NK;
      const int kslot = kcount % NK;
      auto issue_k = [&] {
        if (kcount >= NK) mbar_wait(&sm->k_free[kslot], ((kcount / NK) - 1) & 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&sm->k_full[kslot], BK * D * 2);
          for (int kb = 0; kb < D / 64; ++kb)
            tma_load_3d(sm->k[kslot] + kb * BK * 64, mk, &sm->k_full[kslot], kb * 64, it.k0, it.u);
        }
        __syncwarp();
      };
      if (NK > 1) issue_k();
      // V (free once the last item's last dP is done), then the first Q/dO slots (then K when
      // single-buffered: free only after the last item's last dQ)
      if (kcount > 0) mbar_wait(&sm->v_free, (kcount - 1) & 1);
      if (elect_one()) {
        TR(0, 9);
        mbar_arrive_expect_tx(&sm->v_full, BK * D * 2);
        for (int kb = 0; kb < D / 64; ++kb) tma_load_3d(sm->v + kb * BK * 64, mv, &sm->v_full, kb * 64, it.k0, it.u);
      }
      __syncwarp();
      const int npre = it.nsteps < NSQ ? it.nsteps : NSQ;
      for (int i = 0; i < npre; ++i) issue_q(i);
      if (NK == 1) issue_k();
      for (int i = npre; i < it.nsteps; ++i) issue_q(i);
      // the NEXT item's K/V into L2 now -- about NSQ steps before this item ends (its loads can
      // only start once this item's last dP / dQ MMAs are done); earlier prefetches are evicted
      // by the traffic in between.  (No bulk L2 prefetch of later Q/dO tiles: the burst would
      // queue in front of the ring's own loads in the SM's TMA unit.)
      if (w + (int)gridDim.x < n_items && elect_one()) {
        const Item nx = item_of(w + gridDim.x);
        const CUtensorMap* nk = nx.is_sum ? &mKs : &mK;
        const CUtensorMap* nv = nx.is_sum ? &mVs : &mV;
        for (int kb = 0; kb < D / 64; ++kb) {
          tma_prefetch_l2_3d(nk, kb * 64, nx.k0, nx.u);
          tma_prefetch_l2_3d(nv, kb * 64, nx.k0, nx.u);
        }
      }
      __syncwarp();
      ++kcount;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(BK, BQ, false);        // S^T, dP^T
    constexpr uint32_t idesc_g = idesc_bf16_f32(BK, D, true);          // dV, dK (B MN-major)
    // dQ: d = 128 -> dQ^T = K^T dS^T (M = d, N = BQ); d = 64 -> dQ = dS K (M = BQ, N = d);
    // A and B both MN-major, two 64-wide atoms along M 16 KB apart (LBO)
    constexpr uint32_t idesc_q = TT::DQT ? idesc_bf16_f32_ab(D, BQ, true, true)
                                         : idesc_bf16_f32_ab(BQ, D, true, true);
    uint32_t k_addr = smem_u32(sm->k[0]);  // the current item's K slot (set per item)
    const uint32_t v_addr = smem_u32(sm->v);
    auto issue_dq = [&](int j) {  // dQ(j)^T = K^T dS^T(j), global step j
      if (j > 0) mbar_wait(&sm->dq_free, (j - 1) & 1);  // the epilogue has read dQ(j-1)
      tc_fence_after();
      if (elect_one()) {
        const uint32_t ds_addr = smem_u32(sm->ds[j & 1]);
        const uint32_t a_addr = TT::DQT ? k_addr : ds_addr, b_addr = TT::DQT ? ds_addr : k_addr;
#pragma unroll
        for (int ks = 0; ks < BK / 16; ++ks)
          mma_ss(tmem + TM_DQ, smem_desc_sw128(a_addr + ks * 16 * 128, BK * 128, 1024),
                 smem_desc_sw128(b_addr + ks * 16 * 128, BK * 128, 1024), idesc_q, ks > 0 ? 1u : 0u);
        mma_commit(&sm->dq_full);
        mma_commit(&sm->ds_free[j & 1]);
      }
      __syncwarp();
    };
    auto issue_s = [&](int g) {  // S^T(g) = K Q^T, dP^T(g) = V dO^T
      const int s = g % NSQ;
      const uint32_t q_addr = smem_u32(sm->q[s]), do_addr = smem_u32(sm->dO[s]);
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
          mma_ss(tmem + TM_S, smem_desc_sw128(k_addr + kb * (BK * 128) + off, 16, 1024),
                 smem_desc_sw128(q_addr + kb * (BQ * 128) + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
          mma_ss(tmem + TM_DP, smem_desc_sw128(v_addr + kb * (BK * 128) + off, 16, 1024),
                 smem_desc_sw128(do_addr + kb * (BQ * 128) + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
        }
        mma_commit(&sm->s_full);
      }
      __syncwarp();
    };
    if constexpr (TT::PSMEM) {
      // dV(j), dK(j) from P^T / dS^T in shared memory, then dQ(j)
      auto grad_step = [&](int j, int ij, int kc, bool last) {
        const int s = j % NSQ;
        const uint32_t q_addr = smem_u32(sm->q[s]), do_addr = smem_u32(sm->dO[s]);
        const uint32_t p_addr = smem_u32(sm->p[j % TT::PBUF]), ds_addr = smem_u32(sm->ds[j & 1]);
        mbar_wait(&sm->p_full, j & 1);
        if (ij == 0 && kc > 0) mbar_wait(&sm->acc_free, (kc - 1) & 1);  // dK/dV drained
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < BQ / 16; ++ks) {
            const uint32_t acc = (ij > 0 || ks > 0) ? 1u : 0u;
            const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
            mma_ss(tmem + TM_DV, smem_desc_sw128(p_addr + kb * (BK * 128) + off, 16, 1024),
                   smem_desc_sw128(do_addr + ks * 16 * 128, BQ * 128, 1024), idesc_g, acc);
            mma_ss(tmem + TM_DK, smem_desc_sw128(ds_addr + kb * (BK * 128) + off, 16, 1024),
                   smem_desc_sw128(q_addr + ks * 16 * 128, BQ * 128, 1024), idesc_g, acc);
          }
          mma_commit(&sm->q_empty[s]);
          mma_commit(&sm->p_free[j % TT::PBUF]);
          if (last) mma_commit(&sm->acc_done);
        }
        __syncwarp();
        issue_dq(j);
      };
      int g = 0, kcount = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const Item it = item_of(w);
        if (it.nsteps == 0) continue;
        k_addr = smem_u32(sm->k[kcount % TT::NK]);
        mbar_wait(&sm->k_full[kcount % TT::NK], (kcount / TT::NK) & 1);
        mbar_wait(&sm->v_full, kcount & 1);
        if (lane == 0) TR(1, 10);
        for (int i = 0; i < it.nsteps; ++i, ++g) {
          mbar_wait(&sm->q_full[g % NSQ], (g / NSQ) & 1);
          if (g > 0) mbar_wait(&sm->s_free, (g - 1) & 1);  // softmax has loaded S/dP(g-1)
          tc_fence_after();
          if (lane == 0) TR(1, 2);
          issue_s(g);
          if (i == it.nsteps - 1) {  // the item's last dP has been issued: V is free after it
            if (elect_one()) mma_commit(&sm->v_free);
            __syncwarp();
          }
          if (lane == 0) TR(1, 3);
          if (i > 0) grad_step(g - 1, i - 1, kcount, false);
          if (lane == 0) TR(1, 4);
        }
        grad_step(g - 1, it.nsteps - 1, kcount, true);
        if (lane == 0) TR(1, 5);
        if (elect_one()) mma_commit(&sm->k_free[kcount % TT::NK]);  // K smem free once this dQ completes
        __syncwarp();
        ++kcount;
      }
    } else {
    int g = 0, kcount = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const Item it = item_of(w);
      if (it.nsteps == 0) continue;
      k_addr = smem_u32(sm->k[kcount % TT::NK]);
      mbar_wait(&sm->k_full[kcount % TT::NK], (kcount / TT::NK) & 1);
      mbar_wait(&sm->v_full, kcount & 1);
      for (int i = 0; i < it.nsteps; ++i, ++g) {
        const int s = g % NSQ;
        const uint32_t q_addr = smem_u32(sm->q[s]), do_addr = smem_u32(sm->dO[s]);
        mbar_wait(&sm->q_full[s], (g / NSQ) & 1);
        if (g > 0) mbar_wait(&sm->st_free, (g - 1) & 1);  // dV/dK(g-1) have read P^T, dS^T
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
            mma_ss(tmem + TM_S, smem_desc_sw128(k_addr + kb * (BK * 128) + off, 16, 1024),
                   smem_desc_sw128(q_addr + kb * (BQ * 128) + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
          }
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
            mma_ss(tmem + TM_DP, smem_desc_sw128(v_addr + kb * (BK * 128) + off, 16, 1024),
                   smem_desc_sw128(do_addr + kb * (BQ * 128) + off, 16, 1024), idesc_s, ks > 0 ? 1u : 0u);
          }
          mma_commit(&sm->s_full);
          if (i == it.nsteps - 1) mma_commit(&sm->v_free);  // V is free after the last dP
        }
        __syncwarp();
        if (i > 0) issue_dq(g - 1);
        mbar_wait(&sm->p_full, g & 1);
        if (i == 0 && kcount > 0) mbar_wait(&sm->acc_free, (kcount - 1) & 1);  // dK/dV drained
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < BQ / 16; ++ks) {
            const uint32_t acc = (i > 0 || ks > 0) ? 1u : 0u;
            mma_ts(tmem + TM_DV, tmem + TM_S + ks * 8, smem_desc_sw128(do_addr + ks * 16 * 128, BQ * 128, 1024),
                   idesc_g, acc);
            mma_ts(tmem + TM_DK, tmem + TM_DP + ks * 8, smem_desc_sw128(q_addr + ks * 16 * 128, BQ * 128, 1024),
                   idesc_g, acc);
          }
          mma_commit(&sm->q_empty[s]);
          mma_commit(&sm->st_free);
          if (i == it.nsteps - 1) mma_commit(&sm->acc_done);
        }
        __syncwarp();
      }
      issue_dq(g - 1);
      if (elect_one()) mma_commit(&sm->k_free[kcount % TT::NK]);  // K smem free once this dQ completes
      __syncwarp();
      ++kcount;
    }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ softmax / dS (thread <-> key row)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int tc = (warp - 2) * 32 + lane;  // 0..127 among these warps
    const uint32_t t_lane = tmem + ((uint32_t)(quad * 32) << 16);
    const float sl2 = scale * 1.4426950408889634f;
    int g = 0, kcount = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const Item it = item_of(w);
      if (it.nsteps == 0) {  // a local tile no query sees cannot occur; summaries need no zeros
        continue;
      }
      const int u = it.u;
      const int64_t m = (int64_t)it.k0 + r;
      // queries [vq_lo, vq_hi] minus [xq_lo, xq_hi] see this key; the excluded range is the
      // block holding a summary's chunk under the non-causal partition
      int64_t vq_lo = 1, vq_hi = 0, xq_lo = 1, xq_hi = 0;
      if (r < it.nk) {
        if (it.is_sum) {
          vq_lo = qlo_of_summary(m, C, W, mode);
          vq_hi = T - 1;
          if (mode == EVA_NONCAUSAL) {
            xq_lo = (m * C / W) * (int64_t)W;
            xq_hi = xq_lo + W - 1;
          }
        } else {
          vq_lo = qlo_of_key(m, W, mode);
          vq_hi = min((int64_t)T - 1, qhi_of_key(m, C, W, mode));
        }
      }
      for (int i = 0; i < it.nsteps; ++i, ++g) {
        const int n0 = (it.qt_begin + i) * BQ;
        const int b = g & 1;
        mbar_wait(&sm->s_full, g & 1);
        mbar_wait(&sm->q_full[g % NSQ], (g / NSQ) & 1);  // the producer's lse/D stores
        if (tc == 0) TR(2, 6);
        uint32_t vb[BQ / 32];  // visibility of the step's queries, one bit per column
        {
          const int vlo = (int)max((int64_t)-1, min((int64_t)BQ, vq_lo - n0));
          const int vhi = (int)max((int64_t)-1, min((int64_t)BQ, vq_hi + 1 - n0));
          const int xlo = (int)max((int64_t)-1, min((int64_t)BQ, xq_lo - n0));
          const int xhi = (int)max((int64_t)-1, min((int64_t)BQ, xq_hi + 1 - n0));
#pragma unroll
          for (int h = 0; h < BQ / 32; ++h)
            vb[h] = range_bits(vlo - 32 * h, vhi - 32 * h) & ~range_bits(xlo - 32 * h, xhi - 32 * h);
        }
        const float* lse2 = sm->lse2[g % NSQ];
        const float* Dq = sm->Dq[g % NSQ];
        uint8_t* dsrow = reinterpret_cast<uint8_t*>(sm->ds[b]) + r * 128;
        if constexpr (TT::PSMEM) {
          // load S^T / dP^T, release TMEM at once (the next step's MMAs may overwrite it),
          // then P^T and dS^T into shared memory as K-major A operands of the dV/dK MMAs
          tc_fence_after();
          uint32_t sr[BQ], dr[BQ];
#pragma unroll
          for (int h = 0; h < BQ / 32; ++h) {
            tmem_ld32(t_lane + TM_S + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * h]));
            tmem_ld32(t_lane + TM_DP + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(&dr[32 * h]));
          }
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(&sm->s_free);
          constexpr int PB = TT::PBUF;
          if (g >= PB) mbar_wait(&sm->p_free[g % PB], ((g / PB) - 1) & 1);  // dV(g-PB) read it
          if (g >= 2) mbar_wait(&sm->ds_free[b], ((g >> 1) - 1) & 1);      // dK/dQ(g-2) read ds[b]
          uint8_t* prow = reinterpret_cast<uint8_t*>(sm->p[g % PB]) + r * 128;
#pragma unroll
          for (int c16 = 0; c16 < BQ / 8; ++c16) {
            uint32_t pk[4], dk[4];
            float lv[8], dv[8];
            *reinterpret_cast<float4*>(&lv[0]) = lds4(lse2 + 8 * c16);
            *reinterpret_cast<float4*>(&lv[4]) = lds4(lse2 + 8 * c16 + 4);
            *reinterpret_cast<float4*>(&dv[0]) = lds4(Dq + 8 * c16);
            *reinterpret_cast<float4*>(&dv[4]) = lds4(Dq + 8 * c16 + 4);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              float pp[2], gg[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int jj = 2 * c + e, j = 8 * c16 + jj;
                const bool vis = (vb[j >> 5] >> (j & 31)) & 1u;
                pp[e] = vis ? ex2f(fmaf(__uint_as_float(sr[j]), sl2, -lv[jj])) : 0.f;
                gg[e] = pp[e] * (__uint_as_float(dr[j]) - dv[jj]);
              }
              pk[c] = pack2(pp[0], pp[1]);
              dk[c] = pack2(gg[0], gg[1]);
            }
            const int sub = c16 >> 3, cc = c16 & 7;
            const uint32_t off = sub * (BK * 128) + ((cc ^ (r & 7)) * 16);
            *reinterpret_cast<uint4*>(prow + off) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            *reinterpret_cast<uint4*>(dsrow + off) = make_uint4(dk[0], dk[1], dk[2], dk[3]);
          }
          fence_proxy_async_smem();
          mbar_arrive(&sm->p_full);
          if (tc == 0) TR(2, 7);
          continue;
        }
        if (g >= 2) mbar_wait(&sm->ds_free[b], ((g >> 1) - 1) & 1);  // dQ(g-2) has read ds[b]
        tc_fence_after();
        float2 lnext = make_float2(0.f, 0.f), dnext = make_float2(0.f, 0.f);
#pragma unroll
        for (int h = 0; h < BQ / 32; ++h) {
          uint32_t sr[32], dr[32];
          tmem_ld32(t_lane + TM_S + 32 * h, sr);
          tmem_ld32(t_lane + TM_DP + 32 * h, dr);
          tmem_wait_ld();
          uint32_t pk[16], dk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            float p[2], gg[2];
            float2 lv2, dv2;
            if ((c & 1) == 0) {
              const float4 l4 = lds4(lse2 + 32 * h + 2 * c), d4 = lds4(Dq + 32 * h + 2 * c);
              lv2 = make_float2(l4.x, l4.y);
              dv2 = make_float2(d4.x, d4.y);
              lnext = make_float2(l4.z, l4.w);
              dnext = make_float2(d4.z, d4.w);
            } else {
              lv2 = lnext;
              dv2 = dnext;
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int jj = 2 * c + e;
              const bool vis = (vb[h] >> jj) & 1u;
              p[e] = vis ? ex2f(fmaf(__uint_as_float(sr[jj]), sl2, -(e ? lv2.y : lv2.x))) : 0.f;
              gg[e] = p[e] * (__uint_as_float(dr[jj]) - (e ? dv2.y : dv2.x));
            }
            pk[c] = pack2(p[0], p[1]);
            dk[c] = pack2(gg[0], gg[1]);
          }
          tmem_st16(t_lane + TM_S + 16 * h, pk);
          tmem_st16(t_lane + TM_DP + 16 * h, dk);
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int q16 = 4 * h + c4;           // 16-byte chunk of the row (8 queries)
            const int sub = q16 >> 3, c16 = q16 & 7;  // 64-query sub-tile, chunk within it
            uint4 w4;
            w4.x = dk[4 * c4 + 0];
            w4.y = dk[4 * c4 + 1];
            w4.z = dk[4 * c4 + 2];
            w4.w = dk[4 * c4 + 3];
            *reinterpret_cast<uint4*>(dsrow + sub * (BK * 128) + ((c16 ^ (r & 7)) * 16)) = w4;
          }
        }
        fence_proxy_async_smem();
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&sm->p_full);
      }
      ++kcount;
    }
  } else {
    // ------------------------------------------------------------ dQ epilogue (thread <-> channel)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;          // channel
    const int et = (warp - 6) * 32 + lane;   // 0..127 among these warps
    const uint32_t t_lane = tmem + ((uint32_t)(quad * 32) << 16);
    int g = 0, kcount = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const Item it = item_of(w);
      for (int i = 0; i < it.nsteps; ++i, ++g) {
        const int n0 = (it.qt_begin + i) * BQ;
        if (fz.dK != nullptr && !it.is_sum && i == it.nsteps - 1 && r < it.nk) {
          // the fused drain reads this thread's key row, its (w, da) and the chunk
          // coefficients: into L1 one step ahead (they were written a launch ago and are
          // mostly out of L2 by now)
          const int64_t m = (int64_t)it.k0 + r;
          const size_t row = (size_t)it.u * T + m;
          const char* kr = reinterpret_cast<const char*>(fz.K + row * D);
#pragma unroll
          for (int l = 0; l < D * 2 / 128; ++l) prefetch_l1(kr + 128 * l);
          if (m < (int64_t)nC * C) {
            if ((r & 31) == 0) {
              prefetch_l1(fz.w + row);
              prefetch_l1(fz.da + row);
            }
            const size_t crow = ((size_t)it.u * nC + m / C) * D;
            const int l = r % (3 * D / 32);  // one 128-byte line of omega / dkt / dbeta per thread
            const float* base = l < D / 32 ? fz.om : l < D / 16 ? fz.dkt : ws.dVs;
            prefetch_l1(base + crow + 32 * (l % (D / 32)));
          }
        }
        mbar_wait(&sm->dq_full, g & 1);
        if (r == 0) TR(3, 8);
        tc_fence_after();
        uint32_t qv[64];
        tmem_ld32(t_lane + TM_DQ, *reinterpret_cast<uint32_t(*)[32]>(&qv[0]));
        tmem_ld32(t_lane + TM_DQ + 32, *reinterpret_cast<uint32_t(*)[32]>(&qv[32]));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&sm->dq_free);
        if constexpr (!TT::DQT) {
          // d = 64: thread <-> query row n0 + r; its 64 channels go to a padded staging row
          // and are reduce-added by this thread's own 256-byte bulk operation
          bulk_wait_read_all();  // this thread's previous reduce has read its staging row
          float* st = sm->dqs + r * 68;
#pragma unroll
          for (int e = 0; e < 16; ++e)
            *reinterpret_cast<float4*>(st + 4 * e) =
                make_float4(scale * __uint_as_float(qv[4 * e]), scale * __uint_as_float(qv[4 * e + 1]),
                            scale * __uint_as_float(qv[4 * e + 2]), scale * __uint_as_float(qv[4 * e + 3]));
          fence_proxy_async_smem();
          if (n0 + r < T) {
            bulk_reduce_add_f32(ws.dQ + ((size_t)it.u * T + n0 + r) * D, st, (uint32_t)(D * 4));
            tma_store_commit();
          }
          continue;
        }
        // stage dQ [64 queries][d] and reduce-add it into the fp32 accumulator with bulk TMA
        // operations, in two halves of 32 queries through a [32][d] staging buffer (the
        // previous reduce must have finished reading it)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          if (et == 0) bulk_wait_read_all();
          named_bar_sync(2, 128);
          float* st = sm->dqs + r;
#pragma unroll
          for (int j = 0; j < 32; ++j) st[j * D] = scale * __uint_as_float(qv[32 * hf + j]);
          fence_proxy_async_smem();
          named_bar_sync(2, 128);
          if (et == 0) {
            const int nv = min(32, T - n0 - 32 * hf);
            if (nv > 0) {
              bulk_reduce_add_f32(ws.dQ + ((size_t)it.u * T + n0 + 32 * hf) * D, sm->dqs,
                                  (uint32_t)(nv * D * 4));
              tma_store_commit();
            }
          }
        }
      }
      // ---- dK, dV of this key tile (here, so the softmax warps go straight on to the next
      // item): drain TMEM, release it, then write to global
      if (it.nsteps == 0) continue;
      drain(it, kcount, quad);
      ++kcount;
    }
    if (et == 0 || !TT::DQT) bulk_wait_read_all();  // smem may be released once read; the
                                         // global reduction completes asynchronously before grid end
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if (TRACE && trace && blockIdx.x == 0 && threadIdx.x == 0) {
    long long t0 = g_bwd_trs[1][0] >> 8;
    for (int role = 0; role < 4; ++role) {
      for (int k = 0; k < min(g_bwd_trn[role], TRN); ++k)
        printf("TR role=%d ev=%d t=%lld\n", role, (int)(g_bwd_trs[role][k] & 0xff), (g_bwd_trs[role][k] >> 8) - t0);
      g_bwd_trn[role] = 0;
    }
  }
}

}  // namespace

bool backward_sm100_supported(const eva_config& cfg) {
  CUtensorMap probe;
  static const bool have_tma = make_tma_map_bf16(&probe, reinterpret_cast<void*>(0x1000), 1, 128, 128, 64);
  return cfg.dtype == EVA_BF16 && (cfg.d_head == 128 || cfg.d_head == 64) && have_tma;
}

namespace {
// phase: 0 every item (unfused), 1 the summary items only, 2 the local items only (fz set)
template <int D>
cudaError_t launch_bwd_main(const eva_config& cfg, const void* Q, const void* K, const void* V,
                            const void* Ksum, const void* Vsum, const void* dO, const float* lse,
                            const BwdWsT& ws, const BwdFused& fz, int phase, cudaStream_t s) {
  constexpr int BQ = BwdT<D>::BQ;
  const int BH = cfg.bh_count, T = cfg.T, C = cfg.chunk, W = cfg.window, nC = T / C;
  CUtensorMap mK, mV, mKs, mVs, mQ, mdO;
  bool ok = make_tma_map_bf16(&mK, K, BH, T, D, BK) && make_tma_map_bf16(&mV, V, BH, T, D, BK) &&
            make_tma_map_bf16(&mQ, Q, BH, T, D, BQ) && make_tma_map_bf16(&mdO, dO, BH, T, D, BQ);
  if (nC > 0) {
    ok = ok && make_tma_map_bf16(&mKs, Ksum, BH, nC, D, BK) && make_tma_map_bf16(&mVs, Vsum, BH, nC, D, BK);
  } else {
    mKs = mK;
    mVs = mV;
  }
  if (!ok) return cudaErrorInvalidValue;
  // Summary tiles are cut into segments of `seg` query tiles (one work item each; their
  // dK~/dbeta partials meet in fp32 reductions).  Long segments cost fewer item switches and
  // reductions; short ones keep small problems parallel: the longest seg (<= 32) that still
  // leaves >= 4 work items per SM.
  const int n_local_items = (T + BK - 1) / BK;
  static const int seg_max = [] {  // EVA_BWD_SEG: the longest segment (tuning knob, default 32)
    const char* e = getenv("EVA_BWD_SEG");
    const int v = e ? atoi(e) : 32;
    return v >= 1 && v <= 1024 ? v : 32;
  }();
  int seg = seg_max, n_sum_items = 0;
  for (;; seg /= 2) {
    n_sum_items = 0;
    for (int st = 0; st * BK < nC; ++st) n_sum_items += sum_segs<BQ>(st, T, C, W, cfg.mode, seg);
    if (seg <= 4 || (int64_t)(n_sum_items + n_local_items) * BH >= 4 * num_sms()) break;
  }
  const size_t smem = sizeof(BwdSm<D>) + 1024;
  static const bool trace = getenv("EVA_BWD_TRACE") != nullptr;  // debug timeline of CTA 0
  auto kern = trace ? bwd_main_sm100_kernel<D, true> : bwd_main_sm100_kernel<D, false>;
  {
    cudaError_t e = set_smem_attr((const void*)kern, smem);
    if (e != cudaSuccess) return e;
  }
  const int items_per_unit = phase == 1 ? n_sum_items : phase == 2 ? n_local_items : n_sum_items + n_local_items;
  const int item_base = phase == 2 ? n_sum_items : 0;
  const int n_items = items_per_unit * BH;
  if (n_items == 0) return cudaSuccess;
  const int grid = std::max(1, std::min(n_items, num_sms()));
  kern<<<grid, BWD_TC_THREADS, smem, s>>>(mK, mV, mKs, mVs, mQ, mdO, T, C, W, cfg.mode, cfg.scale,
                                          cfg.summary_bias * 1.4426950408889634f, lse, ws, fz, n_sum_items,
                                          items_per_unit, item_base, n_items, seg, trace ? 1 : 0);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_backward_main_sm100(const eva_config& cfg, const void* Q, const void* K, const void* V,
                                       const void* Ksum, const void* Vsum, const void* dO, const float* lse,
                                       float* wsD, float* wsdQ, float* wsdK, float* wsdV, float* wsdKs,
                                       float* wsdVs, const BwdFusedArgs* fused, int phase, cudaStream_t s) {
  const BwdWsT ws{wsD, wsdQ, wsdK, wsdV, wsdKs, wsdVs};
  BwdFused fz{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  if (fused)
    fz = BwdFused{fused->w, fused->da, fused->om, fused->dkt, static_cast<const __nv_bfloat16*>(K),
                  static_cast<__nv_bfloat16*>(fused->dK), static_cast<__nv_bfloat16*>(fused->dV)};
  if (cfg.d_head == 128) return launch_bwd_main<128>(cfg, Q, K, V, Ksum, Vsum, dO, lse, ws, fz, phase, s);
  if (cfg.d_head == 64) return launch_bwd_main<64>(cfg, Q, K, V, Ksum, Vsum, dO, lse, ws, fz, phase, s);
  return cudaErrorInvalidValue;
}

}  // namespace eva
