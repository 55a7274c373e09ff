// summarize_bulk.cu -- bandwidth-shaped chunk summaries for bf16 (the default eva_summarize path
// for d in {64, 128}, C in {16, 32, 64, 128}).
//
// Per chunk c of unit u (Eq.10 reading R1; Eq.15 readings R2, R3; log xi P:49;
// P:92 Eq.9 with S = 1):
//   k~_c    = (1/C) sum_i k_{cC+i}
//   omega_c = lambda * clip(k~_c + eps_c)     (or R3's alternative, cfg.omega_mode)
//   a_i     = omega_c . k_i - |k_i|^2 / 2
//   beta^_c = sum_i softmax(a)_i v_i
//
// Why a separate kernel: the register summariser kernel (summarize_reg_kernel, one 128-thread CTA
// per chunk) loads a whole chunk from global memory into registers and stops streaming while it
// computes; with 105 registers it fits 4 CTAs per SM -- 0.66 of HBM at configs[2] (ncu: 24 %
// warps active, long-scoreboard stalls on the loads).  Here a persistent CTA (grid = SMs x CTAs
// per SM) walks chunks i = blockIdx.x, + gridDim.x, ...; a chunk's C key rows and C value rows
// are each ONE contiguous C*d*2-byte block, brought into shared memory by a single bulk copy
// (cp.async.bulk, mbarrier complete_tx), into NST stages (launch_bulk_t chooses), the summariser
// re-reading its pieces from shared memory -- few registers, so many CTAs per SM keep chunks
// streaming while others compute.  The arithmetic is summarize_chunk_reg's (summarize_reg.cuh) with its
// loads served from shared memory: the summaries are bitwise those of the register kernel, the
// cache append and the decode step.
#include <cuda.h>
#include <cmath>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "launch.h"
#include "sm100.cuh"
#include "summarize_reg.cuh"

namespace eva {
namespace {

using namespace sm100;
constexpr int SB_THREADS = 128;

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct LdShared {
  template <typename P>
  __device__ __forceinline__ uint4 operator()(const P* p) const {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
  }
};

template <int D, int CC, int NST>
struct alignas(128) SumSmem {
  __nv_bfloat16 k[NST][CC * D];
  __nv_bfloat16 v[NST][CC * D];
  uint64_t full[NST];
};

// RoPE of the landed key rows (the summaries of the rotated keys, R18/R19, for
// eva_attn_prefill_rope): theta_j from a host double table; rd a power of two.
struct BulkRope {
  double th[64];
  int rd;
  int style;  // EVA_ROPE_INTERLEAVED / EVA_ROPE_NEOX
};

// Rotate rows [0, C) of a plain row-major [C][D] bf16 tile in shared memory, row r at position
// pos0 + r.  Thread t takes item t % NI (interleaved: the 16-byte piece `item`, 4 pairs;
// half-split: pieces item and item + rd/16, 8 pairs) of rows t / NI + k * (128 / NI); the first
// row's angles in double (reduced mod 2 pi), every next row by the recurrence e^{i step theta_j}.
struct RopeRows {
  float sc[8], ss[8];  // one row-step rotation per pair (the same for every chunk: set once)
  int item, g, rstep, np;
  bool active;
  __device__ __forceinline__ static void angle(double a, float& co, float& si) {
    a -= 6.283185307179586 * rint(a * 0.15915494309189535);
    __sincosf((float)a, &si, &co);
  }
  __device__ __forceinline__ void init(const BulkRope& br, int t) {
    const bool neox = br.style == EVA_ROPE_NEOX;
    const int NI = neox ? br.rd / 16 : br.rd / 8;
    item = t % NI;
    g = t / NI;
    rstep = SB_THREADS / NI;
    np = neox ? 8 : 4;
    active = g < rstep;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < np) angle((double)rstep * br.th[np * item + q], sc[q], ss[q]);
  }
  // Rotate rows [0, C) of a plain row-major [C][D] bf16 tile in shared memory, row r at
  // position pos0 + r: thread t takes item t % NI (interleaved: the 16-byte piece `item`, 4
  // pairs; half-split: pieces item and item + rd/16, 8 pairs) of rows g + k * rstep; the first
  // row's angles in double (reduced mod 2 pi), every next row by the recurrence.
  template <int D>
  __device__ __forceinline__ void run(__nv_bfloat16* tile, int C, int64_t pos0, const BulkRope& br) const {
    if (!active || g >= C) return;
    const bool neox = br.style == EVA_ROPE_NEOX;
    float c[8], sn[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < np) angle((double)(pos0 + g) * br.th[np * item + q], c[q], sn[q]);
    const int cha = 8 * item, chb = cha + br.rd / 2;
    for (int r = g; r < C; r += rstep) {
      uint4* pa = reinterpret_cast<uint4*>(tile + (size_t)r * D + cha);
      if (neox) {
        uint4* pb = reinterpret_cast<uint4*>(tile + (size_t)r * D + chb);
        uint4 xa = *pa, xb = *pb;
        uint32_t* wa = reinterpret_cast<uint32_t*>(&xa);
        uint32_t* wb = reinterpret_cast<uint32_t*>(&xb);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 a2 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&wa[q]));
          const float2 b2 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&wb[q]));
          const int i0 = 2 * q, i1 = 2 * q + 1;
          const __nv_bfloat162 ya = __floats2bfloat162_rn(a2.x * c[i0] - b2.x * sn[i0], a2.y * c[i1] - b2.y * sn[i1]);
          const __nv_bfloat162 yb = __floats2bfloat162_rn(a2.x * sn[i0] + b2.x * c[i0], a2.y * sn[i1] + b2.y * c[i1]);
          wa[q] = *reinterpret_cast<const uint32_t*>(&ya);
          wb[q] = *reinterpret_cast<const uint32_t*>(&yb);
        }
        *pa = xa;
        *pb = xb;
      } else {
        uint4 xa = *pa;
        uint32_t* wa = reinterpret_cast<uint32_t*>(&xa);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 a2 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&wa[q]));
          const __nv_bfloat162 y = __floats2bfloat162_rn(a2.x * c[q] - a2.y * sn[q], a2.x * sn[q] + a2.y * c[q]);
          wa[q] = *reinterpret_cast<const uint32_t*>(&y);
        }
        *pa = xa;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < np) {
          const float cn = c[q] * sc[q] - sn[q] * ss[q];
          sn[q] = sn[q] * sc[q] + c[q] * ss[q];
          c[q] = cn;
        }
      }
    }
  }
};

// debug timeline (eva_debug_trace_prefill with EVA_TRACE_OVERLAP=1): CTA entry / exit globaltimer
__device__ unsigned long long* g_sum_trace = nullptr;

template <int D, int CC, int NST, bool TR = false, bool ROPE = false>
__global__ void __launch_bounds__(SB_THREADS) summarize_bulk_kernel(eva_config cfg, const __nv_bfloat16* __restrict__ K,
                                                                   const __nv_bfloat16* __restrict__ V,
                                                                   const float* __restrict__ eps,
                                                                   __nv_bfloat16* __restrict__ Ksum,
                                                                   __nv_bfloat16* __restrict__ Vsum, int c0,
                                                                   int total, const __grid_constant__ BulkRope br) {
  using S = SumSmem<D, CC, NST>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  constexpr uint32_t BYTES = CC * D * 2;
  const int t = threadIdx.x;
  const int nC = cfg.T / CC;
  if constexpr (TR) {
    if (t == 0 && g_sum_trace && blockIdx.x < 4096) g_sum_trace[2 * blockIdx.x] = globaltimer_ns();
  }
  if (t == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&sm.full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  auto src_row = [&](int i) { return (size_t)(i / nC) * cfg.T + (size_t)(i % nC) * CC; };
  auto issue = [&](int k, int i) {  // chunk i into stage k % NST
    const int s = k % NST;
    mbar_arrive_expect_tx(&sm.full[s], 2 * BYTES);
    bulk_load(sm.k[s], K + src_row(i) * D, BYTES, &sm.full[s]);
    bulk_load(sm.v[s], V + src_row(i) * D, BYTES, &sm.full[s]);
  };
  if (t == 0) {
    for (int k = 0; k < NST; ++k) {
      const int i = blockIdx.x + k * gridDim.x;
      if (i < total) issue(k, i);
    }
  }
  constexpr int NI = summ_reg_ni<__nv_bfloat16, D>(CC);
  auto rowK_of = [](const __nv_bfloat16* base) { return [base](int r) { return base + (size_t)r * D; }; };
  // The chunk's random draws (Eq.15, reading R9) do not depend on its data: generated into shared
  // memory while its bulk copy is in flight (the summariser then reads them like caller eps).
  __shared__ __align__(16) float eps_s[D];
  RopeRows rr;
  if constexpr (ROPE) rr.init(br, t);
  int k = 0;
  for (int i = blockIdx.x; i < total; i += gridDim.x, ++k) {
    const int s = k % NST;
    const int u = i / nC, c = i % nC;
    if (!eps && t < D / 4) {
      const float4 z = philox_normal4(cfg.seed, cfg.layer, (uint32_t)(cfg.bh_begin + u), (uint32_t)(c0 + c), (uint32_t)t);
      *reinterpret_cast<float4*>(&eps_s[4 * t]) = z;
    }
    mbar_wait(&sm.full[s], (k / NST) & 1);
    if constexpr (ROPE) {  // the chunk's keys rotated in place before they are summarised
      rr.template run<D>(sm.k[s], CC, (int64_t)(c0 + c) * CC, br);
      __syncthreads();
    }
    const __nv_bfloat16* Ks = sm.k[s];
    const __nv_bfloat16* Vs = sm.v[s];
    summarize_chunk_reg<__nv_bfloat16, D, NI, decltype(rowK_of(Ks)), decltype(rowK_of(Vs)), NoKXform, LdShared, true>(
        rowK_of(Ks), rowK_of(Vs), CC,
        eps ? eps + ((size_t)u * nC + c) * D : eps_s, (uint32_t)(cfg.bh_begin + u), (uint32_t)(c0 + c), cfg,
        Ksum + ((size_t)u * nC + c) * D, Vsum + ((size_t)u * nC + c) * D, nullptr, NoKXform(), LdShared());
    __syncthreads();  // every thread is done with stage s
    if (t == 0) {     // the chunk NST iterations ahead streams into it now
      const int i2 = i + NST * gridDim.x;
      if (i2 < total) issue(k + NST, i2);
    }
  }
  if constexpr (TR) {
    if (t == 0 && g_sum_trace && blockIdx.x < 4096) g_sum_trace[2 * blockIdx.x + 1] = globaltimer_ns();
  }
}

template <int D, int CC, int NST>
cudaError_t launch_bulk_nst(const eva_config& cfg, const void* K, const void* V, const float* eps, void* Ksum,
                            void* Vsum, int c0, cudaStream_t s, int max_ctas, const BulkRope* br = nullptr) {
  using S = SumSmem<D, CC, NST>;
  const size_t smem = sizeof(S);
  static const bool tr = getenv("EVA_TRACE_OVERLAP") != nullptr;  // debug timeline only
  auto kern = br ? summarize_bulk_kernel<D, CC, NST, false, true>
                 : tr ? summarize_bulk_kernel<D, CC, NST, true> : summarize_bulk_kernel<D, CC, NST>;
  cudaError_t e = set_smem_attr((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SB_THREADS, smem);
  if (e != cudaSuccess) return e;
  const int total = (cfg.T / CC) * cfg.bh_count;
  int grid = std::max(1, std::min(total, std::max(1, per_sm) * num_sms()));
  if (max_ctas > 0) grid = std::min(grid, max_ctas);
  static const int per_sm_cap = [] {  // EVA_SUMM_PER_SM=k: at most k CTAs per SM (measurements)
    const char* e = getenv("EVA_SUMM_PER_SM");
    return e ? atoi(e) : 0;
  }();
  if (per_sm_cap > 0) grid = std::min(grid, per_sm_cap * num_sms());
  e = launch_pdl(kern, dim3(grid), dim3(SB_THREADS), smem, s, cfg, (const __nv_bfloat16*)K,
                 (const __nv_bfloat16*)V, eps, (__nv_bfloat16*)Ksum, (__nv_bfloat16*)Vsum, c0, total,
                 br ? *br : BulkRope{});
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

// Stages per CTA.  The summariser re-reads its pieces from shared memory (~48 registers), so
// shared memory sets the CTAs per SM: one stage (7 CTAs per SM at d = 128, C = 64, chunks
// overlapping ACROSS CTAs) measured 0.203 ms = 0.83 of HBM at configs[2], two stages (3 CTAs,
// overlap within a CTA) 0.252 ms; small launches (< 8 chunks per SM) keep two stages (configs[1]:
// 10.3 vs 11.1 us).  EVA_SUMM_NST = 1 / 2 forces either.
template <int D, int CC>
cudaError_t launch_bulk_t(const eva_config& cfg, const void* K, const void* V, const float* eps, void* Ksum,
                          void* Vsum, int c0, cudaStream_t s, int max_ctas, const BulkRope* br = nullptr) {
  static const int nst_env = [] {
    const char* e = getenv("EVA_SUMM_NST");
    return e ? atoi(e) : 0;
  }();
  const int64_t total = (int64_t)(cfg.T / CC) * cfg.bh_count;
  const int nst = nst_env ? nst_env : (total >= 8LL * num_sms() ? 1 : 2);
  if (nst == 1 || 2 * CC * D * 2 * 2 > 160 * 1024)
    return launch_bulk_nst<D, CC, 1>(cfg, K, V, eps, Ksum, Vsum, c0, s, max_ctas, br);
  return launch_bulk_nst<D, CC, 2>(cfg, K, V, eps, Ksum, Vsum, c0, s, max_ctas, br);
}

}  // namespace

// The summaries of the rotated keys on the bulk summariser (eva_attn_prefill_rope's summaries):
// bf16, d in {64, 128}, C in {16..128}, rotary_dim a power of two (>= 16), else NotSupported.
cudaError_t launch_summarize_bulk_rope(const eva_config& cfg, const eva_rope_params& rp, const void* K,
                                       const void* V, const float* eps, void* Ksum, void* Vsum, cudaStream_t s) {
  if (cfg.bh_count == 0 || cfg.T / cfg.chunk == 0) return cudaSuccess;
  const int rd = rp.rotary_dim ? rp.rotary_dim : cfg.d_head;
  if (!summarize_bulk_supported(cfg) || rd < 16 || (rd & (rd - 1)) != 0 || rd > cfg.d_head)
    return cudaErrorNotSupported;
  BulkRope br{};
  br.rd = rd;
  br.style = rp.style;
  for (int j = 0; j < rd / 2; ++j) br.th[j] = std::exp2(std::log2((double)rp.base) * (-2.0 * (double)j / (double)rd));
#define EVA_BULK_RC(D_)                                                                             \
  switch (cfg.chunk) {                                                                              \
    case 16: return launch_bulk_t<D_, 16>(cfg, K, V, eps, Ksum, Vsum, 0, s, 0, &br);                \
    case 32: return launch_bulk_t<D_, 32>(cfg, K, V, eps, Ksum, Vsum, 0, s, 0, &br);                \
    case 64: return launch_bulk_t<D_, 64>(cfg, K, V, eps, Ksum, Vsum, 0, s, 0, &br);                \
    case 128: return launch_bulk_t<D_, 128>(cfg, K, V, eps, Ksum, Vsum, 0, s, 0, &br);              \
    default: return cudaErrorNotSupported;                                                          \
  }
  if (cfg.d_head == 128) EVA_BULK_RC(128)
  EVA_BULK_RC(64)
#undef EVA_BULK_RC
}

cudaError_t debug_set_summ_trace(unsigned long long* p, cudaStream_t s) {
  return cudaMemcpyToSymbolAsync(g_sum_trace, &p, sizeof(p), 0, cudaMemcpyHostToDevice, s);
}

bool summarize_bulk_supported(const eva_config& cfg) {
  return cfg.dtype == EVA_BF16 && (cfg.d_head == 64 || cfg.d_head == 128) &&
         (cfg.chunk == 16 || cfg.chunk == 32 || cfg.chunk == 64 || cfg.chunk == 128);
}

cudaError_t launch_summarize_bulk(const eva_config& cfg, const void* K, const void* V, const float* eps,
                                  void* Ksum, void* Vsum, int c0, cudaStream_t s, int max_ctas) {
  if (cfg.bh_count == 0 || cfg.T / cfg.chunk == 0) return cudaSuccess;
#define EVA_BULK_C(D_)                                                                 \
  switch (cfg.chunk) {                                                                  \
    case 16: return launch_bulk_t<D_, 16>(cfg, K, V, eps, Ksum, Vsum, c0, s, max_ctas);           \
    case 32: return launch_bulk_t<D_, 32>(cfg, K, V, eps, Ksum, Vsum, c0, s, max_ctas);           \
    case 64: return launch_bulk_t<D_, 64>(cfg, K, V, eps, Ksum, Vsum, c0, s, max_ctas);           \
    case 128: return launch_bulk_t<D_, 128>(cfg, K, V, eps, Ksum, Vsum, c0, s, max_ctas);         \
    default: return cudaErrorNotSupported;                                              \
  }
  if (cfg.d_head == 128) EVA_BULK_C(128)
  if (cfg.d_head == 64) EVA_BULK_C(64)
#undef EVA_BULK_C
  return cudaErrorNotSupported;
}

}  // namespace eva
