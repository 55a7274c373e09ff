// backward_simt.cu -- gradient of the FlashEVA prefill (the paper
// trains with it: "forward and backward pass").  For L = sum_n dO_n . o_n:
//
//   attention (Eq.12-14), P_nx = exp(s q_n.key_x - lse_n):
//     D_n = dO_n . o_n,  dS_nx = P_nx (dO_n . val_x - D_n)
//     dq_n = s sum_x dS_nx key_x
//     local key m   : dk_m += s sum_n dS_nm q_n,   dv_m += sum_n P_nm dO_n
//     summary key c : dk~_c = s sum_n dS_nc q_n,   dbeta_c = sum_n P_nc dO_n
//   summaries (Eq.9, Eq.10, Eq.15), chunk c with rows i:
//     w_i = softmax_i(omega.k_i - |k_i|^2/2),  beta = sum_i w_i v_i
//     dv_i += w_i dbeta;  da_i = w_i (dbeta.v_i - dbeta.beta)
//     dk_i += da_i (omega - k_i);  domega = sum_i da_i k_i
//     dk~ += (d omega / d k~) domega   (lambda [|k~+eps| <= clip] as printed, 1 shifted)
//     dk_i += dk~ / C                  (k~ = mean of the chunk's keys)
//
// Three kernels (fp32 arithmetic, cfg.dtype I/O, fp32 workspace):
//   bwd_prep      : D_n = dO_n . o_n; zero the dQ and summary-gradient accumulators.
//   bwd_main      : key-tile-major.  A CTA owns one tile of 64 keys (locals of one tile,
//                   or 64 summaries), keeps its dK/dV in registers and walks the query
//                   tiles that see it (locals: the next W + 64 queries; summaries: a
//                   segment of the queries after the window -- split across CTAs and
//                   combined with fp32 atomics).  Per 64x64 pair: S = Q K^T and
//                   dP = dO V^T as a register-tiled SIMT product from shared memory,
//                   P / dS elementwise, dV += P^T dO, dK += dS^T Q, and dQ += dS K
//                   added to the fp32 accumulator with red.global.add.
//   bwd_finalize  : one CTA per chunk: the summary chain rule above, then dQ, dK, dV
//                   of the chunk's rows are written in cfg.dtype (tail rows are copied).
// bf16 with d in {64, 128} replaces bwd_main with the tcgen05 main pass of
// backward_sm100.cu (fused schedule: summary items, bwd_finalize_reg<COEF> writing the
// chain-rule coefficients, local items applying them, bwd_dq_convert); the SIMT main pass
// serves fp32 and the other head dims.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace eva {

namespace {

constexpr int BT = 64;        // keys per tile, queries per tile
constexpr int BWD_THREADS = 256;

// Queries that see local key m: [local_qlo, local_qhi] (inverse of visible_set).  Causal:
// from m itself to the last query whose window still starts at or before m; non-causal
// (R15): m's whole block of W.
__host__ __device__ __forceinline__ int64_t local_qlo(int64_t m, int W, int mode) {
  return mode == EVA_NONCAUSAL ? (m / W) * (int64_t)W : m;
}
__host__ __device__ __forceinline__ int64_t local_qhi(int64_t m, int C, int W, int mode) {
  if (mode == EVA_WINDOW_SLIDING) return (m / C + W / C) * (int64_t)C - 1;
  return (m / W + 1) * (int64_t)W - 1;
}
// First query that sees summary c: causal c < nsum(n); non-causal every query outside the
// block holding chunk c sees it, so the query walk starts at 0 (the block is masked).
__host__ __device__ __forceinline__ int64_t summary_qlo(int64_t c, int C, int W, int mode) {
  if (mode == EVA_NONCAUSAL) return 0;
  if (mode == EVA_WINDOW_SLIDING) return (c + W / C) * (int64_t)C;
  return (c / (W / C) + 1) * (int64_t)W;
}

struct BwdWs {
  float* D;    // [bh, T]
  float* dQ;   // [bh, T, d]
  float* dK;   // [bh, T, d]  local-attention part
  float* dV;   // [bh, T, d]
  float* dKs;  // [bh, nC, d] d k~ from the attention
  float* dVs;  // [bh, nC, d] d beta
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

BwdWs carve(const eva_config& cfg, void* base) {
  const size_t BH = (size_t)cfg.bh_count, T = (size_t)cfg.T, d = (size_t)cfg.d_head;
  const size_t nC = (size_t)(cfg.T / cfg.chunk);
  char* p = static_cast<char*>(base);
  BwdWs w;
  w.D = reinterpret_cast<float*>(p);   p += align256(BH * T * 4);
  w.dQ = reinterpret_cast<float*>(p);  p += align256(BH * T * d * 4);
  w.dK = reinterpret_cast<float*>(p);  p += align256(BH * T * d * 4);
  w.dV = reinterpret_cast<float*>(p);  p += align256(BH * T * d * 4);
  w.dKs = reinterpret_cast<float*>(p); p += align256(BH * nC * d * 4);
  w.dVs = reinterpret_cast<float*>(p);
  return w;
}

// Query tiles per summary work item (balances the summary CTAs against the local ones).
constexpr int kSumSegTiles = 8;

struct ItemPlan {
  int n_sum_items, n_local_items;
};

__host__ __device__ __forceinline__ int n_qtiles(int T) { return (T + BT - 1) / BT; }

// Summary tile s covers chunks [64 s, 64 s + 64); its query tiles start at the one holding
// the first query that sees chunk 64 s.
__host__ __device__ __forceinline__ int sum_tile_qt0(int s, int T, int C, int W, int mode) {
  const int64_t q = summary_qlo((int64_t)s * BT, C, W, mode);
  return q >= T ? n_qtiles(T) : (int)(q / BT);
}
__host__ __device__ __forceinline__ int sum_tile_segs(int s, int T, int C, int W, int mode) {
  const int nq = n_qtiles(T) - sum_tile_qt0(s, T, C, W, mode);
  return (nq + kSumSegTiles - 1) / kSumSegTiles;
}

ItemPlan plan_items(const eva_config& cfg) {
  const int T = cfg.T, C = cfg.chunk, W = cfg.window, nC = T / C;
  ItemPlan p{0, n_qtiles(T)};
  for (int s = 0; s * BT < nC; ++s) p.n_sum_items += sum_tile_segs(s, T, C, W, cfg.mode);
  return p;
}

// ------------------------------------------------------------------ bwd_prep
// A row is read by TPR = D*sizeof(T)/16 lanes with one 16-byte load of O and of dO each
// (RPW = 32/TPR rows per warp, 4 warps per CTA); every lane zeroes its VEC fp32 accumulator
// entries with 16-byte stores.  Needs D*sizeof(T) >= 16 (d >= 8 bf16 / 4 fp32).
template <typename T, int D>
__global__ void __launch_bounds__(128) bwd_prep_kernel(eva_config cfg, const T* __restrict__ O,
                                                       const T* __restrict__ dO, BwdWs ws) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int TPR = D / VEC < 32 ? D / VEC : 32;
  constexpr int RPW = 32 / TPR;
  constexpr int PER = D / (TPR * VEC);  // 16-byte pieces per lane and row
  const int Tn = cfg.T, nC = Tn / cfg.chunk;
  const int u = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int grp = lane / TPR, gl = lane % TPR;
  const int n = (blockIdx.x * 4 + warp) * RPW + grp;
  const bool ok = n < Tn;
  const size_t row = (size_t)u * Tn + (ok ? n : 0);
  float s = 0.f;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int ch = (k * TPR + gl) * VEC;
    if (ok) {
      float a[VEC], b[VEC];
      unpack16<T>(ldg16_stream(O + row * D + ch), a);
      unpack16<T>(ldg16_stream(dO + row * D + ch), b);
#pragma unroll
      for (int j = 0; j < VEC; ++j) s += a[j] * b[j];
      float4* q = reinterpret_cast<float4*>(ws.dQ + row * D + ch);
#pragma unroll
      for (int j = 0; j < VEC / 4; ++j) q[j] = z;
    }
  }
  s = group_sum<TPR>(s);
  if (ok && gl == 0) ws.D[row] = s;
  if (ok && n < nC) {
    const size_t srow = (size_t)u * nC + n;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int ch = (k * TPR + gl) * VEC;
#pragma unroll
      for (int j = 0; j < VEC / 4; ++j) {
        reinterpret_cast<float4*>(ws.dKs + srow * D + ch)[j] = z;
        reinterpret_cast<float4*>(ws.dVs + srow * D + ch)[j] = z;
      }
    }
  }
}

// ------------------------------------------------------------------ bwd_main
template <int D>
struct MainSmem {
  float Ks[BT][D + 1], Vs[BT][D + 1], Qs[BT][D + 1], dOs[BT][D + 1];
  float Ps[BT][BT + 1], dSs[BT][BT + 1];
  float lse2[BT], Dd[BT];
  int rlo[BT], rhi[BT], rs1[BT], rs2[BT];
};

template <typename T, int D>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    bwd_main_kernel(eva_config cfg, const T* __restrict__ Q, const T* __restrict__ K,
                    const T* __restrict__ V, const T* __restrict__ Ksum, const T* __restrict__ Vsum,
                    const T* __restrict__ dO, const float* __restrict__ lse, BwdWs ws, int n_sum_items) {
  constexpr int CE = D / 16;  // channels per thread in the [64 x D] products (D >= 16)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MainSmem<D>& sm = *reinterpret_cast<MainSmem<D>*>(smem_raw);
  const int Tn = cfg.T, C = cfg.chunk, W = cfg.window, mode = cfg.mode, nC = Tn / C;
  const int u = blockIdx.y;
  const int tid = threadIdx.x;
  const float scale = cfg.scale;
  const float sl2 = scale * 1.4426950408889634f;
  const float bias2 = cfg.summary_bias * 1.4426950408889634f;

  // ---- decode the work item
  bool is_sum;
  int k0, nk, qt_begin, qt_end;
  {
    int item = blockIdx.x;
    if (item < n_sum_items) {
      is_sum = true;
      int s = 0;
      for (;; ++s) {
        const int ns = sum_tile_segs(s, Tn, C, W, mode);
        if (item < ns) break;
        item -= ns;
      }
      k0 = s * BT;
      nk = min(BT, nC - k0);
      const int qt0 = sum_tile_qt0(s, Tn, C, W, mode);
      qt_begin = qt0 + item * kSumSegTiles;
      qt_end = min(n_qtiles(Tn), qt_begin + kSumSegTiles);
    } else {
      is_sum = false;
      const int t = item - n_sum_items;
      k0 = t * BT;
      nk = min(BT, Tn - k0);
      qt_begin = (int)(local_qlo(k0, W, mode) / BT);
      const int64_t qhi = min((int64_t)Tn - 1, local_qhi(k0 + nk - 1, C, W, mode));
      qt_end = (int)(qhi / BT) + 1;
    }
  }
  const T* kb = is_sum ? Ksum + (size_t)u * nC * D : K + (size_t)u * Tn * D;
  const T* vb = is_sum ? Vsum + (size_t)u * nC * D : V + (size_t)u * Tn * D;
  for (int i = tid; i < BT * D; i += BWD_THREADS) {
    const int r = i / D, c = i % D;
    const bool ok = r < nk;
    sm.Ks[r][c] = ok ? Elem<T>::to_f(kb[(size_t)(k0 + r) * D + c]) : 0.f;
    sm.Vs[r][c] = ok ? Elem<T>::to_f(vb[(size_t)(k0 + r) * D + c]) : 0.f;
  }

  const int ty = tid / 16, tx = tid % 16;  // S/dP block: rows ty*4+a, cols tx+16b
  float dk[4][CE], dv[4][CE];
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int e = 0; e < CE; ++e) dk[b][e] = dv[b][e] = 0.f;

  const T* qb = Q + (size_t)u * Tn * D;
  const T* gb = dO + (size_t)u * Tn * D;
  for (int qt = qt_begin; qt < qt_end; ++qt) {
    const int n0 = qt * BT;
    __syncthreads();  // previous tile's readers are done (and the K/V tile is staged)
    for (int i = tid; i < BT * D; i += BWD_THREADS) {
      const int r = i / D, c = i % D;
      const bool ok = n0 + r < Tn;
      sm.Qs[r][c] = ok ? Elem<T>::to_f(qb[(size_t)(n0 + r) * D + c]) : 0.f;
      sm.dOs[r][c] = ok ? Elem<T>::to_f(gb[(size_t)(n0 + r) * D + c]) : 0.f;
    }
    if (tid < BT) {
      const int64_t n = (int64_t)n0 + tid;
      if (n < Tn) {
        const Vis vs = visible_set(n, C, W, mode, Tn);
        sm.rlo[tid] = (int)vs.lo;
        sm.rhi[tid] = (int)vs.hi;
        sm.rs1[tid] = (int)vs.s1;
        sm.rs2[tid] = (int)min(vs.s2, (int64_t)nC);
        // P = exp2(s S log2e + bias log2e - lse log2e) for summary keys (R16): the bias
        // is folded into the per-row constant
        sm.lse2[tid] = lse[(size_t)u * Tn + n] * 1.4426950408889634f - (is_sum ? bias2 : 0.f);
        sm.Dd[tid] = ws.D[(size_t)u * Tn + n];
      } else {
        sm.rlo[tid] = 1 << 30;  // nothing visible
        sm.rhi[tid] = 0;
        sm.rs1[tid] = 0;
        sm.rs2[tid] = 1 << 30;
        sm.lse2[tid] = 0.f;
        sm.Dd[tid] = 0.f;
      }
    }
    __syncthreads();

    // S = Q K^T and dP = dO V^T for rows ty*4+a, cols tx+16b
    {
      float s[4][4], dp[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) s[a][b] = dp[a][b] = 0.f;
#pragma unroll 4
      for (int k = 0; k < D; ++k) {
        float qa[4], ga[4], kk[4], vv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          qa[a] = sm.Qs[ty * 4 + a][k];
          ga[a] = sm.dOs[ty * 4 + a][k];
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          kk[b] = sm.Ks[tx + 16 * b][k];
          vv[b] = sm.Vs[tx + 16 * b][k];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            s[a][b] = fmaf(qa[a], kk[b], s[a][b]);
            dp[a][b] = fmaf(ga[a], vv[b], dp[a][b]);
          }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = ty * 4 + a;
        const int lo = sm.rlo[i], hi = sm.rhi[i], s1 = sm.rs1[i], s2 = sm.rs2[i];
        const float l2 = sm.lse2[i], Dn = sm.Dd[i];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int j = tx + 16 * b;
          const int x = k0 + j;
          const bool vis = j < nk && (is_sum ? (x < s1 || x >= s2) : (x >= lo && x < hi));
          const float p = vis ? exp2f(fmaf(s[a][b], sl2, -l2)) : 0.f;
          sm.Ps[i][j] = p;
          sm.dSs[i][j] = p * (dp[a][b] - Dn);
        }
      }
    }
    __syncthreads();

    // dV += P^T dO, dK += dS^T Q: keys ty*4+b, channels tx+16e
#pragma unroll 2
    for (int i = 0; i < BT; ++i) {
      float pb[4], db[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        pb[b] = sm.Ps[i][ty * 4 + b];
        db[b] = sm.dSs[i][ty * 4 + b];
      }
#pragma unroll
      for (int e = 0; e < CE; ++e) {
        const float g = sm.dOs[i][tx + 16 * e], q = sm.Qs[i][tx + 16 * e];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          dv[b][e] = fmaf(pb[b], g, dv[b][e]);
          dk[b][e] = fmaf(db[b], q, dk[b][e]);
        }
      }
    }

    // dQ += s dS K: rows ty*4+a, channels tx+16e
    {
      float dq[4][CE];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int e = 0; e < CE; ++e) dq[a][e] = 0.f;
#pragma unroll 2
      for (int j = 0; j < BT; ++j) {
        float da[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) da[a] = sm.dSs[ty * 4 + a][j];
#pragma unroll
        for (int e = 0; e < CE; ++e) {
          const float kv = sm.Ks[j][tx + 16 * e];
#pragma unroll
          for (int a = 0; a < 4; ++a) dq[a][e] = fmaf(da[a], kv, dq[a][e]);
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int n = n0 + ty * 4 + a;
        if (n < Tn) {
          float* dst = ws.dQ + ((size_t)u * Tn + n) * D;
#pragma unroll
          for (int e = 0; e < CE; ++e) atomicAdd(dst + tx + 16 * e, scale * dq[a][e]);
        }
      }
    }
  }

  // write the key tile's gradients
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int r = ty * 4 + b;
    if (r >= nk) continue;
    if (is_sum) {
      float* dks = ws.dKs + ((size_t)u * nC + k0 + r) * D;
      float* dvs = ws.dVs + ((size_t)u * nC + k0 + r) * D;
#pragma unroll
      for (int e = 0; e < CE; ++e) {
        atomicAdd(dks + tx + 16 * e, scale * dk[b][e]);
        atomicAdd(dvs + tx + 16 * e, dv[b][e]);
      }
    } else {
      float* dkl = ws.dK + ((size_t)u * Tn + k0 + r) * D;
      float* dvl = ws.dV + ((size_t)u * Tn + k0 + r) * D;
#pragma unroll
      for (int e = 0; e < CE; ++e) {
        dkl[tx + 16 * e] = scale * dk[b][e];
        dvl[tx + 16 * e] = dv[b][e];
      }
    }
  }
}

// ------------------------------------------------------------------ bwd_finalize
// Block x < nC: chunk x (summary chain rule + output of its C rows); x >= nC: tail rows
// [nC*C + (x-nC)*C, ...) that belong to no complete chunk (copy-out only).
template <typename T, int D>
__global__ void __launch_bounds__(128) bwd_finalize_kernel(eva_config cfg, const T* __restrict__ K,
                                                           const T* __restrict__ V,
                                                           const float* __restrict__ eps, BwdWs ws,
                                                           T* __restrict__ dQ, T* __restrict__ dK,
                                                           T* __restrict__ dV) {
  constexpr int CH = (D + 31) / 32;
  const int Tn = cfg.T, C = cfg.chunk, nC = Tn / C;
  const int u = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int bx = blockIdx.x;
  const int r0 = bx * C;
  const int r1 = min(Tn, r0 + C);
  const size_t ub = (size_t)u * Tn;
  if (bx >= nC) {
    for (int r = r0 + warp; r < r1; r += 4) {
      const size_t o = (ub + r) * D;
      for (int j = lane; j < D; j += 32) {
        dQ[o + j] = Elem<T>::from_f(ws.dQ[o + j]);
        dK[o + j] = Elem<T>::from_f(ws.dK[o + j]);
        dV[o + j] = Elem<T>::from_f(ws.dV[o + j]);
      }
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* part = reinterpret_cast<float*>(smem_raw);  // [4][D]
  float* kt = part + 4 * D;
  float* om = kt + D;
  float* beta = om + D;
  float* dbeta = beta + D;
  float* dkt = dbeta + D;
  float* stat = dkt + D;  // [8]
  float* w = stat + 8;    // [C]
  float* da = w + C;      // [C]
  const int c = bx;
  const T* Kc = K + (ub + r0) * D;
  const T* Vc = V + (ub + r0) * D;
  const size_t srow = ((size_t)u * nC + c) * D;

  // k~ = mean of the chunk's keys
  float acc[CH];
#pragma unroll
  for (int e = 0; e < CH; ++e) acc[e] = 0.f;
  for (int r = warp; r < C; r += 4)
#pragma unroll
    for (int e = 0; e < CH; ++e)
      if (lane + 32 * e < D) acc[e] += Elem<T>::to_f(Kc[(size_t)r * D + lane + 32 * e]);
#pragma unroll
  for (int e = 0; e < CH; ++e)
    if (lane + 32 * e < D) part[warp * D + lane + 32 * e] = acc[e];
  __syncthreads();
  if (threadIdx.x < D) {
    const int j = threadIdx.x;
    const float s = part[j] + part[D + j] + part[2 * D + j] + part[3 * D + j];
    const float k_t = s * (1.0f / (float)C);
    const uint32_t bh = (uint32_t)(cfg.bh_begin + u);
    const float e = eps ? eps[((size_t)u * nC + c) * D + j]
                        : philox_normal1(cfg.seed, cfg.layer, bh, (uint32_t)c, (uint32_t)j);
    kt[j] = k_t;
    om[j] = omega_of(k_t, e, cfg);
    dbeta[j] = ws.dVs[srow + j];
    // d omega / d k~ (Eq.15 as printed: lambda inside the clip range, inclusive)
    float g;
    if (cfg.omega_mode == EVA_OMEGA_AS_PRINTED) {
      const float x = k_t + e;
      g = (x >= -cfg.clip && x <= cfg.clip) ? cfg.lambda : 0.f;
    } else {
      g = 1.f;
    }
    dkt[j] = g;  // factor for now; the gradient is assembled below
  }
  __syncthreads();
  // a_i = omega . k_i - |k_i|^2 / 2
  for (int r = warp; r < C; r += 4) {
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int j = lane + 32 * e;
      if (j < D) {
        const float k = Elem<T>::to_f(Kc[(size_t)r * D + j]);
        s += k * (om[j] - 0.5f * k);
      }
    }
    s = warp_sum(s);
    if (lane == 0) w[r] = s;
  }
  __syncthreads();
  if (warp == 0) {
    float m = -INFINITY;
    for (int r = lane; r < C; r += 32) m = fmaxf(m, w[r]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float z = 0.f;
    for (int r = lane; r < C; r += 32) z += __expf(w[r] - m);
    z = warp_sum(z);
    const float iz = 1.f / z;
    for (int r = lane; r < C; r += 32) w[r] = __expf(w[r] - m) * iz;
  }
  __syncthreads();
  // beta = sum_i w_i v_i
#pragma unroll
  for (int e = 0; e < CH; ++e) acc[e] = 0.f;
  for (int r = warp; r < C; r += 4) {
    const float wr = w[r];
#pragma unroll
    for (int e = 0; e < CH; ++e)
      if (lane + 32 * e < D) acc[e] += wr * Elem<T>::to_f(Vc[(size_t)r * D + lane + 32 * e]);
  }
#pragma unroll
  for (int e = 0; e < CH; ++e)
    if (lane + 32 * e < D) part[warp * D + lane + 32 * e] = acc[e];
  __syncthreads();
  if (warp == 0) {
    float s = 0.f;
    for (int j = lane; j < D; j += 32) {
      const float b = part[j] + part[D + j] + part[2 * D + j] + part[3 * D + j];
      beta[j] = b;
      s += b * dbeta[j];
    }
    s = warp_sum(s);
    if (lane == 0) stat[0] = s;  // dbeta . beta
  }
  __syncthreads();
  // da_i = w_i (dbeta . v_i - dbeta . beta); domega = sum_i da_i k_i
  const float dbb = stat[0];
#pragma unroll
  for (int e = 0; e < CH; ++e) acc[e] = 0.f;
  for (int r = warp; r < C; r += 4) {
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int j = lane + 32 * e;
      if (j < D) s += dbeta[j] * Elem<T>::to_f(Vc[(size_t)r * D + j]);
    }
    s = warp_sum(s);
    const float d_a = w[r] * (s - dbb);
    if (lane == 0) da[r] = d_a;
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int j = lane + 32 * e;
      if (j < D) acc[e] += d_a * Elem<T>::to_f(Kc[(size_t)r * D + j]);
    }
  }
#pragma unroll
  for (int e = 0; e < CH; ++e)
    if (lane + 32 * e < D) part[warp * D + lane + 32 * e] = acc[e];
  __syncthreads();
  if (threadIdx.x < D) {
    const int j = threadIdx.x;
    const float dom = part[j] + part[D + j] + part[2 * D + j] + part[3 * D + j];
    dkt[j] = (ws.dKs[srow + j] + dkt[j] * dom) * (1.0f / (float)C);  // d k~ / C
  }
  __syncthreads();
  // rows of the chunk
  for (int r = warp; r < C; r += 4) {
    const size_t o = (ub + r0 + r) * D;
    const float wr = w[r], dar = da[r];
    for (int j = lane; j < D; j += 32) {
      const float k = Elem<T>::to_f(Kc[(size_t)r * D + j]);
      dQ[o + j] = Elem<T>::from_f(ws.dQ[o + j]);
      dV[o + j] = Elem<T>::from_f(ws.dV[o + j] + wr * dbeta[j]);
      dK[o + j] = Elem<T>::from_f(ws.dK[o + j] + dar * (om[j] - k) + dkt[j]);
    }
  }
}

// Register-resident finalize (bf16 with 16-byte rows, C <= 8 rows per lane slot): the same
// chain rule as bwd_finalize_kernel with the chunk's K and V rows loaded once into registers
// (lane mapping of summarize_chunk_reg: a row is read by TPR = D*2/16 lanes, warp w owns row
// slots w*RPW + 4*RPW*i) and every reduction done with group shuffles + one smem merge.
// COEF (the fused path of the tcgen05 main pass): instead of the rows, write the chain-rule
// coefficients the local items apply -- w_i, da_i per row into cf.w / cf.da, omega and
// d k~ / C per chunk into cf.om / cf.dkt (BwdFusedArgs); grid = complete chunks only.
// Projection (Pk != nullptr, NEXT row 4 reading R17: k~ = P_h mean): k~ and omega from P mean,
// and at the end the chunk's total k~ gradient g is mapped back through P (d mean = P^T g,
// spread over the rows as before) and stored with the mean for dP = sum_c g_c mean_c^T
// (bwd_dp_kernel): proj_g / proj_mean [bh, nC, d] fp32.
template <typename T, int D, int NI, bool COEF = false>
__global__ void __launch_bounds__(128, COEF ? 5 : 4) bwd_finalize_reg_kernel(eva_config cfg, const T* __restrict__ K,
                                                               const T* __restrict__ V,
                                                               const float* __restrict__ eps, BwdWs ws,
                                                               T* __restrict__ dQ, T* __restrict__ dK,
                                                               T* __restrict__ dV, BwdFusedArgs cf,
                                                               const float* __restrict__ Pk = nullptr,
                                                               float* __restrict__ proj_g = nullptr,
                                                               float* __restrict__ proj_mean = nullptr) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int TPR = D / VEC;
  constexpr int RPW = 32 / TPR;
  __shared__ float sh_red[4][D];
  __shared__ float sh_om[D], sh_g[D], sh_db[D], sh_dkt[D], sh_mean[D];
  __shared__ float sh_w[8];
  const int Tn = cfg.T, C = cfg.chunk, nC = Tn / C;
  const int u = blockIdx.y, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / TPR, gl = lane % TPR, ch0 = gl * VEC;
  const size_t ub = (size_t)u * Tn;
  if (c >= nC) {  // tail rows that belong to no complete chunk: copy-out only
    const int r0 = c * C, r1 = min(Tn, r0 + C);
    for (int r = r0 + warp; r < r1; r += 4) {
      const size_t o = (ub + r) * D;
      for (int j = lane; j < D; j += 32) {
        dQ[o + j] = Elem<T>::from_f(ws.dQ[o + j]);
        dK[o + j] = Elem<T>::from_f(ws.dK[o + j]);
        dV[o + j] = Elem<T>::from_f(ws.dV[o + j]);
      }
    }
    return;
  }
  const T* Kc = K + (ub + (size_t)c * C) * D;
  const T* Vc = V + (ub + (size_t)c * C) * D;
  const size_t srow = ((size_t)u * nC + c) * D;
  uint4 kx[NI], vx[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = warp * RPW + 4 * RPW * i + grp;
    if (r < C) {
      kx[i] = ldg16_stream(Kc + (size_t)r * D + ch0);
      vx[i] = ldg16_stream(Vc + (size_t)r * D + ch0);
    } else {  // unused slots: zeros (they enter sums with weight 0)
      kx[i] = make_uint4(0u, 0u, 0u, 0u);
      vx[i] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  // the 4 warps' partial column sums over their rows, merged through sh_red
  auto merge_cols = [&](float (&acc)[VEC]) {
#pragma unroll
    for (int o = TPR; o < 32; o <<= 1)
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (grp == 0) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) sh_red[warp][ch0 + j] = acc[j];
    }
  };
  float acc[VEC];
  // ---- k~ = mean of the chunk's keys; omega (Eq.15) and d omega / d k~
#pragma unroll
  for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = warp * RPW + 4 * RPW * i + grp;
    if (r < C) {
      float k[VEC];
      unpack16<T>(kx[i], k);
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] += k[j];
    }
  }
  merge_cols(acc);
  __syncthreads();
  const float* Ph = Pk ? Pk + (size_t)((cfg.bh_begin + u) % cfg.H) * D * D : nullptr;
  if (Ph) {  // the chunk mean first: every projected channel reads all of it
    if (threadIdx.x < D) {
      const int j = threadIdx.x;
      sh_mean[j] = (sh_red[0][j] + sh_red[1][j] + sh_red[2][j] + sh_red[3][j]) * (1.0f / (float)C);
      proj_mean[srow + j] = sh_mean[j];
    }
    __syncthreads();
  }
  if (threadIdx.x < D) {
    const int j = threadIdx.x;
    float kt;
    if (Ph) {
      kt = 0.f;
      for (int l = 0; l < D; ++l) kt = fmaf(__ldg(Ph + (size_t)j * D + l), sh_mean[l], kt);
    } else {
      kt = (sh_red[0][j] + sh_red[1][j] + sh_red[2][j] + sh_red[3][j]) * (1.0f / (float)C);
    }
    const uint32_t bh = (uint32_t)(cfg.bh_begin + u);
    const float e = eps ? eps[srow + j] : philox_normal1(cfg.seed, cfg.layer, bh, (uint32_t)c, (uint32_t)j);
    sh_om[j] = omega_of(kt, e, cfg);
    if (cfg.omega_mode == EVA_OMEGA_AS_PRINTED) {
      const float x = kt + e;
      sh_g[j] = (x >= -cfg.clip && x <= cfg.clip) ? cfg.lambda : 0.f;
    } else {
      sh_g[j] = 1.f;
    }
    sh_db[j] = ws.dVs[srow + j];
  }
  __syncthreads();
  float om[VEC], db[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    om[j] = sh_om[ch0 + j];
    db[j] = sh_db[ch0 + j];
  }
  // ---- a_i = omega . k_i - |k_i|^2 / 2, w = softmax(a) over the chunk
  float w[NI];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = warp * RPW + 4 * RPW * i + grp;
    float part = 0.f;
    if (r < C) {
      float k[VEC];
      unpack16<T>(kx[i], k);
#pragma unroll
      for (int j = 0; j < VEC; ++j) part += k[j] * (om[j] - 0.5f * k[j]);
    }
    part = group_sum<TPR>(part);
    w[i] = r < C ? part : -INFINITY;
    mx = fmaxf(mx, w[i]);
  }
#pragma unroll
  for (int o = TPR; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) sh_w[warp] = mx;
  __syncthreads();
  const float M = fmaxf(fmaxf(sh_w[0], sh_w[1]), fmaxf(sh_w[2], sh_w[3]));
  float z = 0.f;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = warp * RPW + 4 * RPW * i + grp;
    w[i] = r < C ? __expf(w[i] - M) : 0.f;
    if (gl == 0) z += w[i];
  }
  z = warp_sum(z);
  if (lane == 0) sh_w[4 + warp] = z;
  __syncthreads();
  const float iz = 1.f / (sh_w[4] + sh_w[5] + sh_w[6] + sh_w[7]);
  // ---- beta = sum_i w_i v_i; s_i = dbeta . v_i
  float sdv[NI];
#pragma unroll
  for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    w[i] *= iz;
    float v[VEC];
    unpack16<T>(vx[i], v);
    float part = 0.f;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      acc[j] += w[i] * v[j];
      part += db[j] * v[j];
    }
    sdv[i] = group_sum<TPR>(part);
  }
  merge_cols(acc);
  __syncthreads();
  // dbeta . beta (thread ch < D holds beta[ch] * dbeta[ch]; warp sums + smem)
  float bb = 0.f;
  if (threadIdx.x < D) {
    const int j = threadIdx.x;
    bb = (sh_red[0][j] + sh_red[1][j] + sh_red[2][j] + sh_red[3][j]) * sh_db[j];
  }
  bb = warp_sum(bb);
  __syncthreads();  // everyone has read sh_red (beta); sh_w[0..3] is free
  if (lane == 0) sh_w[warp] = bb;
  __syncthreads();
  const float dbb = sh_w[0] + sh_w[1] + sh_w[2] + sh_w[3];
  // ---- da_i = w_i (dbeta . v_i - dbeta . beta); d omega = sum_i da_i k_i
  float da[NI];
#pragma unroll
  for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    da[i] = w[i] * (sdv[i] - dbb);
    float k[VEC];
    unpack16<T>(kx[i], k);
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] += da[i] * k[j];
  }
  merge_cols(acc);
  __syncthreads();
  if (threadIdx.x < D) {
    const int j = threadIdx.x;
    const float dom = sh_red[0][j] + sh_red[1][j] + sh_red[2][j] + sh_red[3][j];
    const float gj = ws.dKs[srow + j] + sh_g[j] * dom;  // total gradient of k~_j
    if (Ph) {
      sh_mean[j] = gj;  // (the mean itself is no longer needed here: stored above)
      proj_g[srow + j] = gj;
    } else {
      sh_dkt[j] = gj * (1.0f / (float)C);  // d k~ / C
    }
  }
  __syncthreads();
  if (Ph) {  // d mean = P^T g, spread over the C rows
    if (threadIdx.x < D) {
      const int l = threadIdx.x;
      float dm = 0.f;
      for (int j = 0; j < D; ++j) dm = fmaf(__ldg(Ph + (size_t)j * D + l), sh_mean[j], dm);
      sh_dkt[l] = dm * (1.0f / (float)C);
    }
    __syncthreads();
  }
  if constexpr (COEF) {
    if (threadIdx.x < D) {
      cf.om[srow + threadIdx.x] = sh_om[threadIdx.x];
      cf.dkt[srow + threadIdx.x] = sh_dkt[threadIdx.x];
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int r = warp * RPW + 4 * RPW * i + grp;
      if (r < C && gl == 0) {
        cf.w[ub + (size_t)c * C + r] = w[i];
        cf.da[ub + (size_t)c * C + r] = da[i];
      }
    }
    return;
  }
  // ---- the chunk's rows
  float dkt[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) dkt[j] = sh_dkt[ch0 + j];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int r = warp * RPW + 4 * RPW * i + grp;
    if (r >= C) continue;
    const size_t o = (ub + (size_t)c * C + r) * D + ch0;
    float k[VEC], q[VEC], gk[VEC], gv[VEC];
    unpack16<T>(kx[i], k);
#pragma unroll
    for (int j = 0; j < VEC; j += 4) {
      const float4 a = *reinterpret_cast<const float4*>(ws.dQ + o + j);
      const float4 b = *reinterpret_cast<const float4*>(ws.dK + o + j);
      const float4 e = *reinterpret_cast<const float4*>(ws.dV + o + j);
      q[j] = a.x; q[j + 1] = a.y; q[j + 2] = a.z; q[j + 3] = a.w;
      gk[j] = b.x; gk[j + 1] = b.y; gk[j + 2] = b.z; gk[j + 3] = b.w;
      gv[j] = e.x; gv[j + 1] = e.y; gv[j + 2] = e.z; gv[j + 3] = e.w;
    }
    T oq[VEC], ok[VEC], ov[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      oq[j] = Elem<T>::from_f(q[j]);
      ov[j] = Elem<T>::from_f(gv[j] + w[i] * db[j]);
      ok[j] = Elem<T>::from_f(gk[j] + da[i] * (om[j] - k[j]) + dkt[j]);
    }
    *reinterpret_cast<uint4*>(dQ + o) = *reinterpret_cast<const uint4*>(oq);
    *reinterpret_cast<uint4*>(dK + o) = *reinterpret_cast<const uint4*>(ok);
    *reinterpret_cast<uint4*>(dV + o) = *reinterpret_cast<const uint4*>(ov);
  }
}

// dP_h = sum over the units u of head h and their chunks c of g_{u,c} mean_{u,c}^T (the learned
// projection's gradient, R17).  Block = one 32 x 32 tile of one head's [D, D]; the (unit, chunk)
// rows are walked in batches of 32 staged in shared memory; 256 threads x 4 outputs.
template <int D>
__global__ void __launch_bounds__(256) bwd_dp_kernel(eva_config cfg, const float* __restrict__ g,
                                                     const float* __restrict__ mean, float* __restrict__ dP) {
  __shared__ float sg[32][33], sm[32][33];
  const int h = blockIdx.z, j0 = blockIdx.y * 32, l0 = blockIdx.x * 32;
  const int nC = cfg.T / cfg.chunk;
  const int tj = threadIdx.x / 8, tl = (threadIdx.x % 8) * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  // units of head h in this shard: u with (bh_begin + u) % H == h
  const int u_first = ((h - cfg.bh_begin) % cfg.H + cfg.H) % cfg.H;
  const int n_units = u_first < cfg.bh_count ? (cfg.bh_count - 1 - u_first) / cfg.H + 1 : 0;
  const int rows = n_units * nC;
  for (int r0 = 0; r0 < rows; r0 += 32) {
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
      const int rr = i / 32, cc = i % 32, r = r0 + rr;
      float gv = 0.f, mv = 0.f;
      if (r < rows) {
        const int u = u_first + (r / nC) * cfg.H, c = r % nC;
        const size_t row = ((size_t)u * nC + c) * D;
        gv = g[row + j0 + cc];
        mv = mean[row + l0 + cc];
      }
      sg[rr][cc] = gv;
      sm[rr][cc] = mv;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const float gv = sg[rr][tj];
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = fmaf(gv, sm[rr][tl + k], acc[k]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) dP[((size_t)h * D + j0 + tj) * D + l0 + tl + k] = acc[k];
}

// dQ of the fused path: the fp32 accumulator to cfg.dtype, 8 elements per thread.
template <typename T>
__global__ void __launch_bounds__(256) bwd_dq_convert_kernel(const float* __restrict__ src, T* __restrict__ dst,
                                                             size_t n8) {
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n8; i += (size_t)gridDim.x * 256) {
    const float4 a = __ldcs(reinterpret_cast<const float4*>(src) + 2 * i);
    const float4 b = __ldcs(reinterpret_cast<const float4*>(src) + 2 * i + 1);
    const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    T o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = Elem<T>::from_f(f[j]);
    if constexpr (sizeof(T) == 2) {
      reinterpret_cast<uint4*>(dst)[i] = *reinterpret_cast<const uint4*>(o);
    } else {
      reinterpret_cast<uint4*>(dst)[2 * i] = *reinterpret_cast<const uint4*>(o);
      reinterpret_cast<uint4*>(dst)[2 * i + 1] = *reinterpret_cast<const uint4*>(o + 4);
    }
  }
}

#define BWD_DISPATCH_D(D_, ...)                               \
  switch (D_) {                                               \
    case 16: { constexpr int D = 16; __VA_ARGS__; } break;    \
    case 32: { constexpr int D = 32; __VA_ARGS__; } break;    \
    case 64: { constexpr int D = 64; __VA_ARGS__; } break;    \
    case 128: { constexpr int D = 128; __VA_ARGS__; } break;  \
    default: return cudaErrorInvalidValue;                    \
  }
#define BWD_DISPATCH_T(dt, ...)                                                 \
  if ((dt) == EVA_BF16) { using T = __nv_bfloat16; __VA_ARGS__; }               \
  else { using T = float; __VA_ARGS__; }

// EVA_BACKWARD_SIMT=1 forces the SIMT main pass for bf16, d = 128 (parity cross-check knob).
bool backward_force_simt() {
  static const bool v = [] {
    const char* e = getenv("EVA_BACKWARD_SIMT");
    return e && atoi(e) != 0;
  }();
  return v;
}
// EVA_BACKWARD_UNFUSED=1 keeps the tcgen05 main pass in one launch with the fp32 dK / dV
// workspace and the finalize kernel (A/B timing and cross-check knob).
bool backward_force_unfused() {
  static const bool v = [] {
    const char* e = getenv("EVA_BACKWARD_UNFUSED");
    return e && atoi(e) != 0;
  }();
  return v;
}
// EVA_BACKWARD_FUSED=1 takes the fused schedule at any size (parity tests of small cases).
bool backward_force_fused() {
  static const bool v = [] {
    const char* e = getenv("EVA_BACKWARD_FUSED");
    return e && atoi(e) != 0;
  }();
  return v;
}

}  // namespace

size_t backward_workspace_bytes(const eva_config& cfg) {
  const size_t BH = (size_t)cfg.bh_count, T = (size_t)cfg.T, d = (size_t)cfg.d_head;
  const size_t nC = (size_t)(cfg.T / cfg.chunk);
  return align256(BH * T * 4) + 3 * align256(BH * T * d * 4) + 2 * align256(BH * nC * d * 4);
}

size_t backward_proj_extra_bytes(const eva_config& cfg) {
  return 2 * align256((size_t)cfg.bh_count * (size_t)(cfg.T / cfg.chunk) * cfg.d_head * 4);
}

bool backward_proj_supported(const eva_config& cfg) {
  const int D = cfg.d_head;
  if (cfg.dtype != EVA_BF16 || (D != 32 && D != 64 && D != 128)) return false;
  const int rpw = 32 / (D * 2 / 16);
  return (cfg.chunk + 4 * rpw - 1) / (4 * rpw) <= 8;  // the register finalize takes the chunk
}

cudaError_t launch_backward(const eva_config& cfg, const void* Q, const void* K, const void* V,
                            const void* Ksum, const void* Vsum, const void* O, const float* lse,
                            const void* dO, const float* eps, void* dQ, void* dK, void* dV,
                            void* workspace, cudaStream_t s, const float* Pk, float* dPk) {
  const BwdWs ws = carve(cfg, workspace);
  // projection: [g | mean] per chunk after the regular workspace
  float* proj_g = nullptr;
  float* proj_mean = nullptr;
  if (Pk) {
    char* extra = static_cast<char*>(workspace) + backward_workspace_bytes(cfg);
    proj_g = reinterpret_cast<float*>(extra);
    proj_mean = reinterpret_cast<float*>(extra + backward_proj_extra_bytes(cfg) / 2);
  }
  const int Tn = cfg.T, C = cfg.chunk, nC = Tn / C;
  const ItemPlan plan = plan_items(cfg);
  cudaError_t err = cudaSuccess;
  BWD_DISPATCH_T(cfg.dtype, BWD_DISPATCH_D(cfg.d_head, {
    {
      constexpr int VEC = 16 / sizeof(T);
      constexpr int RPW = 32 / (D / VEC < 32 ? D / VEC : 32);
      const int rows_per_cta = 4 * RPW;
      bwd_prep_kernel<T, D><<<dim3((Tn + rows_per_cta - 1) / rows_per_cta, cfg.bh_count), 128, 0, s>>>(
          cfg, (const T*)O, (const T*)dO, ws);
    }
    const bool tc = (D == 128 || D == 64) && cfg.dtype == EVA_BF16 && backward_sm100_supported(cfg) &&
                    !backward_force_simt();
    constexpr int RPW_ = 32 / (D * (int)sizeof(T) / 16 > 32 ? 32 : D * (int)sizeof(T) / 16);
    const int ni_ = (C + 4 * RPW_ - 1) / (4 * RPW_);
    // the fused schedule pays two extra launches and a split of the persistent main pass; it
    // wins once the fp32 round trip it removes is large (measured: configs[2] 3.42 -> 3.33 ms,
    // configs[1] 0.063 -> 0.070 ms)
    const bool big = (size_t)cfg.bh_count * (size_t)Tn * D >= ((size_t)1 << 25);
    if (tc && sizeof(T) == 2 && ni_ <= 8 && (big || backward_force_fused()) && !backward_force_unfused()) {
      // fused: summary items -> chain-rule coefficients -> local items writing bf16 dK / dV
      // -> dQ conversion.  The coefficients live in the (then unused) fp32 dK / dV workspace.
      const size_t BH = (size_t)cfg.bh_count;
      BwdFusedArgs cf{ws.dK, ws.dK + BH * Tn, ws.dV, ws.dV + BH * (size_t)nC * D, dK, dV};
      err = launch_backward_main_sm100(cfg, Q, K, V, Ksum, Vsum, dO, lse, ws.D, ws.dQ, ws.dK, ws.dV,
                                       ws.dKs, ws.dVs, nullptr, 1, s);
      if (err != cudaSuccess) return err;
      if (nC > 0) {
        if constexpr (sizeof(T) == 2 && D * sizeof(T) >= 64) {
          auto fn = ni_ <= 2 ? bwd_finalize_reg_kernel<T, D, 2, true>
                             : ni_ <= 4 ? bwd_finalize_reg_kernel<T, D, 4, true> : bwd_finalize_reg_kernel<T, D, 8, true>;
          fn<<<dim3(nC, cfg.bh_count), 128, 0, s>>>(cfg, (const T*)K, (const T*)V, eps, ws, (T*)dQ, (T*)dK,
                                                    (T*)dV, cf, Pk, proj_g, proj_mean);
        }
      }
      err = launch_backward_main_sm100(cfg, Q, K, V, Ksum, Vsum, dO, lse, ws.D, ws.dQ, ws.dK, ws.dV,
                                       ws.dKs, ws.dVs, &cf, 2, s);
      if (err != cudaSuccess) return err;
      const size_t n8 = BH * (size_t)Tn * D / 8;
      const int blocks = (int)std::min<size_t>((n8 + 255) / 256, (size_t)num_sms() * 8);
      bwd_dq_convert_kernel<T><<<std::max(blocks, 1), 256, 0, s>>>(ws.dQ, (T*)dQ, n8);
      if (Pk) {
        if (nC > 0) bwd_dp_kernel<D><<<dim3(D / 32, D / 32, cfg.H), 256, 0, s>>>(cfg, proj_g, proj_mean, dPk);
        else err = cudaMemsetAsync(dPk, 0, (size_t)cfg.H * D * D * 4, s);
        note_launch(1);
      }
      note_launch(3 + (nC > 0 ? 1 : 0) + (plan.n_sum_items > 0 ? 1 : 0));
      return err != cudaSuccess ? err : cudaGetLastError();
    }
    if (tc) {
      err = launch_backward_main_sm100(cfg, Q, K, V, Ksum, Vsum, dO, lse, ws.D, ws.dQ, ws.dK, ws.dV,
                                       ws.dKs, ws.dVs, nullptr, 0, s);
      if (err != cudaSuccess) return err;
    } else {
      const size_t sm = sizeof(MainSmem<D>);
      err = set_smem_attr((const void*)bwd_main_kernel<T, D>, sm);
      if (err != cudaSuccess) return err;
      bwd_main_kernel<T, D><<<dim3(plan.n_sum_items + plan.n_local_items, cfg.bh_count),
                              BWD_THREADS, sm, s>>>(cfg, (const T*)Q, (const T*)K, (const T*)V,
                                                    (const T*)Ksum, (const T*)Vsum, (const T*)dO,
                                                    lse, ws, plan.n_sum_items);
    }
    const int n_tail = (Tn - nC * C + C - 1) / C;
    constexpr int RPW = 32 / (D * (int)sizeof(T) / 16 > 32 ? 32 : D * (int)sizeof(T) / 16);
    const int ni = (C + 4 * RPW - 1) / (4 * RPW);
    if (sizeof(T) == 2 && D * sizeof(T) >= 64 && ni <= 8 && !backward_force_simt()) {
      auto fn = ni <= 2 ? bwd_finalize_reg_kernel<T, D, 2> : ni <= 4 ? bwd_finalize_reg_kernel<T, D, 4>
                                                                     : bwd_finalize_reg_kernel<T, D, 8>;
      fn<<<dim3(nC + n_tail, cfg.bh_count), 128, 0, s>>>(cfg, (const T*)K, (const T*)V, eps, ws, (T*)dQ,
                                                         (T*)dK, (T*)dV, BwdFusedArgs{}, Pk, proj_g, proj_mean);
      if (Pk) {
        if (nC > 0) bwd_dp_kernel<D><<<dim3(D / 32, D / 32, cfg.H), 256, 0, s>>>(cfg, proj_g, proj_mean, dPk);
        else err = cudaMemsetAsync(dPk, 0, (size_t)cfg.H * D * D * 4, s);
        note_launch(1);
        if (err != cudaSuccess) return err;
      }
    } else if (Pk) {
      return cudaErrorNotSupported;  // the projection lives in the register finalize only
    } else {
      const size_t fsm = (size_t)(9 * D + 8 + 2 * C) * sizeof(float);
      err = set_smem_attr((const void*)bwd_finalize_kernel<T, D>, fsm);
      if (err != cudaSuccess) return err;
      bwd_finalize_kernel<T, D><<<dim3(nC + n_tail, cfg.bh_count), 128, fsm, s>>>(
          cfg, (const T*)K, (const T*)V, eps, ws, (T*)dQ, (T*)dK, (T*)dV);
    }
    note_launch(3);
    err = cudaGetLastError();
  }));
  return err;
}

}  // namespace eva
