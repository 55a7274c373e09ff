// api.cu -- the C ABI of libeva.so (include/eva.h): synchronous argument
// validation, kernel selection and launch on the caller's stream.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>
#include <algorithm>

#include "../../include/eva.h"
#include "../../include/eva_debug.h"
#include "common.cuh"
#include "launch.h"

namespace eva {
static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
}  // namespace eva

namespace {

thread_local std::string g_err;

eva_status fail(eva_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

eva_status ok() {
  g_err.clear();
  return EVA_OK;
}

eva_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return ok();
  return fail(EVA_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool d_supported(int d) { return d == 16 || d == 32 || d == 64 || d == 128; }

// Validation shared by all entry points.  need_T: the call uses cfg.T.
eva_status check_cfg(const eva_config* cfg, bool need_T) {
  if (!cfg) return fail(EVA_ERR_INVALID_ARG, "cfg is NULL");
  if (cfg->B < 1 || cfg->H < 1) return fail(EVA_ERR_INVALID_ARG, "B=%d H=%d must be >= 1", cfg->B, cfg->H);
  const int64_t BH = (int64_t)cfg->B * cfg->H;
  if (cfg->bh_begin < 0 || cfg->bh_count < 0 || (int64_t)cfg->bh_begin + cfg->bh_count > BH)
    return fail(EVA_ERR_INVALID_ARG, "shard [%d, %d+%d) outside [0, B*H=%lld)", cfg->bh_begin,
                cfg->bh_begin, cfg->bh_count, (long long)BH);
  if (need_T && cfg->T < 1) return fail(EVA_ERR_INVALID_ARG, "T=%d must be >= 1", cfg->T);
  if (cfg->d_head < 1) return fail(EVA_ERR_INVALID_ARG, "d_head=%d must be >= 1", cfg->d_head);
  if (cfg->chunk < 1 || cfg->window < 1)
    return fail(EVA_ERR_INVALID_ARG, "chunk=%d window=%d must be >= 1", cfg->chunk, cfg->window);
  if (cfg->window % cfg->chunk != 0)
    return fail(EVA_ERR_INVALID_ARG, "window %d is not a multiple of chunk %d (S:211)", cfg->window,
                cfg->chunk);
  if (cfg->mode != EVA_WINDOW_SLIDING && cfg->mode != EVA_WINDOW_BLOCK && cfg->mode != EVA_NONCAUSAL)
    return fail(EVA_ERR_INVALID_ARG, "mode=%d", cfg->mode);
  if (!std::isfinite(cfg->summary_bias) || cfg->reserved != 0)
    return fail(EVA_ERR_INVALID_ARG, "summary_bias must be finite and reserved 0");
  if (cfg->dtype != EVA_F32 && cfg->dtype != EVA_BF16)
    return fail(EVA_ERR_INVALID_ARG, "dtype=%d", cfg->dtype);
  if (cfg->omega_mode != EVA_OMEGA_AS_PRINTED && cfg->omega_mode != EVA_OMEGA_SHIFTED_NOISE)
    return fail(EVA_ERR_INVALID_ARG, "omega_mode=%d", cfg->omega_mode);
  if (!std::isfinite(cfg->scale) || !std::isfinite(cfg->lambda) || !std::isfinite(cfg->clip) ||
      cfg->clip < 0.f || !(cfg->scale > 0.f))
    return fail(EVA_ERR_INVALID_ARG, "scale must be finite and > 0, lambda finite, clip finite >= 0");
  if (cfg->samples != 1)
    return fail(EVA_ERR_UNSUPPORTED, "samples=%d: only S=1 makes beta query-independent (P:101)",
                cfg->samples);
  if (!d_supported(cfg->d_head))
    return fail(EVA_ERR_UNSUPPORTED, "d_head=%d not in {16,32,64,128}", cfg->d_head);
  return EVA_OK;
}

// Decode, cache and the query-range prefill are causal by construction (R15).
eva_status check_causal(const eva_config* cfg, const char* what) {
  if (cfg->mode == EVA_NONCAUSAL)
    return fail(EVA_ERR_UNSUPPORTED, "%s is causal; EVA_NONCAUSAL applies to the prefill only", what);
  return EVA_OK;
}

eva_status check_ptrs(int n, const void* const* ptrs, const char* const* names) {
  for (int i = 0; i < n; ++i) {
    if (!ptrs[i]) return fail(EVA_ERR_INVALID_ARG, "%s is NULL", names[i]);
    if (!aligned16(ptrs[i])) return fail(EVA_ERR_INVALID_ARG, "%s is not 16-byte aligned", names[i]);
  }
  return EVA_OK;
}

}  // namespace

extern "C" {

void eva_config_default(eva_config* cfg, int32_t B, int32_t H, int32_t T, int32_t d,
                        int32_t chunk, int32_t window) {
  if (!cfg) return;
  cfg->B = B;
  cfg->H = H;
  cfg->bh_begin = 0;
  cfg->bh_count = B * H;
  cfg->T = T;
  cfg->d_head = d;
  cfg->chunk = chunk;
  cfg->window = window;
  cfg->samples = 1;
  cfg->mode = EVA_WINDOW_SLIDING;
  cfg->dtype = EVA_BF16;
  cfg->omega_mode = EVA_OMEGA_AS_PRINTED;
  cfg->scale = d > 0 ? 1.0f / std::sqrt((float)d) : 1.0f;
  cfg->lambda = 0.1f;
  cfg->clip = 1.0f;
  cfg->layer = 0;
  cfg->seed = 1234;
  cfg->summary_bias = 0.f;
  cfg->reserved = 0;
}

eva_status eva_summarize(const eva_config* cfg, const void* K, const void* V, const float* eps,
                         void* Ksum, void* Vsum, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (cfg->bh_count == 0 || cfg->T / cfg->chunk == 0) return ok();
  const void* p[] = {K, V, Ksum, Vsum};
  const char* nm[] = {"K", "V", "Ksum", "Vsum"};
  if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  return cuda_status(eva::launch_summarize(*cfg, K, V, eps, Ksum, Vsum, (cudaStream_t)stream),
                     "eva_summarize");
}

}  // extern "C"

namespace {
// R19: base > 1 finite; rotary_dim 0 (= d) or even, <= d, a multiple of 2 * (16 / elem); style 0/1.
eva_status check_rope(const eva_config* cfg, const eva_rope_params* rp, bool fused_producer) {
  if (!rp) return fail(EVA_ERR_INVALID_ARG, "rope params are NULL");
  if (!(rp->base > 1.f) || !std::isfinite(rp->base))
    return fail(EVA_ERR_INVALID_ARG, "rope base=%g must be finite and > 1", (double)rp->base);
  if (rp->style != EVA_ROPE_INTERLEAVED && rp->style != EVA_ROPE_NEOX)
    return fail(EVA_ERR_INVALID_ARG, "rope style=%d", rp->style);
  if (rp->reserved != 0) return fail(EVA_ERR_INVALID_ARG, "rope reserved must be 0");
  const int rd = rp->rotary_dim ? rp->rotary_dim : cfg->d_head;
  const int vec2 = 2 * (cfg->dtype == EVA_BF16 ? 8 : 4);
  if (rd < 0 || rd > cfg->d_head || rd % vec2 != 0)
    return fail(EVA_ERR_INVALID_ARG, "rotary_dim=%d: needs 0 < rd <= d=%d and rd %% %d == 0", rd, cfg->d_head, vec2);
  if (fused_producer && rp->style == EVA_ROPE_NEOX) {
    const int off = rd / vec2;
    if (off & (off - 1))
      return fail(EVA_ERR_UNSUPPORTED, "half-split rotary_dim=%d: rd / %d must be a power of two in the fused "
                                       "producer", rd, vec2);
  }
  return EVA_OK;
}
}  // namespace

extern "C" {

eva_status eva_rope(const eva_config* cfg, float rope_base, const void* X, void* Y, int64_t pos0,
                    int32_t inverse, eva_stream_t stream) {
  const eva_rope_params rp{rope_base, 0, EVA_ROPE_INTERLEAVED, 0};
  return eva_rope_ex(cfg, &rp, X, Y, pos0, nullptr, inverse, stream);
}

eva_status eva_rope_ex(const eva_config* cfg, const eva_rope_params* rp, const void* X, void* Y, int64_t pos0,
                       const int64_t* pos, int32_t inverse, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if ((st = check_rope(cfg, rp, false)) != EVA_OK) return st;
  if (pos0 < 0) return fail(EVA_ERR_INVALID_ARG, "pos0=%lld", (long long)pos0);
  if (cfg->bh_count == 0 || cfg->T == 0) return ok();
  const void* p[] = {X, Y};
  const char* nm[] = {"X", "Y"};
  if ((st = check_ptrs(2, p, nm)) != EVA_OK) return st;
  if (pos && (reinterpret_cast<uintptr_t>(pos) & 7u)) return fail(EVA_ERR_INVALID_ARG, "pos is not 8-byte aligned");
  return cuda_status(eva::launch_rope(*cfg, *rp, X, Y, pos0, pos, inverse != 0, (cudaStream_t)stream), "eva_rope");
}

eva_status eva_rope_summarize(const eva_config* cfg, float rope_base, const void* Q, const void* K,
                              const void* V, const float* eps, void* Qr, void* Kr, void* Ksum, void* Vsum,
                              eva_stream_t stream) {
  const eva_rope_params rp{rope_base, 0, EVA_ROPE_INTERLEAVED, 0};
  return eva_rope_summarize_ex(cfg, &rp, Q, K, V, eps, Qr, Kr, Ksum, Vsum, stream);
}

eva_status eva_rope_summarize_ex(const eva_config* cfg, const eva_rope_params* rp, const void* Q, const void* K,
                                 const void* V, const float* eps, void* Qr, void* Kr, void* Ksum, void* Vsum,
                                 eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if ((st = check_rope(cfg, rp, true)) != EVA_OK) return st;
  if (cfg->bh_count == 0 || cfg->T == 0) return ok();
  const void* p[] = {Q, K, V, Qr, Kr};
  const char* nm[] = {"Q", "K", "V", "Qr", "Kr"};
  if ((st = check_ptrs(5, p, nm)) != EVA_OK) return st;
  if (cfg->T / cfg->chunk > 0) {
    const void* p2[] = {Ksum, Vsum};
    const char* nm2[] = {"Ksum", "Vsum"};
    if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
  }
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  const cudaError_t e = eva::launch_rope_summarize(*cfg, *rp, Q, K, V, eps, Qr, Kr, Ksum, Vsum, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(EVA_ERR_UNSUPPORTED, "eva_rope_summarize: chunk=%d too long for the register summariser",
                cfg->chunk);
  return cuda_status(e, "eva_rope_summarize");
}

eva_status eva_summarize_proj(const eva_config* cfg, const void* K, const void* V, const float* eps,
                              const float* Pk, void* Ksum, void* Vsum, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (!Pk) return fail(EVA_ERR_INVALID_ARG, "Pk is NULL");
  if (!aligned16(Pk)) return fail(EVA_ERR_INVALID_ARG, "Pk is not 16-byte aligned");
  if (cfg->bh_count == 0 || cfg->T / cfg->chunk == 0) return ok();
  const void* p[] = {K, V, Ksum, Vsum};
  const char* nm[] = {"K", "V", "Ksum", "Vsum"};
  if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  const cudaError_t e = eva::launch_summarize(*cfg, K, V, eps, Ksum, Vsum, (cudaStream_t)stream, 0, Pk);
  if (e == cudaErrorNotSupported)
    return fail(EVA_ERR_UNSUPPORTED, "eva_summarize_proj: chunk=%d too long for the register summariser",
                cfg->chunk);
  return cuda_status(e, "eva_summarize_proj");
}

eva_status eva_attn_prefill(const eva_config* cfg, const void* Q, const void* K, const void* V,
                            void* Ksum, void* Vsum, const float* eps, void* O, float* lse,
                            uint32_t flags, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (flags & ~(EVA_SUMMARIES_PROVIDED | EVA_SUMMARIES_FUSED | EVA_SUMMARIES_SEPARATE | EVA_PREFILL_SIMT |
                EVA_PREFILL_OVERLAP))
    return fail(EVA_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
  const uint32_t sum_flags = flags & (EVA_SUMMARIES_PROVIDED | EVA_SUMMARIES_FUSED | EVA_SUMMARIES_SEPARATE);
  if (sum_flags & (sum_flags - 1))
    return fail(EVA_ERR_INVALID_ARG, "flags 0x%x: at most one of EVA_SUMMARIES_{PROVIDED,FUSED,SEPARATE}", flags);
  if ((flags & EVA_SUMMARIES_FUSED) && (flags & EVA_PREFILL_SIMT))
    return fail(EVA_ERR_INVALID_ARG, "EVA_SUMMARIES_FUSED runs on the tensor-core kernel, not EVA_PREFILL_SIMT");
  if ((flags & EVA_PREFILL_OVERLAP) && !(flags & EVA_SUMMARIES_PROVIDED))
    return fail(EVA_ERR_INVALID_ARG, "EVA_PREFILL_OVERLAP needs EVA_SUMMARIES_PROVIDED");
  if (cfg->mode == EVA_NONCAUSAL && cfg->T % cfg->chunk != 0)
    return fail(EVA_ERR_INVALID_ARG, "non-causal prefill needs T %% C == 0 (T=%d, C=%d; reading R15)", cfg->T,
                cfg->chunk);
  if ((flags & EVA_SUMMARIES_FUSED) && !eva::prefill_fused_supported(*cfg))
    return fail(EVA_ERR_UNSUPPORTED,
                "EVA_SUMMARIES_FUSED: needs bf16, d in {64,128}, a causal mode and C in {16,32,64} "
                "(d=%d C=%d mode=%d)", cfg->d_head, cfg->chunk, cfg->mode);
  if (cfg->bh_count == 0) return ok();
  const void* p[] = {Q, K, V, O};
  const char* nm[] = {"Q", "K", "V", "O"};
  if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
  const bool have_sums = cfg->T / cfg->chunk > 0;
  if (have_sums) {
    const void* p2[] = {Ksum, Vsum};
    const char* nm2[] = {"Ksum", "Vsum"};
    if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
  }
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  if (lse && !aligned16(lse)) return fail(EVA_ERR_INVALID_ARG, "lse is not 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  const bool tc = cfg->dtype == EVA_BF16 && !(flags & EVA_PREFILL_SIMT) &&
                  eva::prefill_sm100_supported(*cfg);
  // In-kernel summaries only when asked for: measured slower than the two launches on B200 at
  // both benchmark shapes ("K-prefill-fused"), so flags 0 keeps them separate.
  const bool fused = have_sums && (flags & EVA_SUMMARIES_FUSED) && tc;
  if (fused) {
    cudaError_t e = eva::launch_prefill_sm100_fused(*cfg, Q, K, V, eps, Ksum, Vsum, O, lse, s);
    if (e == cudaErrorStreamCaptureUnsupported)
      return fail(EVA_ERR_INVALID_ARG, "eva_attn_prefill: the fused-summary workspace for this shape must be "
                                       "allocated before graph capture (eva_prefill_reserve)");
    return cuda_status(e, "eva_attn_prefill(sm100, fused summaries)");
  }
  const uint32_t variant = (flags & EVA_PREFILL_OVERLAP) ? 0x100u : 0u;
  if (have_sums && !(flags & EVA_SUMMARIES_PROVIDED)) {
    // (A capped summariser grid with the prefill's local tiles overlapped on the other SMs was
    // measured slower at configs[1] -- 27.6 us with 74 summariser CTAs, 74.8 us with 16 -- the
    // per-chunk summary latency, not the SM count, bounds that launch.)
    cudaError_t e = eva::launch_summarize(*cfg, K, V, eps, Ksum, Vsum, s);
    if (e != cudaSuccess) return cuda_status(e, "eva_attn_prefill(summaries)");
  }
  // EVA_PREFILL_OVERLAP (caller-asserted): the summarize kernel is the previous grid and Q, K, V
  // predate it, so the prefill may start its local tiles before the summaries are complete.
  const eva::PrefillRange rg = eva::full_range(*cfg);
  cudaError_t e = tc ? eva::launch_prefill_sm100(*cfg, rg, Q, K, V, Ksum, Vsum, O, lse, variant, s)
                     : eva::launch_prefill_simt(*cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
  return cuda_status(e, tc ? "eva_attn_prefill(sm100)" : "eva_attn_prefill(simt)");
}

eva_status eva_attn_prefill_rope(const eva_config* cfg, const eva_rope_params* rp, const void* Q, const void* K,
                                 const void* V, const float* eps, void* Ksum, void* Vsum, void* O, float* lse,
                                 uint32_t flags, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if ((st = check_rope(cfg, rp, true)) != EVA_OK) return st;
  if (flags & ~(EVA_SUMMARIES_PROVIDED | EVA_ROPE_K_ROTATED))
    return fail(EVA_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
  const bool k_rot = (flags & EVA_ROPE_K_ROTATED) != 0;
  if (cfg->mode == EVA_NONCAUSAL && cfg->T % cfg->chunk != 0)
    return fail(EVA_ERR_INVALID_ARG, "non-causal prefill needs T %% C == 0 (T=%d, C=%d; reading R15)", cfg->T,
                cfg->chunk);
  if (!eva::prefill_rope_supported(*cfg, rp->rotary_dim, rp->style))
    return fail(EVA_ERR_UNSUPPORTED,
                "eva_attn_prefill_rope: needs bf16, d in {64,128} and a power-of-two rotary_dim (>= 8 "
                "interleaved, >= 16 half-split); got dtype=%d d=%d rotary_dim=%d style=%d",
                (int)cfg->dtype, cfg->d_head, rp->rotary_dim, rp->style);
  if (cfg->bh_count == 0) return ok();
  const void* p[] = {Q, K, V, O};
  const char* nm[] = {"Q", "K", "V", "O"};
  if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
  const bool have_sums = cfg->T / cfg->chunk > 0;
  if (have_sums) {
    const void* p2[] = {Ksum, Vsum};
    const char* nm2[] = {"Ksum", "Vsum"};
    if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
  }
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  if (lse && !aligned16(lse)) return fail(EVA_ERR_INVALID_ARG, "lse is not 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  if (have_sums && !(flags & EVA_SUMMARIES_PROVIDED) && k_rot) {
    // K holds rotated keys already: the plain summariser gives the summaries of the rotated keys
    const cudaError_t e = eva::launch_summarize(*cfg, K, V, eps, Ksum, Vsum, s);
    if (e != cudaSuccess) return cuda_status(e, "eva_attn_prefill_rope(summaries)");
  } else if (have_sums && !(flags & EVA_SUMMARIES_PROVIDED)) {
    // the summaries of the rotated keys, without writing RoPE(Q) / RoPE(K): the bulk summariser
    // rotating the landed key rows, else the register RoPE summariser
    cudaError_t e = eva::launch_summarize_bulk_rope(*cfg, *rp, K, V, eps, Ksum, Vsum, s);
    if (e == cudaErrorNotSupported)
      e = eva::launch_rope_summarize(*cfg, *rp, Q, K, V, eps, nullptr, nullptr, Ksum, Vsum, s);
    if (e == cudaErrorNotSupported)
      return fail(EVA_ERR_UNSUPPORTED, "eva_attn_prefill_rope: chunk=%d too long for the register summariser",
                  cfg->chunk);
    if (e != cudaSuccess) return cuda_status(e, "eva_attn_prefill_rope(summaries)");
  }
  return cuda_status(eva::launch_prefill_sm100_rope(*cfg, std::log2((double)rp->base), rp->rotary_dim, rp->style,
                                                    Q, K, V, Ksum, Vsum, O, lse, s, k_rot),
                     "eva_attn_prefill_rope");
}

eva_status eva_prefill_reserve(const eva_config* cfg, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (cfg->bh_count == 0 || !eva::prefill_fused_supported(*cfg)) return ok();
  cudaError_t e = eva::prefill_fused_reserve(*cfg, (cudaStream_t)stream);
  if (e == cudaErrorStreamCaptureUnsupported)
    return fail(EVA_ERR_INVALID_ARG, "eva_prefill_reserve: stream is capturing");
  return cuda_status(e, "eva_prefill_reserve");
}

eva_status eva_summarize_range(const eva_config* cfg, int32_t chunk0, const void* K, const void* V,
                               const float* eps, void* Ksum, void* Vsum, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (chunk0 < 0) return fail(EVA_ERR_INVALID_ARG, "chunk0=%d must be >= 0", chunk0);
  if (cfg->bh_count == 0 || cfg->T / cfg->chunk == 0) return ok();
  const void* p[] = {K, V, Ksum, Vsum};
  const char* nm[] = {"K", "V", "Ksum", "Vsum"};
  if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  return cuda_status(eva::launch_summarize(*cfg, K, V, eps, Ksum, Vsum, (cudaStream_t)stream, chunk0),
                     "eva_summarize_range");
}

eva_status eva_summarize_range_bcast(const eva_config* cfg, int32_t chunk0, const void* K, const void* V,
                                     const float* eps, const uint64_t* dst_ksum, const uint64_t* dst_vsum,
                                     int32_t n_dst, int32_t dst_rows, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (chunk0 < 0) return fail(EVA_ERR_INVALID_ARG, "chunk0=%d must be >= 0", chunk0);
  if (n_dst < 0 || n_dst > 64) return fail(EVA_ERR_INVALID_ARG, "n_dst=%d outside [0, 64]", n_dst);
  const int nC = cfg->T / cfg->chunk;
  if (dst_rows < chunk0 + nC)
    return fail(EVA_ERR_INVALID_ARG, "dst_rows=%d < chunk0 + T/C = %d", dst_rows, chunk0 + nC);
  if (cfg->bh_count == 0 || nC == 0 || n_dst == 0) return ok();
  const void* p[] = {K, V, dst_ksum, dst_vsum};
  const char* nm[] = {"K", "V", "dst_ksum", "dst_vsum"};
  if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  cudaError_t e = eva::launch_summarize_bcast(*cfg, chunk0, K, V, eps,
                                              reinterpret_cast<const unsigned long long*>(dst_ksum),
                                              reinterpret_cast<const unsigned long long*>(dst_vsum), n_dst,
                                              dst_rows, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(EVA_ERR_UNSUPPORTED, "chunk %d too large for the broadcasting summariser", cfg->chunk);
  return cuda_status(e, "eva_summarize_range_bcast");
}

eva_status eva_attn_prefill_range(const eva_config* cfg, int64_t q0, int32_t n_q, int64_t k0,
                                  int32_t n_kv, const void* Q, const void* K, const void* V,
                                  const void* Ksum, const void* Vsum, int32_t n_sum, void* O,
                                  float* lse, uint32_t flags, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, false);
  if (st != EVA_OK) return st;
  if ((st = check_causal(cfg, "eva_attn_prefill_range")) != EVA_OK) return st;
  if (flags & ~EVA_PREFILL_SIMT) return fail(EVA_ERR_INVALID_ARG, "flags 0x%x: only EVA_PREFILL_SIMT", flags);
  if (q0 < 0 || n_q < 0 || k0 < 0 || n_kv < 0 || n_sum < 0)
    return fail(EVA_ERR_INVALID_ARG, "q0=%lld n_q=%d k0=%lld n_kv=%d n_sum=%d must be >= 0",
                (long long)q0, n_q, (long long)k0, n_kv, n_sum);
  if (cfg->bh_count == 0 || n_q == 0) return ok();
  const int C = cfg->chunk, W = cfg->window;
  const eva::Range rf = eva::mask_range(q0, C, W, cfg->mode);
  const eva::Range rl = eva::mask_range(q0 + n_q - 1, C, W, cfg->mode);
  if (k0 > rf.lo)
    return fail(EVA_ERR_INVALID_ARG, "k0=%lld > lo(q0)=%lld: the window halo of the first query is missing",
                (long long)k0, (long long)rf.lo);
  if (k0 + n_kv < q0 + n_q)
    return fail(EVA_ERR_INVALID_ARG, "keys end at %lld < last query + 1 = %lld", (long long)(k0 + n_kv),
                (long long)(q0 + n_q));
  if (n_sum < rl.nsum)
    return fail(EVA_ERR_INVALID_ARG, "n_sum=%d < nsum(last query)=%lld", n_sum, (long long)rl.nsum);
  const void* p[] = {Q, K, V, O};
  const char* nm[] = {"Q", "K", "V", "O"};
  if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
  if (n_sum > 0) {
    const void* p2[] = {Ksum, Vsum};
    const char* nm2[] = {"Ksum", "Vsum"};
    if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
  }
  if (lse && !aligned16(lse)) return fail(EVA_ERR_INVALID_ARG, "lse is not 16-byte aligned");
  eva::PrefillRange rg;
  rg.q0 = q0;
  rg.nq = n_q;
  rg.pad0 = 0;
  rg.k0 = k0;
  rg.nkv = n_kv;
  rg.nsl = n_sum;
  cudaStream_t s = (cudaStream_t)stream;
  const bool tc = cfg->dtype == EVA_BF16 && !(flags & EVA_PREFILL_SIMT) && eva::prefill_sm100_supported(*cfg);
  cudaError_t e = tc ? eva::launch_prefill_sm100(*cfg, rg, Q, K, V, Ksum, Vsum, O, lse, 0u, s)
                     : eva::launch_prefill_simt(*cfg, rg, Q, K, V, Ksum, Vsum, O, lse, s);
  return cuda_status(e, tc ? "eva_attn_prefill_range(sm100)" : "eva_attn_prefill_range(simt)");
}

eva_status eva_cache_append(eva_cache* cache, const void* K_new, const void* V_new, int32_t n_new,
                            const float* eps, eva_stream_t stream) {
  if (!cache) return fail(EVA_ERR_INVALID_ARG, "cache is NULL");
  eva_status st = check_cfg(&cache->cfg, false);
  if (st != EVA_OK) return st;
  if ((st = check_causal(&cache->cfg, "the decode cache")) != EVA_OK) return st;
  if (n_new < 1) return fail(EVA_ERR_INVALID_ARG, "n_new=%d must be >= 1", n_new);
  if (cache->pos < 0 || cache->cap_chunks < 0)
    return fail(EVA_ERR_INVALID_ARG, "pos=%lld cap_chunks=%d", (long long)cache->pos, cache->cap_chunks);
  if ((cache->pos + n_new) / cache->cfg.chunk > cache->cap_chunks)
    return fail(EVA_ERR_CAPACITY, "append of %d at pos %lld needs %lld summaries > cap %d", n_new,
                (long long)cache->pos, (long long)((cache->pos + n_new) / cache->cfg.chunk),
                cache->cap_chunks);
  if (cache->cfg.bh_count > 0) {
    const void* p[] = {K_new, V_new, cache->ring_k, cache->ring_v};
    const char* nm[] = {"K_new", "V_new", "ring_k", "ring_v"};
    if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
    if (cache->cap_chunks > 0) {
      const void* p2[] = {cache->sum_k, cache->sum_v};
      const char* nm2[] = {"sum_k", "sum_v"};
      if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
    }
    if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
    cudaError_t e = eva::launch_cache_append(*cache, K_new, V_new, n_new, eps, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "eva_cache_append");
  }
  cache->pos += n_new;
  return ok();
}

eva_status eva_cache_load(eva_cache* cache, const void* K, const void* V, const void* Ksum,
                          const void* Vsum, int32_t n, eva_stream_t stream) {
  if (!cache) return fail(EVA_ERR_INVALID_ARG, "cache is NULL");
  eva_status st = check_cfg(&cache->cfg, false);
  if (st != EVA_OK) return st;
  if ((st = check_causal(&cache->cfg, "the decode cache")) != EVA_OK) return st;
  if (n < 1) return fail(EVA_ERR_INVALID_ARG, "n=%d must be >= 1", n);
  if (cache->pos != 0) return fail(EVA_ERR_INVALID_ARG, "eva_cache_load needs an empty cache (pos=%lld)", (long long)cache->pos);
  const int nC = n / cache->cfg.chunk;
  if (nC > cache->cap_chunks) return fail(EVA_ERR_CAPACITY, "%d summaries > cap %d", nC, cache->cap_chunks);
  if (cache->cfg.bh_count > 0) {
    const void* p[] = {K, V, cache->ring_k, cache->ring_v};
    const char* nm[] = {"K", "V", "ring_k", "ring_v"};
    if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
    // Ksum/Vsum may BE the cache's summary buffers (the summariser wrote them in place, rows =
    // cap_chunks = nC): then only the ring is copied, and the copy does not depend on the summaries
    const bool ak = Ksum == cache->sum_k, av = Vsum == cache->sum_v;
    if (ak != av) return fail(EVA_ERR_INVALID_ARG, "Ksum and Vsum must both alias the cache's summaries or neither");
    if (ak && nC > 0 && cache->cap_chunks != nC)
      return fail(EVA_ERR_INVALID_ARG, "in-place summaries need cap_chunks == n / chunk (%d vs %d)", cache->cap_chunks, nC);
    if (nC > 0) {
      const void* p2[] = {Ksum, Vsum, cache->sum_k, cache->sum_v};
      const char* nm2[] = {"Ksum", "Vsum", "sum_k", "sum_v"};
      if ((st = check_ptrs(4, p2, nm2)) != EVA_OK) return st;
    }
    cudaError_t e = eva::launch_cache_load(*cache, K, V, Ksum, Vsum, n, (cudaStream_t)stream, !ak);
    if (e != cudaSuccess) return cuda_status(e, "eva_cache_load");
  }
  cache->pos = n;
  return ok();
}

size_t eva_decode_workspace_bytes(const eva_cache* cache) {
  if (!cache || cache->pos < 1 || cache->cfg.chunk < 1 || cache->cfg.window < 1 ||
      !d_supported(cache->cfg.d_head))
    return 0;
  const int S = eva::decode_splits(*cache);
  if (S <= 1) return 0;
  // one merge counter per unit (fixed offset, padded to 16 bytes) + the split partials
  // (m, l, acc[d]) per (unit, split)
  return ((size_t)cache->cfg.bh_count + 3) / 4 * 4 * sizeof(unsigned) +
         (size_t)cache->cfg.bh_count * S * (cache->cfg.d_head + 2) * sizeof(float);
}

eva_status eva_attn_decode(const eva_cache* cache, const void* Q, void* O, float* lse,
                           void* workspace, size_t workspace_bytes, eva_stream_t stream) {
  if (!cache) return fail(EVA_ERR_INVALID_ARG, "cache is NULL");
  eva_status st = check_cfg(&cache->cfg, false);
  if (st != EVA_OK) return st;
  if ((st = check_causal(&cache->cfg, "the decode cache")) != EVA_OK) return st;
  if (cache->pos < 1) return fail(EVA_ERR_INVALID_ARG, "decode needs pos >= 1 (pos=%lld)", (long long)cache->pos);
  if (cache->cfg.bh_count == 0) return ok();
  const void* p[] = {Q, O, cache->ring_k, cache->ring_v};
  const char* nm[] = {"Q", "O", "ring_k", "ring_v"};
  if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
  const eva::Range r = eva::mask_range(cache->pos - 1, cache->cfg.chunk, cache->cfg.window, cache->cfg.mode);
  if (r.nsum > 0) {
    if (r.nsum > cache->cap_chunks)
      return fail(EVA_ERR_CAPACITY, "query needs %lld summaries > cap %d", (long long)r.nsum, cache->cap_chunks);
    const void* p2[] = {cache->sum_k, cache->sum_v};
    const char* nm2[] = {"sum_k", "sum_v"};
    if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
  }
  if (lse && !aligned16(lse)) return fail(EVA_ERR_INVALID_ARG, "lse is not 16-byte aligned");
  const int S = eva::decode_splits(*cache);
  const size_t need = eva_decode_workspace_bytes(cache);
  if (need > 0 && (!workspace || workspace_bytes < need))
    return fail(EVA_ERR_INVALID_ARG, "workspace of %zu bytes needed (got %zu)", need, workspace_bytes);
  if (workspace && !aligned16(workspace)) return fail(EVA_ERR_INVALID_ARG, "workspace is not 16-byte aligned");
  return cuda_status(eva::launch_decode(*cache, Q, O, lse, (float*)workspace, S, (cudaStream_t)stream),
                     "eva_attn_decode");
}

eva_status eva_decode_step(eva_cache* cache, const void* Q, const void* K_new, const void* V_new,
                           const float* eps, void* O, float* lse, void* workspace,
                           size_t workspace_bytes, eva_stream_t stream) {
  if (!cache) return fail(EVA_ERR_INVALID_ARG, "cache is NULL");
  eva_status st = check_cfg(&cache->cfg, false);
  if (st != EVA_OK) return st;
  if ((st = check_causal(&cache->cfg, "the decode cache")) != EVA_OK) return st;
  if (cache->pos < 0) return fail(EVA_ERR_INVALID_ARG, "pos=%lld", (long long)cache->pos);
  if ((cache->pos + 1) / cache->cfg.chunk > cache->cap_chunks)
    return fail(EVA_ERR_CAPACITY, "append at pos %lld needs %lld summaries > cap %d", (long long)cache->pos,
                (long long)((cache->pos + 1) / cache->cfg.chunk), cache->cap_chunks);
  if (cache->cfg.bh_count == 0) {
    cache->pos += 1;
    return ok();
  }
  const void* p[] = {Q, K_new, V_new, O, cache->ring_k, cache->ring_v};
  const char* nm[] = {"Q", "K_new", "V_new", "O", "ring_k", "ring_v"};
  if ((st = check_ptrs(6, p, nm)) != EVA_OK) return st;
  if (cache->cap_chunks > 0) {
    const void* p2[] = {cache->sum_k, cache->sum_v};
    const char* nm2[] = {"sum_k", "sum_v"};
    if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
  }
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  if (lse && !aligned16(lse)) return fail(EVA_ERR_INVALID_ARG, "lse is not 16-byte aligned");
  eva_cache after = *cache;
  after.pos += 1;
  const int S = eva::decode_splits(after);
  const size_t need = eva_decode_workspace_bytes(&after);
  if (need > 0 && (!workspace || workspace_bytes < need))
    return fail(EVA_ERR_INVALID_ARG, "workspace of %zu bytes needed (got %zu)", need, workspace_bytes);
  if (workspace && !aligned16(workspace)) return fail(EVA_ERR_INVALID_ARG, "workspace is not 16-byte aligned");
  // A token that completes a chunk needs its chunk summarised (append kernel).  Large
  // batches also take the two-launch path: there the decode is a pure HBM stream and the
  // separate append measured faster (0.478 vs 0.518 ms/token at configs[3]); the fused
  // launch pays off when the step is launch-latency bound (small batch x heads).
  // Every check the decode half needs (lse/workspace alignment and size for pos + 1, the
  // summary capacity) was done above, so nothing is enqueued unless both halves can run.
  if ((cache->pos + 1) % cache->cfg.chunk == 0 || cache->cfg.bh_count >= 1024) {
    st = eva_cache_append(cache, K_new, V_new, 1, eps, stream);
    if (st != EVA_OK) return st;
    return cuda_status(eva::launch_decode(*cache, Q, O, lse, (float*)workspace, S, (cudaStream_t)stream),
                       "eva_decode_step");
  }
  cudaError_t e = eva::launch_decode_step(after, Q, K_new, V_new, O, lse, (float*)workspace, S,
                                          (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "eva_decode_step");
  cache->pos += 1;
  return ok();
}

// Ragged decode (per-unit positions): the split count is chosen for the longest position the
// cache can hold, so it is valid for every unit whatever its position.
static eva_cache ragged_bound(const eva_cache* cache) {
  eva_cache b = *cache;
  b.pos = (int64_t)cache->cap_chunks * cache->cfg.chunk + cache->cfg.chunk - 1;
  if (b.pos < 1) b.pos = 1;
  return b;
}

size_t eva_decode_ragged_workspace_bytes(const eva_cache* cache) {
  if (!cache || cache->cap_chunks < 0) return 0;
  const eva_cache b = ragged_bound(cache);
  return eva_decode_workspace_bytes(&b);
}

eva_status eva_decode_step_ragged(const eva_cache* cache, int64_t* pos, const void* Q, const void* K_new,
                                  const void* V_new, const float* eps, void* O, float* lse, void* workspace,
                                  size_t workspace_bytes, eva_stream_t stream) {
  return eva_decode_step_ragged_rope(cache, pos, nullptr, Q, K_new, V_new, eps, O, lse, workspace, workspace_bytes,
                                     stream);
}

eva_status eva_decode_step_ragged_rope(const eva_cache* cache, int64_t* pos, const eva_rope_params* rp,
                                       const void* Q, const void* K_new, const void* V_new, const float* eps,
                                       void* O, float* lse, void* workspace, size_t workspace_bytes,
                                       eva_stream_t stream) {
  if (!cache) return fail(EVA_ERR_INVALID_ARG, "cache is NULL");
  eva_status st = check_cfg(&cache->cfg, false);
  if (st != EVA_OK) return st;
  if (rp && (st = check_rope(&cache->cfg, rp, true)) != EVA_OK) return st;
  if ((st = check_causal(&cache->cfg, "the decode cache")) != EVA_OK) return st;
  if (cache->cap_chunks < 0) return fail(EVA_ERR_INVALID_ARG, "cap_chunks=%d", cache->cap_chunks);
  // one launch (the decode kernel appends and summarises with its first warp); the
  // two-launch form (append kernel with the register summariser, then decode) stays behind
  // EVA_RAGGED_TWO_LAUNCH=1 for A/B timing
  static const bool two_launch = [] {
    const char* e = getenv("EVA_RAGGED_TWO_LAUNCH");
    return e && atoi(e) != 0;
  }();
  // (RoPE is folded into the one-launch form only: with rp the step is always one launch)
  if (two_launch && !rp && !eva::ragged_supported(cache->cfg))
    return fail(EVA_ERR_UNSUPPORTED, "eva_decode_step_ragged: chunk=%d too long for the register summariser",
                cache->cfg.chunk);
  if (cache->cfg.bh_count == 0) return ok();
  if (!pos || (reinterpret_cast<uintptr_t>(pos) & 7u))
    return fail(EVA_ERR_INVALID_ARG, "pos is NULL or not 8-byte aligned");
  const void* p[] = {Q, K_new, V_new, O, cache->ring_k, cache->ring_v};
  const char* nm[] = {"Q", "K_new", "V_new", "O", "ring_k", "ring_v"};
  if ((st = check_ptrs(6, p, nm)) != EVA_OK) return st;
  if (cache->cap_chunks > 0) {
    const void* p2[] = {cache->sum_k, cache->sum_v};
    const char* nm2[] = {"sum_k", "sum_v"};
    if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
  }
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  const eva_cache b = ragged_bound(cache);
  const int S = eva::decode_splits(b);
  const size_t need = eva_decode_workspace_bytes(&b);
  if (need > 0 && (!workspace || workspace_bytes < need))
    return fail(EVA_ERR_INVALID_ARG, "workspace of %zu bytes needed (got %zu)", need, workspace_bytes);
  if (workspace && !aligned16(workspace)) return fail(EVA_ERR_INVALID_ARG, "workspace is not 16-byte aligned");
  const cudaError_t e =
      (two_launch && !rp)
          ? eva::launch_decode_step_ragged(*cache, pos, Q, K_new, V_new, eps, O, lse, (float*)workspace, S,
                                           (cudaStream_t)stream)
          : eva::launch_decode_step_ragged_fused(*cache, pos, Q, K_new, V_new, eps, O, lse, (float*)workspace, S,
                                                 (cudaStream_t)stream, rp);
  return cuda_status(e, rp ? "eva_decode_step_ragged_rope" : "eva_decode_step_ragged");
}

}  // extern "C"

// ------------------------------------------------------------------ host-copy pipeline
struct eva_pipeline {
  int max_slices = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<cudaEvent_t> in, done;  // per slice: H2D complete, kernels complete
};

namespace {
void pipeline_free(eva_pipeline* p) {
  if (!p) return;
  for (cudaEvent_t e : p->in) if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : p->done) if (e) cudaEventDestroy(e);
  if (p->fork) cudaEventDestroy(p->fork);
  if (p->join) cudaEventDestroy(p->join);
  if (p->h2d) cudaStreamDestroy(p->h2d);
  if (p->d2h) cudaStreamDestroy(p->d2h);
  delete p;
}
}  // namespace

extern "C" {

eva_status eva_pipeline_create(int32_t max_slices, eva_pipeline** out) {
  if (!out) return fail(EVA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (max_slices < 1 || max_slices > 4096) return fail(EVA_ERR_INVALID_ARG, "max_slices=%d", max_slices);
  eva_pipeline* p = new eva_pipeline;
  p->max_slices = max_slices;
  p->in.assign(max_slices, nullptr);
  p->done.assign(max_slices, nullptr);
  cudaError_t e = cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->join, cudaEventDisableTiming);
  for (int i = 0; i < max_slices && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&p->in[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->done[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    pipeline_free(p);
    return cuda_status(e, "eva_pipeline_create");
  }
  *out = p;
  return ok();
}

void eva_pipeline_destroy(eva_pipeline* pipe) { pipeline_free(pipe); }

eva_status eva_attn_prefill_host(eva_pipeline* pipe, const eva_config* cfg, const void* hQ,
                                 const void* hK, const void* hV, void* hO, float* hlse, void* dQ,
                                 void* dK, void* dV, void* dKsum, void* dVsum, void* dO, float* dlse,
                                 const float* eps, uint32_t flags, int32_t n_slices,
                                 eva_stream_t stream) {
  if (!pipe) return fail(EVA_ERR_INVALID_ARG, "pipe is NULL");
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (flags & EVA_SUMMARIES_PROVIDED)
    return fail(EVA_ERR_INVALID_ARG, "eva_attn_prefill_host always computes the summaries");
  if (n_slices < 1 || n_slices > pipe->max_slices)
    return fail(EVA_ERR_INVALID_ARG, "n_slices=%d outside [1, %d]", n_slices, pipe->max_slices);
  if (cfg->bh_count == 0) return ok();
  const void* hp[] = {hQ, hK, hV, hO};
  const char* hn[] = {"hQ", "hK", "hV", "hO"};
  for (int i = 0; i < 4; ++i)
    if (!hp[i]) return fail(EVA_ERR_INVALID_ARG, "%s is NULL", hn[i]);
  if (hlse && !dlse) return fail(EVA_ERR_INVALID_ARG, "hlse needs the device staging dlse");
  const int units = cfg->bh_count;
  const int ns = std::min(n_slices, units);
  const int per = (units + ns - 1) / ns;
  const size_t elem = cfg->dtype == EVA_BF16 ? 2 : 4;
  const size_t row_b = (size_t)cfg->T * cfg->d_head * elem;             // one unit of Q/K/V/O
  const size_t sum_b = (size_t)(cfg->T / cfg->chunk) * cfg->d_head * elem;  // one unit of Ksum
  const size_t lse_b = (size_t)cfg->T * sizeof(float);
  // Validate every slice before enqueueing anything (nothing is enqueued on error).
  for (int u0 = 0; u0 < units; u0 += per) {
    eva_config sub = *cfg;
    sub.bh_begin = cfg->bh_begin + u0;
    sub.bh_count = std::min(per, units - u0);
    const void* p[] = {(char*)dQ + u0 * row_b, (char*)dK + u0 * row_b, (char*)dV + u0 * row_b,
                       (char*)dO + u0 * row_b};
    const char* nm[] = {"dQ", "dK", "dV", "dO"};
    if ((st = check_ptrs(4, p, nm)) != EVA_OK) return st;
    if (sum_b) {
      const void* p2[] = {(char*)dKsum + u0 * sum_b, (char*)dVsum + u0 * sum_b};
      const char* nm2[] = {"dKsum", "dVsum"};
      if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
    }
    if (dlse && !aligned16((char*)dlse + u0 * lse_b))
      return fail(EVA_ERR_INVALID_ARG, "dlse slice is not 16-byte aligned");
  }
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t eps_b = (size_t)(cfg->T / cfg->chunk) * cfg->d_head * sizeof(float);
  cudaError_t e = cudaEventRecord(pipe->fork, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(pipe->h2d, pipe->fork, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(pipe->d2h, pipe->fork, 0);
  if (e != cudaSuccess) return cuda_status(e, "eva_attn_prefill_host(fork)");
  int i = 0;
  for (int u0 = 0; u0 < units; u0 += per, ++i) {
    const int cnt = std::min(per, units - u0);
    const size_t off = u0 * row_b, nb = cnt * row_b;
    e = cudaMemcpyAsync((char*)dQ + off, (const char*)hQ + off, nb, cudaMemcpyHostToDevice, pipe->h2d);
    if (e == cudaSuccess) e = cudaMemcpyAsync((char*)dK + off, (const char*)hK + off, nb, cudaMemcpyHostToDevice, pipe->h2d);
    if (e == cudaSuccess) e = cudaMemcpyAsync((char*)dV + off, (const char*)hV + off, nb, cudaMemcpyHostToDevice, pipe->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(pipe->in[i], pipe->h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, pipe->in[i], 0);
    if (e != cudaSuccess) return cuda_status(e, "eva_attn_prefill_host(h2d)");
    eva_config sub = *cfg;
    sub.bh_begin = cfg->bh_begin + u0;
    sub.bh_count = cnt;
    st = eva_attn_prefill(&sub, (char*)dQ + off, (char*)dK + off, (char*)dV + off,
                          (char*)dKsum + u0 * sum_b, (char*)dVsum + u0 * sum_b,
                          eps ? (const float*)((const char*)eps + u0 * eps_b) : nullptr,
                          (char*)dO + off, dlse ? (float*)((char*)dlse + u0 * lse_b) : nullptr, flags,
                          stream);
    if (st != EVA_OK) return st;
    e = cudaEventRecord(pipe->done[i], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(pipe->d2h, pipe->done[i], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync((char*)hO + off, (char*)dO + off, nb, cudaMemcpyDeviceToHost, pipe->d2h);
    if (e == cudaSuccess && hlse)
      e = cudaMemcpyAsync((char*)hlse + u0 * lse_b, (char*)dlse + u0 * lse_b, cnt * lse_b,
                          cudaMemcpyDeviceToHost, pipe->d2h);
    if (e != cudaSuccess) return cuda_status(e, "eva_attn_prefill_host(d2h)");
  }
  e = cudaEventRecord(pipe->join, pipe->d2h);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, pipe->join, 0);
  return cuda_status(e, "eva_attn_prefill_host(join)");
}

size_t eva_backward_workspace_bytes(const eva_config* cfg) {
  if (check_cfg(cfg, true) != EVA_OK) return 0;
  return eva::backward_workspace_bytes(*cfg);
}

}  // extern "C"
namespace {
// Validation and launch shared by eva_attn_backward and eva_attn_backward_proj (cfg checked).
eva_status backward_common(const eva_config* cfg, const void* Q, const void* K, const void* V,
                           const void* Ksum, const void* Vsum, const void* O, const float* lse,
                           const void* dO, const float* eps, void* dQ, void* dK, void* dV,
                           void* workspace, size_t workspace_bytes, eva_stream_t stream, const float* Pk,
                           float* dPk) {
  eva_status st = EVA_OK;
  if (cfg->mode == EVA_NONCAUSAL && cfg->T % cfg->chunk != 0)
    return fail(EVA_ERR_INVALID_ARG, "EVA_NONCAUSAL needs T %% chunk == 0 (T=%d chunk=%d)", cfg->T,
                cfg->chunk);
  if (cfg->bh_count == 0) return ok();
  const void* p[] = {Q, K, V, O, lse, dO, dQ, dK, dV, workspace};
  const char* nm[] = {"Q", "K", "V", "O", "lse", "dO", "dQ", "dK", "dV", "workspace"};
  if ((st = check_ptrs(10, p, nm)) != EVA_OK) return st;
  if (cfg->T / cfg->chunk > 0) {
    const void* p2[] = {Ksum, Vsum};
    const char* nm2[] = {"Ksum", "Vsum"};
    if ((st = check_ptrs(2, p2, nm2)) != EVA_OK) return st;
  }
  if (eps && !aligned16(eps)) return fail(EVA_ERR_INVALID_ARG, "eps is not 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0)
    return fail(EVA_ERR_INVALID_ARG, "workspace is not 256-byte aligned");
  const size_t need = eva::backward_workspace_bytes(*cfg);
  if (workspace_bytes < need)
    return fail(EVA_ERR_INVALID_ARG, "workspace_bytes %zu < %zu", workspace_bytes, need);
  const cudaError_t e = eva::launch_backward(*cfg, Q, K, V, Ksum, Vsum, O, lse, dO, eps, dQ, dK, dV, workspace,
                                             (cudaStream_t)stream, Pk, dPk);
  if (e == cudaErrorNotSupported) return fail(EVA_ERR_UNSUPPORTED, "eva_attn_backward: projection path");
  return cuda_status(e, "eva_attn_backward");
}
}  // namespace
extern "C" {

size_t eva_backward_proj_workspace_bytes(const eva_config* cfg) {
  if (!cfg) return 0;
  return eva::backward_workspace_bytes(*cfg) + eva::backward_proj_extra_bytes(*cfg);
}

eva_status eva_attn_backward_proj(const eva_config* cfg, const float* Pk, const void* Q, const void* K,
                                  const void* V, const void* Ksum, const void* Vsum, const void* O,
                                  const float* lse, const void* dO, const float* eps, void* dQ, void* dK,
                                  void* dV, float* dPk, void* workspace, size_t workspace_bytes,
                                  eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if ((st = check_causal(cfg, "eva_attn_backward_proj")) != EVA_OK) return st;
  if (cfg->summary_bias != 0.f) return fail(EVA_ERR_UNSUPPORTED, "eva_attn_backward_proj: summary_bias must be 0");
  if (!eva::backward_proj_supported(*cfg))
    return fail(EVA_ERR_UNSUPPORTED, "eva_attn_backward_proj: bf16, d in {32,64,128} and a chunk the register "
                                     "finalize takes (d=%d C=%d)", cfg->d_head, cfg->chunk);
  if (!Pk || !dPk) return fail(EVA_ERR_INVALID_ARG, "Pk / dPk is NULL");
  if (!aligned16(Pk) || !aligned16(dPk)) return fail(EVA_ERR_INVALID_ARG, "Pk / dPk not 16-byte aligned");
  const size_t need = eva_backward_proj_workspace_bytes(cfg);
  if (workspace_bytes < need)
    return fail(EVA_ERR_INVALID_ARG, "workspace_bytes %zu < %zu", workspace_bytes, need);
  return backward_common(cfg, Q, K, V, Ksum, Vsum, O, lse, dO, eps, dQ, dK, dV, workspace, workspace_bytes,
                         stream, Pk, dPk);
}

eva_status eva_attn_backward(const eva_config* cfg, const void* Q, const void* K, const void* V,
                             const void* Ksum, const void* Vsum, const void* O, const float* lse,
                             const void* dO, const float* eps, void* dQ, void* dK, void* dV,
                             void* workspace, size_t workspace_bytes, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  return backward_common(cfg, Q, K, V, Ksum, Vsum, O, lse, dO, eps, dQ, dK, dV, workspace, workspace_bytes,
                         stream, nullptr, nullptr);
}

eva_status eva_mask_ranges(const eva_config* cfg, int64_t n_begin, int64_t count, int64_t* lo,
                           int64_t* nsum, eva_stream_t stream) {
  if (!cfg) return fail(EVA_ERR_INVALID_ARG, "cfg is NULL");
  if (cfg->chunk < 1 || cfg->window < 1 || cfg->window % cfg->chunk != 0)
    return fail(EVA_ERR_INVALID_ARG, "chunk=%d window=%d", cfg->chunk, cfg->window);
  if (cfg->mode != EVA_WINDOW_SLIDING && cfg->mode != EVA_WINDOW_BLOCK)
    return fail(EVA_ERR_INVALID_ARG, "mode=%d", cfg->mode);
  if (n_begin < 0 || count < 0) return fail(EVA_ERR_INVALID_ARG, "n_begin/count must be >= 0");
  if (count > 0 && (!lo || !nsum)) return fail(EVA_ERR_INVALID_ARG, "lo/nsum is NULL");
  return cuda_status(eva::launch_mask_ranges(*cfg, n_begin, count, lo, nsum, (cudaStream_t)stream),
                     "eva_mask_ranges");
}

eva_status eva_philox(const uint32_t* in, uint32_t* out, int32_t n, eva_stream_t stream) {
  if (n < 0) return fail(EVA_ERR_INVALID_ARG, "n=%d", n);
  if (n > 0 && (!in || !out)) return fail(EVA_ERR_INVALID_ARG, "in/out is NULL");
  return cuda_status(eva::launch_philox(in, out, n, (cudaStream_t)stream), "eva_philox");
}

eva_status eva_draw_eps(const eva_config* cfg, float* eps, eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (cfg->bh_count > 0 && cfg->T / cfg->chunk > 0 && !eps) return fail(EVA_ERR_INVALID_ARG, "eps is NULL");
  return cuda_status(eva::launch_draw_eps(*cfg, eps, (cudaStream_t)stream), "eva_draw_eps");
}

eva_status eva_debug_trace_prefill(const eva_config* cfg, const void* Q, const void* K,
                                   const void* V, const void* Ksum, const void* Vsum, void* O,
                                   float* lse, unsigned long long* trace, int32_t cap,
                                   eva_stream_t stream) {
  eva_status st = check_cfg(cfg, true);
  if (st != EVA_OK) return st;
  if (cfg->dtype != EVA_BF16 || (cfg->d_head != 64 && cfg->d_head != 128))
    return fail(EVA_ERR_UNSUPPORTED, "trace needs bf16, d in {64,128}");
  if (!trace || cap < 1) return fail(EVA_ERR_INVALID_ARG, "trace buffer");
  return cuda_status(eva::debug_trace_tile(*cfg, Q, K, V, Ksum, Vsum, O, lse, trace, cap == 2,
                                           (cudaStream_t)stream),
                     "eva_debug_trace_prefill(tile)");
}

const char* eva_last_error(void) { return g_err.c_str(); }

const char* eva_version(void) { return "flasheva-b200 0.1 sm_100a"; }

uint64_t eva_launch_count(void) { return eva::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
