// launch.h -- internal (C++) launchers behind the C ABI in api.cu.
// Arguments are validated by api.cu before any of these is called.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/eva.h"

namespace eva {

// eva_summarize: K, V [bh, T, d] -> Ksum, Vsum [bh, nC, d].  c0: absolute index of the first
// chunk (row 0 is position c0 * C; keys the random draws).
// Pk: optional learned summary-key projection [H, d, d] fp32 (register summariser only;
// cudaErrorNotSupported otherwise).
cudaError_t launch_summarize(const eva_config& cfg, const void* K, const void* V, const float* eps,
                             void* Ksum, void* Vsum, cudaStream_t s, int c0 = 0, const float* Pk = nullptr);
// The persistent bulk-copy summariser (summarize_bulk.cu): bf16, d in {64, 128}, C in {16, 32,
// 64, 128}; same contract as launch_summarize without the projection.
bool summarize_bulk_supported(const eva_config& cfg);
// The summaries of the RoPE-rotated keys on the bulk summariser (keys rotated in shared memory
// after they land); cudaErrorNotSupported outside bf16 d in {64, 128}, C in {16..128} and a
// power-of-two rotary_dim >= 16.
cudaError_t launch_summarize_bulk_rope(const eva_config& cfg, const eva_rope_params& rp, const void* K,
                                       const void* V, const float* eps, void* Ksum, void* Vsum, cudaStream_t s);
// max_ctas > 0 caps the persistent grid (the overlapped prefill runs on the other SMs).
cudaError_t launch_summarize_bulk(const eva_config& cfg, const void* K, const void* V, const float* eps,
                                  void* Ksum, void* Vsum, int c0, cudaStream_t s, int max_ctas = 0);
// RoPE (or its inverse) of [bh_count, T, d] rows at positions (pos ? pos[u] : pos0) + t, with the
// rotary_dim / style of rp (R18, R19; validated by the ABI).
cudaError_t launch_rope(const eva_config& cfg, const eva_rope_params& rp, const void* X, void* Y, int64_t pos0,
                        const int64_t* pos, bool inverse, cudaStream_t s);
// Fused RoPE producer (NEXT row 4, R18/R19): Qr, Kr = RoPE(Q, K) and the summaries of the
// rotated keys in one launch (register summariser only: cudaErrorNotSupported otherwise).
cudaError_t launch_rope_summarize(const eva_config& cfg, const eva_rope_params& rp, const void* Q, const void* K,
                                  const void* V, const float* eps, void* Qr, void* Kr, void* Ksum, void* Vsum,
                                  cudaStream_t s);

// Summaries of the chunks of rows [c0*C, ...) stored to row c0 + c of every destination
// [bh, dst_rows, D] buffer (dst_k/dst_v: device arrays of n_dst base addresses).  Returns
// cudaErrorNotSupported when the chunk does not fit the register summariser (C too large).
cudaError_t launch_summarize_bcast(const eva_config& cfg, int c0, const void* K, const void* V,
                                   const float* eps, const unsigned long long* dst_k,
                                   const unsigned long long* dst_v, int n_dst, int dst_rows, cudaStream_t s);

// Row ranges of one prefill call: query rows are absolute positions [q0, q0 + nq), key/value
// rows [k0, k0 + nkv), summary rows chunks [0, nsl).  The whole-sequence call is
// {0, T, 0, T, T / C}.
struct PrefillRange {
  int64_t q0;
  int32_t nq;
  int32_t pad0;
  int64_t k0;
  int32_t nkv;
  int32_t nsl;
};
inline PrefillRange full_range(const eva_config& c) { return {0, c.T, 0, 0, c.T, c.T / c.chunk}; }

// SIMT prefill (fp32 parity path; any supported d, either dtype).
cudaError_t launch_prefill_simt(const eva_config& cfg, const PrefillRange& rg, const void* Q,
                                const void* K, const void* V, const void* Ksum, const void* Vsum,
                                void* O, float* lse, cudaStream_t s);

// tcgen05/TMEM/TMA prefill (bf16, d in {64, 128}).  Returns cudaErrorNotSupported if the
// shape is outside the kernel's envelope (the caller then reports EVA_ERR_UNSUPPORTED).
bool prefill_sm100_supported(const eva_config& cfg);
// variant bit 0x100: EVA_PREFILL_OVERLAP (summaries provided by the previous grid).
cudaError_t launch_prefill_sm100(const eva_config& cfg, const PrefillRange& rg, const void* Q,
                                 const void* K, const void* V, const void* Ksum, const void* Vsum,
                                 void* O, float* lse, uint32_t variant, cudaStream_t s);
// EVA_SUMMARIES_FUSED: summaries computed inside the tensor-core prefill (whole-sequence call,
// causal modes, C in {16, 32, 64}); Ksum/Vsum written, eps as in eva_summarize.
// cudaErrorStreamCaptureUnsupported: the per-stream workspace has to grow while capturing.
bool prefill_fused_supported(const eva_config& cfg);
cudaError_t launch_prefill_sm100_fused(const eva_config& cfg, const void* Q, const void* K, const void* V,
                                       const float* eps, void* Ksum, void* Vsum, void* O, float* lse,
                                       cudaStream_t s);
cudaError_t prefill_fused_reserve(const eva_config& cfg, cudaStream_t s);
// RoPE inside the tensor-core prefill (eva_attn_prefill_rope): Q, K un-rotated, Ksum/Vsum the
// summaries of the rotated keys; whole-sequence call.  cudaErrorNotSupported outside
// prefill_rope_supported.
bool prefill_rope_supported(const eva_config& cfg, int rotary_dim, int style);
cudaError_t launch_prefill_sm100_rope(const eva_config& cfg, double log2_base, int rotary_dim, int style,
                                      const void* Q, const void* K, const void* V, const void* Ksum,
                                      const void* Vsum, void* O, float* lse, cudaStream_t s,
                                      bool k_rotated = false);

cudaError_t debug_trace_tile(const eva_config& cfg, const void* Q, const void* K, const void* V,
                             const void* Ksum, const void* Vsum, void* O, float* lse,
                             unsigned long long* trace_dev, bool fused, cudaStream_t s);

// Cache append: summaries of chunks completed in [pos, pos+n_new), ring write of the
// last min(n_new, W) tokens.
cudaError_t launch_cache_append(const eva_cache& c, const void* Kn, const void* Vn, int n_new,
                                const float* eps, cudaStream_t s);

// Prefill hand-off with provided summaries (cache.pos == 0): ring + summary copies.
cudaError_t launch_cache_load(const eva_cache& c, const void* K, const void* V, const void* Ksum,
                              const void* Vsum, int n, cudaStream_t s, bool copy_summaries = true);

// Decode: splits chosen by the host (workspace needed when splits > 1).
int decode_splits(const eva_cache& c);
cudaError_t launch_decode(const eva_cache& c, const void* Q, void* O, float* lse, float* ws,
                          int splits, cudaStream_t s);

// Fused append(1) + decode for a token that does not complete a chunk: c_after already
// counts the new token.
cudaError_t launch_decode_step(const eva_cache& c_after, const void* Q, const void* Kn, const void* Vn,
                               void* O, float* lse, float* ws, int splits, cudaStream_t s);
// Ragged decode step (per-unit positions pos[bh_count], device int64, advanced in place):
// ragged_append_kernel then the decode kernel reading each unit's own position.
bool ragged_supported(const eva_config& cfg);  // the register summariser takes cfg.chunk
cudaError_t launch_decode_step_ragged(const eva_cache& c, int64_t* pos, const void* Q, const void* Kn,
                                      const void* Vn, const float* eps, void* O, float* lse, float* ws,
                                      int splits, cudaStream_t s);
// One launch: the decode kernel appends (ring write, chunk summary by one warp) and advances
// pos itself.
cudaError_t launch_decode_step_ragged_fused(const eva_cache& c, int64_t* pos, const void* Q, const void* Kn,
                                            const void* Vn, const float* eps, void* O, float* lse, float* ws,
                                            int splits, cudaStream_t s,
                                            const eva_rope_params* rp = nullptr);

cudaError_t launch_mask_ranges(const eva_config& cfg, int64_t n0, int64_t count, int64_t* lo,
                               int64_t* nsum, cudaStream_t s);
cudaError_t launch_philox(const uint32_t* in, uint32_t* out, int n, cudaStream_t s);
cudaError_t launch_draw_eps(const eva_config& cfg, float* eps, cudaStream_t s);

// Backward of the prefill (backward_simt.cu): dQ, dK, dV of L = sum(dO * O).
size_t backward_workspace_bytes(const eva_config& cfg);
// Pk (optional, R17): the learned summary-key projection [H, d, d]; dPk [H, d, d] fp32 gets the
// sum over this call's units of each head (workspace + backward_proj_extra_bytes).
cudaError_t launch_backward(const eva_config& cfg, const void* Q, const void* K, const void* V,
                            const void* Ksum, const void* Vsum, const void* O, const float* lse,
                            const void* dO, const float* eps, void* dQ, void* dK, void* dV,
                            void* workspace, cudaStream_t s, const float* Pk = nullptr, float* dPk = nullptr);
size_t backward_proj_extra_bytes(const eva_config& cfg);
bool backward_proj_supported(const eva_config& cfg);

// Tensor-core main pass of the backward (backward_sm100.cu): bf16, d in {64, 128}.
// phase 0: every work item, local dK/dV to the fp32 workspace (finalize applies the summary
// chain rule); 1: the summary items only; 2: the local items only, applying the chain rule
// from the coefficients in *fused and writing dK/dV in bf16.
struct BwdFusedArgs {
  float *w, *da, *om, *dkt;  // per row [bh, T]; per chunk [bh, nC, d]
  void *dK, *dV;                   // bf16 outputs [bh, T, d]
};
bool backward_sm100_supported(const eva_config& cfg);
cudaError_t launch_backward_main_sm100(const eva_config& cfg, const void* Q, const void* K, const void* V,
                                       const void* Ksum, const void* Vsum, const void* dO, const float* lse,
                                       float* wsD, float* wsdQ, float* wsdK, float* wsdV, float* wsdKs,
                                       float* wsdVs, const BwdFusedArgs* fused, int phase, cudaStream_t s);

int num_sms();
// 3-D bf16 TMA map over [units, rows, D] with a {64, box_rows, 1} box and 128-byte swizzle
// (prefill_sm100.cu); false if the driver entry point is unavailable.
bool make_tma_map_bf16(CUtensorMap* m, const void* base, int units, int rows, int D, int box_rows);
// Raise a kernel's dynamic shared-memory limit (once per function and size).
cudaError_t set_smem_attr(const void* fn, size_t bytes);

}  // namespace eva
