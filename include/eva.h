/*
 * eva.h -- C ABI of the B200-native FlashEVA hot path (libeva.so).
 *
 * FlashEVA (arxiv 2511.00576) evaluates EVA attention as softmax attention
 * over an augmented key/value set (Eq.12-14): every query
 * n attends to its exact local window E(n) and to one summary pair
 * (k~_c, beta^_c) per chunk c that lies entirely before the window, under the
 * "custom causal mask" of P:124.  Citations: P:NN = PAPER.md line NN,
 * S:NN = SPEC.md line NN; DESIGN.md lists every reading R1..R13 taken where
 * the paper is silent.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All tensor pointers are DEVICE pointers (cudaMalloc / torch CUDA memory)
 *    owned by the caller, except the h* arguments of eva_attn_prefill_host
 *    (host memory).  The library allocates no device memory and keeps no
 *    global state except a thread-local error string and a cache of the
 *    device attributes it queried; the streams and events of the host-copy
 *    pipeline live in an explicit eva_pipeline object.
 *  - Layout: row-major, contiguous.  A "unit" is one (batch, head) pair with
 *    global flattened index u = b*H + h.  Per-unit tensors are [units, rows, d].
 *    Every call works on units [bh_begin, bh_begin + bh_count): tensor
 *    pointers address the FIRST unit of that shard (slot 0 <-> unit bh_begin);
 *    bh_begin only keys the random draws, so a sharded run is bitwise equal
 *    to the same slice of an unsharded run.
 *  - Element type of Q/K/V/O/summaries/ring: cfg.dtype (fp32 or bf16).  LSE
 *    and eps are always fp32.  Accumulation is always fp32.
 *  - All calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream).  Argument validation is synchronous: on any non-OK
 *    status nothing has been enqueued and eva_last_error() says why.
 *  - Positions are 0-indexed.  Chunk c covers positions [c*C, c*C + C).
 *    nC = floor(T / C) complete chunks are summarised; a trailing partial
 *    chunk never is (it is always inside the window, reading R8).
 */
#ifndef EVA_H_
#define EVA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct CUstream_st* eva_stream_t; /* == cudaStream_t */

typedef enum {
  EVA_OK = 0,
  EVA_ERR_INVALID_ARG = 1, /* null pointer, non-positive size, W % C != 0, shard outside [0, B*H), misaligned */
  EVA_ERR_UNSUPPORTED = 2, /* samples != 1, or d_head not supported for the dtype */
  EVA_ERR_CAPACITY = 3,    /* cache append would exceed the summary capacity */
  EVA_ERR_CUDA = 4         /* a CUDA launch/runtime error (message in eva_last_error) */
} eva_status;

typedef enum { EVA_F32 = 0, EVA_BF16 = 1 } eva_dtype;

/* Partition of the past ("local set E and disjoint subsets P_c"; P:126,
 * P:298 "local attention" vs "sliding window"), reading R7:
 *   SLIDING (window start quantised to a chunk boundary):
 *       nsum(n) = max(0, floor(n/C) - W/C + 1),  lo(n) = nsum(n)*C
 *   BLOCK (original EVA's non-overlapping local blocks of width W):
 *       lo(n) = floor(n/W)*W,                    nsum(n) = lo(n)/C
 * Query n attends to locals m in [lo(n), n] and to summaries c < nsum(n). */
typedef enum { EVA_WINDOW_SLIDING = 0, EVA_WINDOW_BLOCK = 1, EVA_NONCAUSAL = 2 } eva_window_mode;
/* EVA_NONCAUSAL (prefill only; "In the non-causal setting ..."; reading R15):
 *   E(n) = n's whole block [lo, min(lo + W, T)), lo = floor(n/W)*W (later positions of the
 *   block included), plus the summaries of EVERY complete chunk outside that block, before
 *   and after it: c < lo/C or c >= (lo + W)/C.  Requires T % C == 0 (every position is a
 *   local or inside exactly one summarised chunk).  Prefill and its backward take it;
 *   decode, cache and the query-range prefill are causal by construction and return
 *   EVA_ERR_UNSUPPORTED. */

/* Proposal of Eq.15, reading R3:
 *   AS_PRINTED:     omega_c = lambda * clip(k~_c + eps_c, -clip, clip)   (default)
 *   SHIFTED_NOISE:  omega_c = k~_c + lambda * clip(eps_c, -clip, clip)   */
typedef enum { EVA_OMEGA_AS_PRINTED = 0, EVA_OMEGA_SHIFTED_NOISE = 1 } eva_omega_mode;

typedef struct {
  int32_t B, H;               /* global batch and heads (the RNG is keyed by b*H + h)   */
  int32_t bh_begin, bh_count; /* this call's shard of units; full problem = (0, B*H)    */
  int32_t T;                  /* sequence length (prefill / summarize); ignored by decode */
  int32_t d_head;             /* head dim d: fp32 {16,32,64,128}, bf16 {16,32,64,128}    */
  int32_t chunk;              /* C: tokens per summary ("number of keys/values compressed") */
  int32_t window;             /* W: local window, W >= C and W % C == 0  */
  int32_t samples;            /* S: random samples per chunk; only 1 is supported */
  int32_t mode;               /* eva_window_mode */
  int32_t dtype;              /* eva_dtype */
  int32_t omega_mode;         /* eva_omega_mode */
  float scale;                /* logit scale s > 0 on q.k and q.k~ (reading R5), e.g. 1/sqrt(d) */
  float lambda;               /* Eq.15 lambda, paper value 0.1                 */
  float clip;                 /* Eq.15 clip bound, paper value 1               */
  uint32_t layer;             /* RNG key component (reading R9)                         */
  uint64_t seed;              /* RNG key when eps == NULL (reading R9)                  */
  float summary_bias;         /* added to every summary logit s q.k~_c (natural-log units):
                                 0 = Eq.10 as printed (reading R4); ln C counts each
                                 summary as the C tokens it replaces (reading R16) */
  int32_t reserved;           /* must be 0 */
} eva_config;

/* Fill *cfg with the paper's defaults for (B, H, T, d, C, W):
 * full shard, S = 1, sliding, scale = 1/sqrt(d), lambda = 0.1, clip = 1,
 * omega as printed, seed = 1234, layer = 0, dtype bf16, summary_bias = 0. */
void eva_config_default(eva_config* cfg, int32_t B, int32_t H, int32_t T, int32_t d,
                        int32_t chunk, int32_t window);

/* ---------------------------------------------------------------- summaries
 * eva_summarize: per-chunk summaries of every complete chunk (S = 1):
 *   k~_c     = (1/C) sum_{i<C} k_{cC+i}                        (Eq.10; reading R1)
 *   omega_c  = Eq.15 with mu_c = k~_c                          (readings R2, R3)
 *   a_i      = omega_c . k_{cC+i} - |k_{cC+i}|^2 / 2           (log xi)
 *   beta^_c  = sum_i softmax(a)_i v_{cC+i}                     (Eq.9 ratio sum g / sum h)
 * K, V : [bh_count, T, d] cfg.dtype
 * eps  : [bh_count, nC, d] fp32 caller-supplied N(0, I) draws, or NULL to draw
 *        them in-kernel with Philox4x32-10 + Box-Muller keyed by
 *        (seed, layer, b*H + h, c) (reading R9; identical to oracle_eps()).
 * Ksum : [bh_count, nC, d] cfg.dtype (out)  -- k~_c
 * Vsum : [bh_count, nC, d] cfg.dtype (out)  -- beta^_c
 * T < C (nC = 0) is valid and enqueues nothing. */
eva_status eva_summarize(const eva_config* cfg, const void* K, const void* V, const float* eps,
                         void* Ksum, void* Vsum, eva_stream_t stream);

/* eva_rope_summarize: the fused RoPE producer of SURVEY §8(f) NEXT row 4 ("RoPE is
 * applied to all tokens prior to the random feature projections"; reading R18).
 * One launch reads the caller's pre-RoPE Q, K (and V) [bh_count, T, d] and writes
 *   Qr, Kr : RoPE(Q), RoPE(K) [bh_count, T, d] cfg.dtype -- consecutive channel pairs
 *            (2j, 2j+1) of the row at position n rotated by n * rope_base^(-2j/d);
 *   Ksum, Vsum : the summaries of the ROTATED keys (eva_summarize's formulas on Kr's values),
 * so the prefill then runs on (Qr, Kr, V, Ksum, Vsum) with EVA_SUMMARIES_PROVIDED.  Saves the
 * separate RoPE pass's second read of K.  Register summariser only (chunk <= 16 * 4 * 32 /
 * (d * sizeof(dtype) / 16)), else EVA_ERR_UNSUPPORTED; rope_base must be finite and > 1. */
eva_status eva_rope_summarize(const eva_config* cfg, float rope_base, const void* Q, const void* K,
                              const void* V, const float* eps, void* Qr, void* Kr, void* Ksum, void* Vsum,
                              eva_stream_t stream);

/* eva_rope: the RoPE of R18 alone, Y = R(pos) X for rows [bh_count, T, d] cfg.dtype at
 * positions pos0 + t (decode: q, k_new at their position with T = 1), or with inverse != 0
 * the transposed rotation Y = R(pos)^T X -- the gradient through RoPE: after
 * eva_attn_backward on (Qr, Kr, V) gives dQr, dKr, the pre-RoPE gradients are
 * dQ = R^T dQr, dK = R^T dKr.  X == Y (in place) is allowed.  = eva_rope_ex with
 * {rope_base, d, EVA_ROPE_INTERLEAVED} and pos = NULL. */
eva_status eva_rope(const eva_config* cfg, float rope_base, const void* X, void* Y, int64_t pos0,
                    int32_t inverse, eva_stream_t stream);

/* Generalised RoPE (reading R19): which channels rotate and how they pair.
 *   base       : > 1, finite (10000 in Pythia / GPT-NeoX)
 *   rotary_dim : 0 = d; else even, <= d, a multiple of 2 * (16 / sizeof(dtype)) (16 for bf16,
 *                8 for fp32) -- channels >= rotary_dim pass through (Pythia: rotary_pct)
 *   style      : EVA_ROPE_INTERLEAVED -- pairs (2j, 2j+1); EVA_ROPE_NEOX -- pairs (j, j + rd/2)
 *                (GPT-NeoX rotate_half); angle pos * base^(-2j/rd) for pair j < rd/2
 *   reserved   : 0 */
#define EVA_ROPE_INTERLEAVED 0
#define EVA_ROPE_NEOX 1
typedef struct eva_rope_params {
  float base;
  int32_t rotary_dim;
  int32_t style;
  int32_t reserved;
} eva_rope_params;

/* eva_rope_ex: Y = R(p) X (inverse: R(p)^T X) for rows [bh_count, T, d] cfg.dtype, row t of unit u
 * at position p = (pos ? pos[u] : pos0) + t.  pos: NULL or a DEVICE int64 array [bh_count] of
 * per-unit positions (>= 0, read by the kernel -- graph-capturable; a ragged decode batch rotates
 * its q / k_new with the same pos array it passes to eva_decode_step_ragged).  X == Y allowed. */
eva_status eva_rope_ex(const eva_config* cfg, const eva_rope_params* rp, const void* X, void* Y, int64_t pos0,
                       const int64_t* pos, int32_t inverse, eva_stream_t stream);

/* eva_rope_summarize_ex: eva_rope_summarize with eva_rope_params (R19).  The half-split style
 * additionally needs rotary_dim / (2 * 16 / sizeof(dtype)) to be a power of two (the partner
 * piece is exchanged between lanes by a butterfly), else EVA_ERR_UNSUPPORTED. */
eva_status eva_rope_summarize_ex(const eva_config* cfg, const eva_rope_params* rp, const void* Q, const void* K,
                                 const void* V, const float* eps, void* Qr, void* Kr, void* Ksum, void* Vsum,
                                 eva_stream_t stream);

/* eva_summarize_proj: eva_summarize with the learned summary-key projection of SURVEY
 * §8(f) NEXT row 4 ("new weights"; EVA's summary key is a learned map of the chunk
 * mean -- reading R17): k~_c = Pk[h] (1/C) sum_i k_{cC+i}, mu_c = k~_c in Eq.15,
 * beta^_c from Eq.9 with the raw keys.  Pk: device fp32 [H, d, d] row-major (head h of unit
 * bh_begin + u is (bh_begin + u) % H), 16-byte aligned, caller-owned, read only.  The
 * outputs feed eva_attn_prefill(EVA_SUMMARIES_PROVIDED) / eva_cache_load like eva_summarize's.
 * Runs on the register summariser (chunk <= 16 * 4 * 32 / (d * sizeof(dtype) / 16) rows);
 * longer chunks -> EVA_ERR_UNSUPPORTED.  Pk == NULL -> EVA_ERR_INVALID_ARG. */
eva_status eva_summarize_proj(const eva_config* cfg, const void* K, const void* V, const float* eps,
                              const float* Pk, void* Ksum, void* Vsum, eva_stream_t stream);

/* ---------------------------------------------------------------- prefill
 * eva_attn_prefill: chunk-causal FlashEVA attention for all T queries
 * (Eq.12-14, mask P:124, sliding window P:126):
 *   o_n = sum_{x in E(n) U {c < nsum(n)}} softmax_x(s q_n . key_x) value_x
 *   lse_n = log sum_x exp(s q_n . key_x)          (natural log)
 * Q, K, V, O : [bh_count, T, d] cfg.dtype
 * Ksum, Vsum : [bh_count, nC, d] cfg.dtype; read when EVA_SUMMARIES_PROVIDED,
 *              otherwise written (they are computed inside this call).
 * eps        : as in eva_summarize (ignored with EVA_SUMMARIES_PROVIDED).
 * lse        : [bh_count, T] fp32 (out) or NULL.
 * flags      : EVA_SUMMARIES_PROVIDED -- use the caller's Ksum/Vsum as is;
 *              EVA_SUMMARIES_FUSED    -- compute the summaries inside the attention kernel, one
 *                                        launch (EVA_ERR_UNSUPPORTED where it does not apply, below);
 *              EVA_SUMMARIES_SEPARATE -- compute them in a separate eva_summarize launch first;
 *              EVA_PREFILL_SIMT       -- force the SIMT kernel (parity/debug; separate summaries);
 *              EVA_PREFILL_OVERLAP    -- see below;
 *              0                      -- separate (measured faster on B200 than the fused launch
 *                                        at configs[1] and configs[2]).
 * bf16 runs the tcgen05/TMEM/TMA kernel for d in {64, 128} (requires 16-byte
 * aligned base pointers); other cases run the SIMT kernel.
 * Fused summaries (section 4.4 names the separate summary pass as FlashEVA's overhead at
 * short L): the CTA of each 128-query tile summarises the complete chunks inside its own
 * query rows from the K/V tiles it has already loaded for the attention, publishes them
 * with a per-tile ready flag, and reads the earlier chunks' summaries once their owners
 * have published (query tiles are dispatched by a monotone ticket, so every awaited owner
 * is resident).  Applies to bf16, d in {64, 128}, causal modes (sliding / block) and chunk
 * sizes C in {16, 32, 64}.  Uses a per-(device, stream) workspace owned by
 * the library, allocated on the first fused call of a shape; a CUDA graph capturing the
 * call needs it allocated first (eva_prefill_reserve), else EVA_ERR_INVALID_ARG.  The
 * summaries equal eva_summarize's up to fp32 summation order (bf16 outputs may differ by
 * one rounding step). */
#define EVA_SUMMARIES_PROVIDED 1u
#define EVA_SUMMARIES_FUSED 2u
#define EVA_PREFILL_SIMT 4u
#define EVA_SUMMARIES_SEPARATE 16u
/* EVA_PREFILL_OVERLAP (with EVA_SUMMARIES_PROVIDED, tensor-core path): the caller asserts that
 * the launch immediately before this one on `stream` is the eva_summarize that writes Ksum/Vsum
 * and that Q, K, V were complete before that launch.  The prefill then starts its local-window
 * tiles while that kernel finishes (programmatic dependent launch) and waits for it only before
 * reading the summaries (measured neutral to slower on B200 -- DESIGN.md §11 -- so off by
 * default). */
#define EVA_PREFILL_OVERLAP 128u
eva_status eva_attn_prefill(const eva_config* cfg, const void* Q, const void* K, const void* V,
                            void* Ksum, void* Vsum, const float* eps, void* O, float* lse,
                            uint32_t flags, eva_stream_t stream);

/* eva_prefill_reserve: allocate (or grow) the library's workspace of the fused-summary prefill
 * for cfg's shape on `stream` (one zero-initialised 32-bit ready flag per (unit, 128-query
 * tile) plus 16 bytes of counters; kept until process exit).  Call it before capturing an
 * eva_attn_prefill into a CUDA graph; synchronises `stream` if an existing buffer is replaced. */
eva_status eva_prefill_reserve(const eva_config* cfg, eva_stream_t stream);

#define EVA_ROPE_K_ROTATED 512u
/* eva_attn_prefill_rope: eva_attn_prefill on RoPE(Q), RoPE(K) with the rotation done INSIDE the
 * tensor-core kernel ("RoPE is applied to all tokens prior to
 * the random feature projections"; readings R18/R19): Q and K [bh_count, T, d] are the caller's
 * un-rotated rows; the kernel rotates the landed Q tile and each local K tile in shared memory
 * (row at position n by n * base^(-2j/rd), rp as in eva_rope_ex), so RoPE(Q) and RoPE(K) are
 * never written.  The summary keys are chunk means of the ROTATED keys:
 *   flags 0                      -- computed first by eva_rope_summarize_ex's summariser in its
 *                                   summaries-only form (Ksum/Vsum written, out);
 *   EVA_SUMMARIES_PROVIDED       -- Ksum/Vsum already hold them (in), e.g. from
 *                                   eva_rope_summarize_ex or a decode cache.
 *   EVA_ROPE_K_ROTATED           -- K (and Ksum/Vsum when provided) hold ROTATED keys already
 *                                   (e.g. eva_rope_ex's output, kept for the decode cache); the
 *                                   kernel rotates Q only, and missing summaries come from the
 *                                   plain eva_summarize on K.  The fastest RoPE prefill when the
 *                                   rotated keys are stored anyway (one rotation per key instead
 *                                   of one per query tile that reads it).
 * Decode hand-off: the cache holds ROTATED keys (eva_decode_step_ragged_rope appends rotated
 * ones), so eva_cache_load takes RoPE(K) -- eva_rope_ex's output, which the EVA_ROPE_K_ROTATED
 * form has at hand -- with these Ksum/Vsum.
 * O (out) and lse (out, may be NULL) as in eva_attn_prefill.  The result equals eva_attn_prefill
 * on eva_rope_ex's outputs up to the rounding of the rotated bf16 values.  Whole-sequence call,
 * every cfg.mode; bf16, d in {64, 128} and rotary_dim (0 = d) a power of two (>= 8 interleaved,
 * >= 16 half-split), else EVA_ERR_UNSUPPORTED; other flags -> EVA_ERR_INVALID_ARG. */
eva_status eva_attn_prefill_rope(const eva_config* cfg, const eva_rope_params* rp, const void* Q, const void* K,
                                 const void* V, const float* eps, void* Ksum, void* Vsum, void* O, float* lse,
                                 uint32_t flags, eva_stream_t stream);

/* ---------------------------------------------------------------- query-range prefill
 * The building blocks of a sequence-sharded (context-parallel) prefill (SURVEY §8(f) NEXT
 * row 2; the paper positions EVA against ring attention): a rank that owns positions
 * [q0, q1) needs only its own keys/values, a halo of the window before q0, and the chunk
 * summaries of the whole prefix (summaries are per-chunk, query-independent).
 *
 * eva_summarize_range: eva_summarize for rows that start at absolute position chunk0 * C:
 * K, V : [bh_count, cfg.T, d] with row r = position chunk0*C + r; Ksum, Vsum : [bh_count,
 * floor(cfg.T / C), d], row c = absolute chunk chunk0 + c (whose random draw it uses; eps,
 * if given, is [bh_count, floor(cfg.T / C), d] for those chunks).  chunk0 >= 0. */
eva_status eva_summarize_range(const eva_config* cfg, int32_t chunk0, const void* K, const void* V,
                               const float* eps, void* Ksum, void* Vsum, eva_stream_t stream);

/* eva_summarize_range_bcast: eva_summarize_range fused with the context-parallel all-gather:
 * the summaries of absolute chunks [chunk0, chunk0 + floor(T/C)) are computed once and stored
 * to rows chunk0 + c of EVERY destination pair (dst_ksum[i], dst_vsum[i]), i < n_dst, each a
 * [bh_count, dst_rows, d] cfg.dtype buffer -- typically every rank's copy of the global
 * summary list reached through NVLink peer pointers (symmetric memory), so the exchange rides
 * on the summarising kernel's own stores.  dst_ksum / dst_vsum are DEVICE arrays of n_dst
 * device addresses (0 <= n_dst <= 64); dst_rows >= chunk0 + floor(T/C).  The caller orders
 * the destinations' readers after this kernel on every rank (e.g. a symmetric-memory barrier).
 * EVA_ERR_UNSUPPORTED if a chunk exceeds the register summariser (C > 256 at d = 128 bf16). */
eva_status eva_summarize_range_bcast(const eva_config* cfg, int32_t chunk0, const void* K, const void* V,
                                     const float* eps, const uint64_t* dst_ksum, const uint64_t* dst_vsum,
                                     int32_t n_dst, int32_t dst_rows, eva_stream_t stream);

/* eva_attn_prefill_range: eva_attn_prefill (summaries provided) for the queries at absolute
 * positions [q0, q0 + n_q) only.
 * Q, O : [bh_count, n_q, d]        row i = position q0 + i
 * K, V : [bh_count, n_kv, d]       row r = position k0 + r
 * Ksum, Vsum : [bh_count, n_sum, d] row c = chunk c (absolute, from 0)
 * lse : [bh_count, n_q] fp32 or NULL.  cfg.T is not used.
 * Requires k0 <= lo(q0) (the window of the first query is present: a halo of at most W - 1
 * rows before q0), k0 + n_kv >= q0 + n_q, and n_sum >= nsum(q0 + n_q - 1); otherwise
 * EVA_ERR_INVALID_ARG.  flags: 0 or EVA_PREFILL_SIMT.  When q0 is a multiple of 128 the rows
 * are bitwise equal to the same rows of a whole-sequence eva_attn_prefill (same tiles, same
 * kernel); otherwise equal up to fp32 summation order. */
eva_status eva_attn_prefill_range(const eva_config* cfg, int64_t q0, int32_t n_q, int64_t k0,
                                  int32_t n_kv, const void* Q, const void* K, const void* V,
                                  const void* Ksum, const void* Vsum, int32_t n_sum, void* O,
                                  float* lse, uint32_t flags, eva_stream_t stream);

/* ---------------------------------------------------------------- decode cache
 * Compressed decode cache ("cache of (compressed) past
 * context"): a ring of the last W tokens plus one summary per
 * completed chunk.  Summaries are written eagerly when a chunk's last token
 * arrives; the attention only ever reads c < nsum(n), so this equals SPEC's
 * lazy compress-on-eviction -- reading R13.
 *   ring_k, ring_v : [bh_count, W, d]           cfg.dtype, slot p mod W holds position p
 *   sum_k,  sum_v  : [bh_count, cap_chunks, d]  cfg.dtype, row c = chunk c
 *   pos            : number of tokens appended so far (uniform over the shard)
 * The descriptor is a plain caller-owned struct; the library only reads it,
 * except eva_cache_append which advances pos.  Single writer. */
typedef struct {
  eva_config cfg; /* cfg.T is ignored */
  int64_t pos;
  int32_t cap_chunks;
  int32_t reserved;
  void* ring_k;
  void* ring_v;
  void* sum_k;
  void* sum_v;
} eva_cache;

/* Append n_new >= 1 tokens per unit at positions [pos, pos + n_new):
 * K_new, V_new : [bh_count, n_new, d] cfg.dtype
 * eps          : [bh_count, cap_chunks, d] fp32 indexed by ABSOLUTE chunk index, or NULL (Philox).
 * Every chunk completed by these tokens is summarised (eva_summarize's formulas),
 * and the last min(n_new, W) tokens are written to the ring.  n_new = T is the
 * prefill hand-off.  EVA_ERR_CAPACITY if (pos + n_new) / C > cap_chunks.
 * On success cache->pos += n_new. */
eva_status eva_cache_append(eva_cache* cache, const void* K_new, const void* V_new, int32_t n_new,
                            const float* eps, eva_stream_t stream);

/* Prefill hand-off when the prompt's summaries already exist (e.g. Ksum/Vsum written
 * by eva_attn_prefill): equivalent to eva_cache_append(cache, K, V, n, eps) on an empty
 * cache (the summaries are the same function of the same chunks, R13), but copies the
 * nC = floor(n / C) summary rows instead of recomputing them.
 * K, V       : [bh_count, n, d] cfg.dtype -- the prompt's keys and values
 * Ksum, Vsum : [bh_count, nC, d] cfg.dtype (may be NULL when nC == 0).  They may BE
 *              cache->sum_k / sum_v (both or neither, and then cap_chunks == nC): the prompt's
 *              summaries were written into the cache directly (eva_summarize / eva_attn_prefill
 *              on the cache's buffers) and only the ring is copied -- a copy that does not
 *              depend on the summaries, so it may run concurrently with the summariser.
 * Requires cache->pos == 0.  EVA_ERR_CAPACITY if nC > cap_chunks.  On success pos = n. */
eva_status eva_cache_load(eva_cache* cache, const void* K, const void* V, const void* Ksum,
                          const void* Vsum, int32_t n, eva_stream_t stream);

/* One query per unit at position n = pos - 1 over the cache (Eq.12, one row):
 * Q, O : [bh_count, d] cfg.dtype;  lse : [bh_count] fp32 or NULL.
 * workspace : device scratch of eva_decode_workspace_bytes(cache) bytes (may be
 *             NULL when that is 0).  It must be zero-filled before its first use; every
 *             call leaves it zero-filled where it matters (split-K merge counters), so
 *             one buffer serves a whole generation.  pos must be >= 1. */
eva_status eva_attn_decode(const eva_cache* cache, const void* Q, void* O, float* lse,
                           void* workspace, size_t workspace_bytes, eva_stream_t stream);
size_t eva_decode_workspace_bytes(const eva_cache* cache);

/* One generation step in one launch: append (K_new, V_new) at position p = pos and attend
 * query Q (the same position) over the cache -- the result equals
 * eva_cache_append(cache, K_new, V_new, 1, eps) followed by eva_attn_decode(cache, Q, ...),
 * bit for bit.  The token's own key/value are read from K_new/V_new and written to the ring by
 * the same launch; a token that completes a chunk, and any step with bh_count >= 1024 (where
 * the decode is a long HBM stream and two launches measured faster), takes the two-launch
 * path (append kernel, then decode).
 * K_new, V_new, Q, O : [bh_count, d] cfg.dtype; eps as in eva_cache_append; lse or NULL.
 * workspace: eva_decode_workspace_bytes() of the cache AFTER the append (pos + 1).
 * On success pos += 1. */
eva_status eva_decode_step(eva_cache* cache, const void* Q, const void* K_new, const void* V_new,
                           const float* eps, void* O, float* lse, void* workspace,
                           size_t workspace_bytes, eva_stream_t stream);

/* eva_decode_step_ragged: one decode token per unit at PER-UNIT positions (SURVEY §8(f) NEXT
 * row 4: "per-sequence positions in decode" -- a serving batch whose sequences have
 * different lengths).  pos: device int64 [bh_count], pos[u] = tokens unit u holds
 * (cache->pos is ignored); for every u the new token (K_new[u], V_new[u], [bh_count, d]) is
 * appended at position pos[u] (ring slot pos[u] mod W; the chunk it completes, if any, is
 * summarised with eva_summarize's formulas, eps as in eva_cache_append), then query Q[u] at
 * position pos[u] attends over its own visible set (a7), O/lse [bh_count, d] / [bh_count],
 * and pos[u] is advanced by one -- all on the device, so the call is graph-capturable.
 * Preconditions (not checkable without a sync): 0 <= pos[u] and (pos[u] + 1) / chunk <=
 * cap_chunks (a chunk past the capacity is not summarised).  workspace: at least
 * eva_decode_ragged_workspace_bytes(cache) bytes (the split count covers the longest
 * position the cache can hold), zero-filled before first use; calls leave it zeroed.
 * One kernel is enqueued: the split-K decode appends the token (split 0 writes the ring
 * slot, its first warp summarises a completed chunk) and the unit's merging CTA advances
 * pos[u].  (EVA_RAGGED_TWO_LAUNCH=1 in the environment selects an append kernel + decode
 * pair instead; that form needs chunk <= 16 * 4 * 32 / (d * sizeof(dtype) / 16), else
 * EVA_ERR_UNSUPPORTED.) */
size_t eva_decode_ragged_workspace_bytes(const eva_cache* cache);
eva_status eva_decode_step_ragged(const eva_cache* cache, int64_t* pos, const void* Q, const void* K_new,
                                  const void* V_new, const float* eps, void* O, float* lse, void* workspace,
                                  size_t workspace_bytes, eva_stream_t stream);

/* eva_decode_step_ragged_rope: eva_decode_step_ragged with RoPE folded into the same launch
 * (readings R18/R19): Q and K_new are the caller's UN-rotated
 * rows; the kernel rotates q and k_new of unit u at its position pos[u] in registers, appends
 * RoPE(k_new) (in dtype) to the ring -- so the cache holds rotated keys, as the prefill hand-off
 * of eva_rope_summarize_ex / eva_attn_prefill_rope leaves it -- summarises a completed chunk
 * from the rotated keys, and attends with RoPE(q).  Equals eva_rope_ex(q), eva_rope_ex(k_new)
 * at pos followed by eva_decode_step_ragged, up to the rounding of RoPE(q) to dtype (kept in
 * fp32 here).  rp as in eva_rope_ex; the half-split style additionally needs
 * rotary_dim / (2 * 16 / sizeof(dtype)) to be a power of two, else EVA_ERR_UNSUPPORTED.
 * rp == NULL: exactly eva_decode_step_ragged.  Always one launch. */
eva_status eva_decode_step_ragged_rope(const eva_cache* cache, int64_t* pos, const eva_rope_params* rp,
                                       const void* Q, const void* K_new, const void* V_new, const float* eps,
                                       void* O, float* lse, void* workspace, size_t workspace_bytes,
                                       eva_stream_t stream);

/* ---------------------------------------------------------------- host-buffer prefill
 * eva_attn_prefill_host: eva_attn_prefill on inputs and outputs in HOST memory, with the
 * host<->device copies overlapped with the kernels (the end-to-end path of a caller whose
 * prompt is on the host).  The units [0, bh_count) are cut into n_slices contiguous slices
 * (each unit's summaries and attention depend on that unit only, P:101 S = 1, so slices
 * are independent); on three streams
 *     copy-in  : H2D of slice i's Q, K, V                     (pipe's h2d stream)
 *     compute  : eva_attn_prefill(slice i, flags)             (`stream`)
 *     copy-out : D2H of slice i's O (and lse)                 (pipe's d2h stream)
 * so slice i's H2D overlaps slice i-1's kernels and slice i-2's D2H.  Both side streams
 * fork from and join back into `stream` (the call is stream-ordered and CUDA-graph
 * capturable).  Results are bitwise equal to one eva_attn_prefill over all units.
 * hQ, hK, hV : host [bh_count, T, d] cfg.dtype (pinned for true asynchrony; pageable
 *              memory works but serialises the copies)
 * hO         : host [bh_count, T, d] cfg.dtype (out);  hlse : host [bh_count, T] fp32 or NULL
 * dQ, dK, dV, dO : device staging [bh_count, T, d] cfg.dtype, caller-owned; on completion
 *              dK, dV hold the prompt (for eva_cache_load) and dO the output
 * dKsum, dVsum : device [bh_count, nC, d] (out: the summaries, for eva_cache_load)
 * dlse       : device [bh_count, T] fp32, required when hlse != NULL, else may be NULL
 * eps, flags : as in eva_attn_prefill (EVA_SUMMARIES_PROVIDED is rejected: summaries are
 *              always computed here from the copied K, V)
 * n_slices   : 1 .. eva_pipeline max_slices (clamped to bh_count)
 * The host buffers must stay valid until `stream` reaches the end of the call. */
typedef struct eva_pipeline eva_pipeline;
/* Creates the two side streams and 2*max_slices+2 events the copy pipeline uses. */
eva_status eva_pipeline_create(int32_t max_slices, eva_pipeline** out);
void eva_pipeline_destroy(eva_pipeline* pipe);
eva_status eva_attn_prefill_host(eva_pipeline* pipe, const eva_config* cfg, const void* hQ,
                                 const void* hK, const void* hV, void* hO, float* hlse, void* dQ,
                                 void* dK, void* dV, void* dKsum, void* dVsum, void* dO, float* dlse,
                                 const float* eps, uint32_t flags, int32_t n_slices,
                                 eva_stream_t stream);

/* ---------------------------------------------------------------- backward (training)
 * eva_attn_backward: gradient of the prefill (the paper
 * trains FlashEVA models with it).  For L = sum_n dO_n . o_n it
 * writes dQ, dK, dV, differentiating through the attention (Eq.12-14) AND the
 * chunk summaries (k~ = chunk mean, omega = Eq.15, beta^ = Eq.9/10); eps is a
 * constant; d clip/dx = 1 on the closed range [-clip, clip] (R14).
 * Every cfg.mode (incl. EVA_NONCAUSAL, T % chunk == 0) and cfg.summary_bias (R16: a
 * constant added to the summary logits, so the summary P carries it and dS keeps its form)
 * are supported; the forward must have used the same cfg.
 * Q, K, V, O, dO, dQ, dK, dV : [bh_count, T, d] cfg.dtype
 * Ksum, Vsum : [bh_count, nC, d] cfg.dtype -- the summaries the forward used
 * O, lse     : the forward's output and natural-log lse ([bh_count, T] fp32)
 * eps        : as in eva_summarize (NULL = the in-kernel Philox draws); must be
 *              what the forward used.
 * workspace  : device scratch of eva_backward_workspace_bytes(cfg) bytes, 256-byte
 *              aligned; no initialisation needed (fp32 D, dQ, dK, dV accumulators).
 * Kernels enqueued on stream: prep, main, finalize -- or, for bf16 with d in {64, 128}
 * (tcgen05 tensor cores, bf16 operands, fp32 accumulation), prep, main over the summary
 * tiles, chain-rule coefficients, main over the local tiles (which applies them and writes
 * dK/dV), dQ conversion.  The main pass is fp32 SIMT otherwise. */
size_t eva_backward_workspace_bytes(const eva_config* cfg);
eva_status eva_attn_backward(const eva_config* cfg, const void* Q, const void* K, const void* V,
                             const void* Ksum, const void* Vsum, const void* O, const float* lse,
                             const void* dO, const float* eps, void* dQ, void* dK, void* dV,
                             void* workspace, size_t workspace_bytes, eva_stream_t stream);

/* eva_attn_backward_proj: eva_attn_backward when the summaries came from eva_summarize_proj
 * (the learned summary-key projection of SURVEY §8(f) NEXT row 4, reading R17:
 * k~_c = Pk[h] mean_c, mu_c = k~_c in Eq.15).  Through the summaries, with g_c the total
 * gradient of k~_c (from the attention plus lambda * clip-gate * d omega):
 *   d mean_c = Pk[h]^T g_c  (spread over the chunk's rows / C),   dPk[h] = sum_{u of head h, c} g_c mean_c^T.
 * Pk    : device fp32 [H, d, d] row-major (as given to eva_summarize_proj), read only
 * dPk   : device fp32 [H, d, d], OVERWRITTEN with the sum over this call's units of each head
 *         (heads with no unit in [bh_begin, bh_begin + bh_count) get zeros); callers sharding
 *         (b,h) across ranks sum dPk over the ranks
 * workspace_bytes >= eva_backward_proj_workspace_bytes(cfg).  bf16, d in {32, 64, 128} and a
 * chunk the register finalize takes (C <= 32 * 8 * 2 / (d * 2 / 16) rows), else
 * EVA_ERR_UNSUPPORTED; causal modes, summary_bias 0. */
size_t eva_backward_proj_workspace_bytes(const eva_config* cfg);
eva_status eva_attn_backward_proj(const eva_config* cfg, const float* Pk, const void* Q, const void* K,
                                  const void* V, const void* Ksum, const void* Vsum, const void* O,
                                  const float* lse, const void* dO, const float* eps, void* dQ, void* dK,
                                  void* dV, float* dPk, void* workspace, size_t workspace_bytes,
                                  eva_stream_t stream);

/* ---------------------------------------------------------------- debug / introspection
 * eva_mask_ranges: the (lo(n), nsum(n)) the kernels use, for n in
 * [n_begin, n_begin + count), written to device int64 arrays lo, nsum
 * (bit-exact mask tests).  Uses cfg.chunk, cfg.window, cfg.mode only. */
eva_status eva_mask_ranges(const eva_config* cfg, int64_t n_begin, int64_t count, int64_t* lo,
                           int64_t* nsum, eva_stream_t stream);

/* eva_philox: the device Philox4x32-10 on n blocks.  in: [n, 6] uint32
 * (ctr0..ctr3, key0, key1), out: [n, 4] uint32.  Device pointers. */
eva_status eva_philox(const uint32_t* in, uint32_t* out, int32_t n, eva_stream_t stream);

/* eva_draw_eps: the eps the kernels draw when eps == NULL, materialised as
 * [bh_count, nC, d] fp32 (nC = floor(cfg.T / C)). */
eva_status eva_draw_eps(const eva_config* cfg, float* eps, eva_stream_t stream);

/* Thread-local text of the last non-OK status ("" if none). */
const char* eva_last_error(void);
/* Library version string, e.g. "flasheva-b200 0.1 sm_100a". */
const char* eva_version(void);
/* Number of kernels this library enqueued since load (a per-process counter). */
uint64_t eva_launch_count(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* EVA_H_ */
