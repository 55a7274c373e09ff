/*
 * eva_debug.h -- developer introspection of libeva.so (not part of the product API).
 */
#ifndef EVA_DEBUG_H_
#define EVA_DEBUG_H_
#include "eva.h"
#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
/* Run the persistent tensor-core prefill (summaries provided) with CTA 0 recording its
 * pipeline timeline: trace[i] = clock64 << 24 | kind << 20 | tile << 16 | index, up to
 * cap entries (device pointer).  With cap < 65536 the one-tile-per-CTA kernel is traced
 * instead (CTAs 0, 1, 150, 151; 4 x 4 x 48 entries), followed by every CTA's entry and exit
 * globaltimer (ns) at trace[768 + 2 * cta + {0, 1}] for cta < 4096.  Event kinds: prefill_sm100.cu. */
eva_status eva_debug_trace_prefill(const eva_config* cfg, const void* Q, const void* K,
                                   const void* V, const void* Ksum, const void* Vsum, void* O,
                                   float* lse, unsigned long long* trace, int32_t cap,
                                   eva_stream_t stream);
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif
