// prefill_sm100.cu -- tcgen05/TMEM/TMA bf16 FlashEVA prefill (placeholder until the
// tensor-core kernel lands; the SIMT kernel serves every shape meanwhile).
#include "launch.h"

namespace eva {
bool prefill_sm100_supported(const eva_config&) { return false; }
cudaError_t launch_prefill_sm100(const eva_config&, const void*, const void*, const void*,
                                 const void*, const void*, void*, float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace eva
