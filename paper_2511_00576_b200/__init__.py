"""paper_2511_00576_b200 -- B200-native FlashEVA attention hot path (arxiv 2511.00576).

libeva.so (CUDA, sm_100a) exposes the C ABI in include/eva.h; ``api`` is the
thin torch binding with the same names.  Importing this package loads
libeva.so and fails loudly if it has not been built.
"""
from .api import (DecodeCache, EvaConfig, EvaError, HostPrefill, eva_attn_prefill_host,  # noqa: F401
                  eva_attn_prefill_range, eva_summarize_range, eva_summarize_range_bcast, eva_attn_backward, eva_attn_decode,  # noqa: F401
                  eva_attn_prefill, eva_prefill_reserve, eva_backward_workspace_bytes,
                  eva_cache_append, eva_cache_load, eva_draw_eps, eva_mask_ranges, eva_philox, eva_summarize, eva_summarize_proj, eva_rope_summarize, eva_rope,
                  eva_attn_prefill_rope,
                  launch_count, make_config, version)

__version__ = "0.1.0"
