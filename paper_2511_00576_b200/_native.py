"""ctypes declarations of libeva.so (include/eva.h).  Argument marshalling only.

The library is loaded from this package directory; if it is missing the import
fails loudly (there is no CPU or eager fallback of any kind).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# EVA_LIB_PATH: load another build of the same library (scripts/mutation_check.sh runs the
# parity tests against deliberately broken builds to show they fail); default: in-tree.
LIB_PATH = os.environ.get("EVA_LIB_PATH") or os.path.join(_HERE, "libeva.so")

EVA_OK, EVA_ERR_INVALID_ARG, EVA_ERR_UNSUPPORTED, EVA_ERR_CAPACITY, EVA_ERR_CUDA = range(5)
EVA_F32, EVA_BF16 = 0, 1
EVA_WINDOW_SLIDING, EVA_WINDOW_BLOCK, EVA_NONCAUSAL = 0, 1, 2
EVA_OMEGA_AS_PRINTED, EVA_OMEGA_SHIFTED_NOISE = 0, 1
EVA_SUMMARIES_PROVIDED = 1
EVA_ROPE_K_ROTATED = 512
EVA_SUMMARIES_FUSED = 2
EVA_PREFILL_SIMT = 4
EVA_SUMMARIES_SEPARATE = 16
EVA_PREFILL_OVERLAP = 128
EVA_ROPE_INTERLEAVED, EVA_ROPE_NEOX = 0, 1

_STATUS = {0: "EVA_OK", 1: "EVA_ERR_INVALID_ARG", 2: "EVA_ERR_UNSUPPORTED", 3: "EVA_ERR_CAPACITY",
           4: "EVA_ERR_CUDA"}


class EvaConfig(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("H", ctypes.c_int32),
                ("bh_begin", ctypes.c_int32), ("bh_count", ctypes.c_int32),
                ("T", ctypes.c_int32), ("d_head", ctypes.c_int32),
                ("chunk", ctypes.c_int32), ("window", ctypes.c_int32),
                ("samples", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("omega_mode", ctypes.c_int32),
                ("scale", ctypes.c_float), ("lambda_", ctypes.c_float), ("clip", ctypes.c_float),
                ("layer", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("summary_bias", ctypes.c_float), ("reserved", ctypes.c_int32)]


class EvaRopeParams(ctypes.Structure):
    _fields_ = [("base", ctypes.c_float), ("rotary_dim", ctypes.c_int32), ("style", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class EvaCache(ctypes.Structure):
    _fields_ = [("cfg", EvaConfig), ("pos", ctypes.c_int64), ("cap_chunks", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("ring_k", ctypes.c_void_p),
                ("ring_v", ctypes.c_void_p), ("sum_k", ctypes.c_void_p), ("sum_v", ctypes.c_void_p)]


EXPORTS = ["eva_config_default", "eva_summarize", "eva_attn_prefill", "eva_cache_append", "eva_cache_load",
           "eva_attn_decode", "eva_decode_workspace_bytes", "eva_mask_ranges", "eva_philox",
           "eva_draw_eps", "eva_last_error", "eva_version", "eva_launch_count",
           "eva_debug_trace_prefill", "eva_decode_step", "eva_backward_workspace_bytes",
           "eva_attn_backward", "eva_pipeline_create", "eva_pipeline_destroy", "eva_attn_prefill_host",
           "eva_summarize_range", "eva_attn_prefill_range", "eva_summarize_range_bcast",
           "eva_summarize_proj", "eva_decode_ragged_workspace_bytes", "eva_decode_step_ragged",
           "eva_rope_summarize", "eva_rope", "eva_prefill_reserve", "eva_rope_ex",
           "eva_rope_summarize_ex", "eva_backward_proj_workspace_bytes", "eva_attn_backward_proj",
           "eva_attn_prefill_rope", "eva_decode_step_ragged_rope"]


class EvaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2511_00576_b200.build` "
                          "(there is no fallback path)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    CFG = ctypes.POINTER(EvaConfig)
    CACHE = ctypes.POINTER(EvaCache)
    st = ctypes.c_int
    sig = {
        "eva_config_default": (None, [CFG] + [ctypes.c_int32] * 6),
        "eva_summarize": (st, [CFG, P, P, P, P, P, P]),
        "eva_summarize_proj": (st, [CFG, P, P, P, P, P, P, P]),
        "eva_rope_summarize": (st, [CFG, ctypes.c_float, P, P, P, P, P, P, P, P, P]),
        "eva_rope": (st, [CFG, ctypes.c_float, P, P, ctypes.c_int64, ctypes.c_int32, P]),
        "eva_rope_ex": (st, [CFG, ctypes.POINTER(EvaRopeParams), P, P, ctypes.c_int64, P, ctypes.c_int32, P]),
        "eva_rope_summarize_ex": (st, [CFG, ctypes.POINTER(EvaRopeParams), P, P, P, P, P, P, P, P, P]),
        "eva_attn_prefill_rope": (st, [CFG, ctypes.POINTER(EvaRopeParams), P, P, P, P, P, P, P, P,
                                       ctypes.c_uint32, P]),
        "eva_decode_ragged_workspace_bytes": (ctypes.c_size_t, [CACHE]),
        "eva_decode_step_ragged": (st, [CACHE, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]),
        "eva_decode_step_ragged_rope": (st, [CACHE, P, ctypes.POINTER(EvaRopeParams), P, P, P, P, P, P, P,
                                             ctypes.c_size_t, P]),
        "eva_attn_prefill": (st, [CFG, P, P, P, P, P, P, P, P, ctypes.c_uint32, P]),
        "eva_prefill_reserve": (st, [CFG, P]),
        "eva_cache_append": (st, [CACHE, P, P, ctypes.c_int32, P, P]),
        "eva_attn_decode": (st, [CACHE, P, P, P, P, ctypes.c_size_t, P]),
        "eva_cache_load": (st, [CACHE, P, P, P, P, ctypes.c_int32, P]),
        "eva_decode_step": (st, [CACHE, P, P, P, P, P, P, P, ctypes.c_size_t, P]),
        "eva_decode_workspace_bytes": (ctypes.c_size_t, [CACHE]),
        "eva_backward_workspace_bytes": (ctypes.c_size_t, [CFG]),
        "eva_attn_backward": (st, [CFG] + [P] * 13 + [ctypes.c_size_t, P]),
        "eva_backward_proj_workspace_bytes": (ctypes.c_size_t, [CFG]),
        "eva_attn_backward_proj": (st, [CFG] + [P] * 15 + [ctypes.c_size_t, P]),
        "eva_mask_ranges": (st, [CFG, ctypes.c_int64, ctypes.c_int64, P, P, P]),
        "eva_philox": (st, [P, P, ctypes.c_int32, P]),
        "eva_draw_eps": (st, [CFG, P, P]),
        "eva_last_error": (ctypes.c_char_p, []),
        "eva_version": (ctypes.c_char_p, []),
        "eva_launch_count": (ctypes.c_uint64, []),
        "eva_debug_trace_prefill": (st, [CFG, P, P, P, P, P, P, P, P, ctypes.c_int32, P]),
        "eva_summarize_range": (st, [CFG, ctypes.c_int32, P, P, P, P, P, P]),
        "eva_summarize_range_bcast": (st, [CFG, ctypes.c_int32, P, P, P, P, P, ctypes.c_int32, ctypes.c_int32, P]),
        "eva_attn_prefill_range": (st, [CFG, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                        P, P, P, P, P, ctypes.c_int32, P, P, ctypes.c_uint32, P]),
        "eva_pipeline_create": (st, [ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
        "eva_pipeline_destroy": (None, [P]),
        "eva_attn_prefill_host": (st, [P, CFG] + [P] * 13 + [ctypes.c_uint32, ctypes.c_int32, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status != EVA_OK:
        raise EvaError(status, lib.eva_last_error().decode())
