"""CPU-side checks of libeva.so: it loads, exports every symbol include/eva.h
declares, and its synchronous host logic (defaults, argument validation,
capacity accounting, workspace sizing) behaves as documented.  No kernel is
launched here (there is no GPU on the build host)."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in sorted(os.listdir(os.path.join(ROOT, "include")))
           if h.endswith(".h")]


@pytest.fixture(scope="module")
def N():
    from paper_2511_00576_b200 import _native
    return _native


def _declared():
    src = "\n".join(open(h).read() for h in HEADERS)
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eva_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(N):
    names = _declared()
    assert "eva_attn_prefill" in names and "eva_cache_append" in names
    for nm in names:
        assert hasattr(N.lib, nm), nm
    assert set(names) == set(N.EXPORTS)


def test_struct_layouts_match_header(N):
    assert ctypes.sizeof(N.EvaConfig) == 16 * 4 + 8 + 2 * 4  # 16 x 4-byte fields + u64 + bias, reserved
    assert N.EvaConfig.seed.offset == 64
    assert N.EvaConfig.summary_bias.offset == 72
    assert N.EvaCache.pos.offset == ctypes.sizeof(N.EvaConfig)
    assert N.EvaCache.ring_k.offset == ctypes.sizeof(N.EvaConfig) + 16


def test_config_defaults(N):
    cfg = N.EvaConfig()
    N.lib.eva_config_default(ctypes.byref(cfg), 8, 32, 8192, 128, 64, 256)
    assert (cfg.B, cfg.H, cfg.bh_begin, cfg.bh_count) == (8, 32, 0, 256)
    assert (cfg.T, cfg.d_head, cfg.chunk, cfg.window, cfg.samples) == (8192, 128, 64, 256, 1)
    assert cfg.mode == N.EVA_WINDOW_SLIDING and cfg.dtype == N.EVA_BF16
    assert abs(cfg.scale - 1 / math.sqrt(128)) < 1e-7
    assert abs(cfg.lambda_ - 0.1) < 1e-7 and cfg.clip == 1.0
    assert N.lib.eva_version().decode().startswith("flasheva-b200")


def _cfg(N, **kw):
    cfg = N.EvaConfig()
    N.lib.eva_config_default(ctypes.byref(cfg), 1, 2, 64, 32, 8, 16)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


FAKE = ctypes.c_void_p(0x10000)  # aligned, never dereferenced: validation fails first


@pytest.mark.parametrize("field,value,status", [
    ("window", 12, 1), ("chunk", 0, 1), ("T", 0, 1), ("B", 0, 1), ("bh_count", 3, 1),
    ("bh_begin", -1, 1), ("mode", 7, 1), ("dtype", 5, 1), ("omega_mode", 2, 1),
    ("samples", 2, 2), ("d_head", 48, 2), ("d_head", 256, 2)])
def test_validation_rejects_bad_configs(N, field, value, status):
    cfg = _cfg(N, **{field: value})
    st = N.lib.eva_summarize(ctypes.byref(cfg), FAKE, FAKE, None, FAKE, FAKE, None)
    assert st == status
    assert len(N.lib.eva_last_error()) > 0
    st = N.lib.eva_attn_prefill(ctypes.byref(cfg), FAKE, FAKE, FAKE, FAKE, FAKE, None, FAKE, None, 0, None)
    assert st == status


def test_validation_rejects_null_and_misaligned_pointers(N):
    cfg = _cfg(N)
    st = N.lib.eva_attn_prefill(ctypes.byref(cfg), None, FAKE, FAKE, FAKE, FAKE, None, FAKE, None, 0, None)
    assert st == N.EVA_ERR_INVALID_ARG and b"Q" in N.lib.eva_last_error()
    st = N.lib.eva_attn_prefill(ctypes.byref(cfg), FAKE, ctypes.c_void_p(0x10002), FAKE, FAKE, FAKE,
                                None, FAKE, None, 0, None)
    assert st == N.EVA_ERR_INVALID_ARG and b"aligned" in N.lib.eva_last_error()
    st = N.lib.eva_attn_prefill(ctypes.byref(cfg), FAKE, FAKE, FAKE, FAKE, FAKE, None, FAKE, None, 0x4000, None)
    assert st == N.EVA_ERR_INVALID_ARG


def _cache(N, pos, cap, **kw):
    c = N.EvaCache()
    c.cfg = _cfg(N, **kw)
    c.pos = pos
    c.cap_chunks = cap
    c.ring_k = c.ring_v = c.sum_k = c.sum_v = 0x10000
    return c


def test_cache_capacity_and_position_logic(N):
    c = _cache(N, 0, 2)  # C = 8: room for 2 summaries -> positions < 24
    assert N.lib.eva_cache_append(ctypes.byref(c), FAKE, FAKE, 24, None, None) == N.EVA_ERR_CAPACITY
    assert c.pos == 0  # unchanged on failure
    assert N.lib.eva_cache_append(ctypes.byref(c), FAKE, FAKE, 0, None, None) == N.EVA_ERR_INVALID_ARG
    d = _cache(N, 0, 1)
    assert N.lib.eva_attn_decode(ctypes.byref(d), FAKE, FAKE, None, None, 0, None) == N.EVA_ERR_INVALID_ARG
    e = _cache(N, 40, 1)  # query 39: nsum = 39//8 - 2 + 1 = 3 > cap 1
    assert N.lib.eva_attn_decode(ctypes.byref(e), FAKE, FAKE, None, None, 0, None) == N.EVA_ERR_CAPACITY


def test_decode_workspace_bytes(N):
    small = _cache(N, 1, 4)  # 2 units, 1 visible entry -> a single split, no workspace
    assert N.lib.eva_decode_workspace_bytes(ctypes.byref(small)) == 0
    long = _cache(N, 4000, 600, bh_count=2)
    ws = N.lib.eva_decode_workspace_bytes(ctypes.byref(long))
    # one merge counter per unit at the front (padded to 16 bytes), then (m, l, acc[d]) per
    # (unit, split); the counters' offset does not depend on the split count
    assert ws > 0 and (ws - 16) % (2 * (32 + 2) * 4) == 0


def test_product_package_does_not_import_oracle():
    """The product path never imports oracle/ (DESIGN.md §4)."""
    pkg = os.path.join(ROOT, "paper_2511_00576_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "eva_oracle" not in txt and "liboracle" not in txt, f


def test_backward_workspace_and_validation(N):
    cfg = _cfg(N)  # bh 2, T 64, d 32, C 8 -> nC 8
    ws = N.lib.eva_backward_workspace_bytes(ctypes.byref(cfg))

    def a256(x):
        return (x + 255) // 256 * 256
    # fp32: D [bh,T], dQ/dK/dV [bh,T,d], d k~ / d beta [bh,nC,d]
    assert ws == a256(2 * 64 * 4) + 3 * a256(2 * 64 * 32 * 4) + 2 * a256(2 * 8 * 32 * 4)
    args = [FAKE] * 13  # Q K V Ksum Vsum O lse dO eps dQ dK dV workspace
    bw = N.lib.eva_attn_backward
    # a NULL gradient output is rejected with its name
    a = list(args)
    a[10] = None  # dK
    assert bw(ctypes.byref(cfg), *a, ws, None) == N.EVA_ERR_INVALID_ARG
    assert b"dK" in N.lib.eva_last_error()
    # too small a workspace
    assert bw(ctypes.byref(cfg), *args, ws - 1, None) == N.EVA_ERR_INVALID_ARG
    assert b"workspace_bytes" in N.lib.eva_last_error()
    # a workspace that is 16- but not 256-byte aligned
    a = list(args)
    a[12] = ctypes.c_void_p(0x10010)
    assert bw(ctypes.byref(cfg), *a, ws, None) == N.EVA_ERR_INVALID_ARG
    assert b"256-byte" in N.lib.eva_last_error()
    bad = _cfg(N, samples=2)
    assert bw(ctypes.byref(bad), *args, ws, None) == N.EVA_ERR_UNSUPPORTED
    assert N.lib.eva_backward_workspace_bytes(ctypes.byref(bad)) == 0


def test_host_pipeline_validation(N):
    """eva_pipeline_create / eva_attn_prefill_host argument checks (synchronous, no launch)."""
    h = ctypes.c_void_p()
    assert N.lib.eva_pipeline_create(0, ctypes.byref(h)) == N.EVA_ERR_INVALID_ARG
    cfg = N.EvaConfig()
    N.lib.eva_config_default(ctypes.byref(cfg), 1, 2, 64, 64, 16, 32)
    buf = (ctypes.c_uint8 * 64)()
    P = ctypes.cast(buf, ctypes.c_void_p)
    args = [P] * 4 + [None] + [P] * 6 + [None, None]
    assert N.lib.eva_attn_prefill_host(None, ctypes.byref(cfg), *args, 0, 1, None) == N.EVA_ERR_INVALID_ARG
    assert b"pipe" in N.lib.eva_last_error()


def test_summarize_proj_validation(N):
    """eva_summarize_proj: NULL or misaligned Pk is EVA_ERR_INVALID_ARG before anything runs."""
    buf = (ctypes.c_uint8 * 4096)()
    P = ctypes.cast(buf, ctypes.c_void_p)
    cfg = N.EvaConfig()
    N.lib.eva_config_default(ctypes.byref(cfg), 1, 1, 64, 64, 16, 32)
    assert N.lib.eva_summarize_proj(ctypes.byref(cfg), P, P, None, None, P, P, None) == N.EVA_ERR_INVALID_ARG
    assert b"Pk" in N.lib.eva_last_error()
    mis = ctypes.c_void_p(ctypes.addressof(buf) + 4)
    assert N.lib.eva_summarize_proj(ctypes.byref(cfg), P, P, None, mis, P, P, None) == N.EVA_ERR_INVALID_ARG


def test_decode_ragged_validation(N):
    """eva_decode_step_ragged: NULL pos is EVA_ERR_INVALID_ARG, the non-causal partition is
    EVA_ERR_UNSUPPORTED; the ragged workspace covers the longest position the cache holds."""
    buf = (ctypes.c_uint8 * 4096)()
    P = ctypes.cast(buf, ctypes.c_void_p)
    cache = N.EvaCache()
    N.lib.eva_config_default(ctypes.byref(cache.cfg), 1, 4, 0, 64, 16, 32)
    cache.cap_chunks = 8
    cache.ring_k = cache.ring_v = cache.sum_k = cache.sum_v = ctypes.addressof(buf)
    args = (P, P, P, None, P, None, P, 1 << 20, None)
    assert N.lib.eva_decode_step_ragged(ctypes.byref(cache), None, *args) == N.EVA_ERR_INVALID_ARG
    assert b"pos" in N.lib.eva_last_error()
    assert N.lib.eva_decode_ragged_workspace_bytes(ctypes.byref(cache)) >= \
        N.lib.eva_decode_workspace_bytes(ctypes.byref(cache))
    cache.cfg.mode = N.EVA_NONCAUSAL
    assert N.lib.eva_decode_step_ragged(ctypes.byref(cache), P, *args) == N.EVA_ERR_UNSUPPORTED


def test_noncausal_and_bias_validation(N):
    """Mode EVA_NONCAUSAL: prefill and backward need T % C == 0; decode/cache/range refuse it
    (EVA_ERR_UNSUPPORTED); a non-finite summary_bias or a nonzero reserved field is invalid."""
    buf = (ctypes.c_uint8 * 4096)()
    P = ctypes.cast(buf, ctypes.c_void_p)
    cfg = N.EvaConfig()
    N.lib.eva_config_default(ctypes.byref(cfg), 1, 1, 70, 64, 16, 32)
    assert cfg.summary_bias == 0.0 and cfg.reserved == 0
    cfg.mode = N.EVA_NONCAUSAL
    assert N.lib.eva_attn_prefill(ctypes.byref(cfg), P, P, P, P, P, None, P, None, 0, None) == N.EVA_ERR_INVALID_ARG
    assert b"T % C" in N.lib.eva_last_error()
    cache = N.EvaCache()
    cache.cfg = cfg
    cache.cap_chunks = 4
    cache.ring_k = cache.ring_v = cache.sum_k = cache.sum_v = ctypes.addressof(buf)
    assert N.lib.eva_cache_append(ctypes.byref(cache), P, P, 1, None, None) == N.EVA_ERR_UNSUPPORTED
    assert N.lib.eva_attn_prefill_range(ctypes.byref(cfg), 0, 0, 0, 0, P, P, P, P, P, 0, P, None, 0,
                                        None) == N.EVA_ERR_UNSUPPORTED
    # the backward takes the non-causal partition, with the prefill's T % C rule
    assert N.lib.eva_attn_backward(ctypes.byref(cfg), P, P, P, P, P, P, P, P, None, P, P, P, P, 1 << 30,
                                   None) == N.EVA_ERR_INVALID_ARG
    assert b"T % chunk" in N.lib.eva_last_error()
    cfg.mode = N.EVA_WINDOW_SLIDING
    cfg.summary_bias = float("inf")
    assert N.lib.eva_summarize(ctypes.byref(cfg), P, P, None, P, P, None) == N.EVA_ERR_INVALID_ARG
    cfg.summary_bias = 0.0
    cfg.reserved = 1
    assert N.lib.eva_summarize(ctypes.byref(cfg), P, P, None, P, P, None) == N.EVA_ERR_INVALID_ARG


def test_rope_entry_points_validate_before_any_launch(N):
    """eva_attn_prefill_rope / eva_decode_step_ragged_rope: the RoPE parameters and flags are
    checked synchronously (nothing is enqueued; no GPU needed for these paths)."""
    cfg = _cfg(N, dtype=N.EVA_BF16, d_head=64)
    good = N.EvaRopeParams(10000.0, 0, N.EVA_ROPE_INTERLEAVED, 0)
    args = (FAKE, FAKE, FAKE, None, FAKE, FAKE, FAKE, None)
    for rp in (N.EvaRopeParams(0.5, 0, 0, 0), N.EvaRopeParams(float("inf"), 0, 0, 0),
               N.EvaRopeParams(10000.0, 0, 7, 0), N.EvaRopeParams(10000.0, 0, 0, 1),
               N.EvaRopeParams(10000.0, 24, 0, 0), N.EvaRopeParams(10000.0, 80, 0, 0)):
        st = N.lib.eva_attn_prefill_rope(ctypes.byref(cfg), ctypes.byref(rp), *args, 0, None)
        assert st == N.EVA_ERR_INVALID_ARG, (rp.base, rp.rotary_dim, rp.style, rp.reserved)
    # unknown flags (EVA_SUMMARIES_FUSED is not a RoPE prefill flag)
    st = N.lib.eva_attn_prefill_rope(ctypes.byref(cfg), ctypes.byref(good), *args, 2, None)
    assert st == N.EVA_ERR_INVALID_ARG and b"flags" in N.lib.eva_last_error()
    # half-split with rotary_dim / 16 = 3: no butterfly partner
    st = N.lib.eva_attn_prefill_rope(ctypes.byref(_cfg(N, dtype=N.EVA_BF16, d_head=64)),
                                     ctypes.byref(N.EvaRopeParams(10000.0, 48, N.EVA_ROPE_NEOX, 0)), *args, 0, None)
    assert st == N.EVA_ERR_UNSUPPORTED
    c = _cache(N, 0, 4, dtype=N.EVA_BF16, d_head=64)
    bad = N.EvaRopeParams(1.0, 0, 0, 0)
    st = N.lib.eva_decode_step_ragged_rope(ctypes.byref(c), FAKE, ctypes.byref(bad), FAKE, FAKE, FAKE, None,
                                           FAKE, None, FAKE, 1 << 20, None)
    assert st == N.EVA_ERR_INVALID_ARG and b"base" in N.lib.eva_last_error()
    st = N.lib.eva_decode_step_ragged_rope(None, FAKE, ctypes.byref(good), FAKE, FAKE, FAKE, None,
                                           FAKE, None, FAKE, 1 << 20, None)
    assert st == N.EVA_ERR_INVALID_ARG
