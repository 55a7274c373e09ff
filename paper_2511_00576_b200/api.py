"""Thin torch-facing binding of libeva.so with the C ABI's names (include/eva.h).

Argument marshalling only: every step of the FlashEVA path runs in the CUDA
kernels behind the C ABI.  Tensors must be CUDA, contiguous, of the dtype the
config names; outputs are allocated with torch (the library allocates nothing).
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional

import torch

from . import _native as N
from ._native import EvaCache, EvaConfig, EvaError, check, lib

__all__ = ["make_config", "eva_summarize", "eva_attn_prefill", "eva_cache_append", "eva_cache_load",
           "eva_attn_decode", "DecodeCache", "eva_mask_ranges", "eva_philox", "eva_draw_eps",
           "EvaConfig", "EvaError", "launch_count", "version", "eva_attn_backward",
           "eva_backward_workspace_bytes", "HostPrefill", "eva_attn_prefill_host",
           "eva_summarize_range", "eva_attn_prefill_range", "eva_summarize_range_bcast"]

_DT = {torch.float32: N.EVA_F32, torch.bfloat16: N.EVA_BF16}
_MODE = {"sliding": N.EVA_WINDOW_SLIDING, "block": N.EVA_WINDOW_BLOCK, "noncausal": N.EVA_NONCAUSAL}


def version() -> str:
    return lib.eva_version().decode()


def launch_count() -> int:
    """Kernels libeva.so has enqueued in this process."""
    return int(lib.eva_launch_count())


def make_config(B: int, H: int, T: int, d: int, chunk: int, window: int, *, bh_begin: int = 0,
                bh_count: Optional[int] = None, mode: str = "sliding", dtype=torch.bfloat16,
                scale: Optional[float] = None, lam: float = 0.1, clip: float = 1.0,
                seed: int = 1234, layer: int = 0, omega_mode: int = 0, samples: int = 1,
                summary_bias: float = 0.0) -> EvaConfig:
    cfg = EvaConfig()
    lib.eva_config_default(ctypes.byref(cfg), B, H, T, d, chunk, window)
    cfg.bh_begin = bh_begin
    cfg.bh_count = B * H - bh_begin if bh_count is None else bh_count
    cfg.mode = _MODE[mode] if isinstance(mode, str) else int(mode)
    cfg.dtype = _DT[dtype]
    cfg.scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    cfg.lambda_ = lam
    cfg.clip = clip
    cfg.seed = seed
    cfg.layer = layer
    cfg.omega_mode = omega_mode
    cfg.samples = samples
    cfg.summary_bias = summary_bias
    return cfg


def _tdtype(cfg) -> torch.dtype:
    return torch.bfloat16 if cfg.dtype == N.EVA_BF16 else torch.float32


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _need(t: torch.Tensor, name: str, shape, dtype) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.dtype != dtype:
        raise ValueError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def eva_summarize(cfg: EvaConfig, K: torch.Tensor, V: torch.Tensor,
                  eps: Optional[torch.Tensor] = None, Ksum: Optional[torch.Tensor] = None,
                  Vsum: Optional[torch.Tensor] = None):
    """Chunk summaries (k~_c, beta^_c) of all complete chunks -> Ksum, Vsum [bh, nC, d]."""
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    nC = T // cfg.chunk
    _need(K, "K", (bh, T, d), dt)
    _need(V, "V", (bh, T, d), dt)
    if eps is not None:
        _need(eps, "eps", (bh, nC, d), torch.float32)
    Ksum = torch.empty(bh, nC, d, dtype=dt, device=K.device) if Ksum is None else Ksum
    Vsum = torch.empty(bh, nC, d, dtype=dt, device=K.device) if Vsum is None else Vsum
    check(lib.eva_summarize(ctypes.byref(cfg), _ptr(K), _ptr(V), _ptr(eps), _ptr(Ksum), _ptr(Vsum),
                            _stream(K.device)))
    return Ksum, Vsum


_ROPE_STYLE = {"interleaved": N.EVA_ROPE_INTERLEAVED, "neox": N.EVA_ROPE_NEOX}


def _rope_params(rope_base, rotary_dim, style):
    return N.EvaRopeParams(float(rope_base), int(rotary_dim or 0),
                           _ROPE_STYLE[style] if isinstance(style, str) else int(style), 0)


def eva_rope_summarize(cfg: EvaConfig, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                       rope_base: float = 10000.0, eps: Optional[torch.Tensor] = None,
                       rotary_dim: Optional[int] = None, style: str = "interleaved"):
    """Fused RoPE producer (NEXT row 4, R18/R19): returns (Qr, Kr, Ksum, Vsum) -- the rotated
    queries/keys and the summaries of the rotated keys, in one launch.  rotary_dim (default d)
    and style ("interleaved" pairs (2j, 2j+1) or "neox" pairs (j, j + rd/2)) as in R19."""
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    nC = T // cfg.chunk
    for t, nm in ((Q, "Q"), (K, "K"), (V, "V")):
        _need(t, nm, (bh, T, d), dt)
    if eps is not None:
        _need(eps, "eps", (bh, nC, d), torch.float32)
    Qr, Kr = torch.empty_like(Q), torch.empty_like(K)
    Ksum = torch.empty(bh, max(nC, 1), d, dtype=dt, device=K.device)[:, :nC]
    Vsum = torch.empty(bh, max(nC, 1), d, dtype=dt, device=K.device)[:, :nC]
    rp = _rope_params(rope_base, rotary_dim, style)
    check(lib.eva_rope_summarize_ex(ctypes.byref(cfg), ctypes.byref(rp), _ptr(Q), _ptr(K), _ptr(V), _ptr(eps),
                                    _ptr(Qr), _ptr(Kr), _ptr(Ksum if nC else None), _ptr(Vsum if nC else None),
                                    _stream(K.device)))
    return Qr, Kr, Ksum, Vsum


def eva_attn_prefill_rope(cfg: EvaConfig, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                          rope_base: float = 10000.0, rotary_dim: Optional[int] = None,
                          style: str = "interleaved", eps: Optional[torch.Tensor] = None,
                          Ksum: Optional[torch.Tensor] = None, Vsum: Optional[torch.Tensor] = None,
                          summaries_provided: bool = False, O: Optional[torch.Tensor] = None,
                          lse: Optional[torch.Tensor] = None, k_rotated: bool = False):
    """Prefill on RoPE(Q), RoPE(K) with the rotation inside the tensor-core kernel (NEXT row 4,
    R18/R19): Q, K un-rotated (k_rotated: K already rotated, only Q is rotated in the kernel).
    Returns (O, lse, Ksum, Vsum); the summaries are those of the rotated keys (computed first
    unless summaries_provided)."""
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    nC = T // cfg.chunk
    for t, nm in ((Q, "Q"), (K, "K"), (V, "V")):
        _need(t, nm, (bh, T, d), dt)
    if eps is not None:
        _need(eps, "eps", (bh, nC, d), torch.float32)
    if summaries_provided:
        _need(Ksum, "Ksum", (bh, nC, d), dt)
        _need(Vsum, "Vsum", (bh, nC, d), dt)
    Ksum = torch.empty(bh, max(nC, 1), d, dtype=dt, device=K.device)[:, :nC] if Ksum is None else Ksum
    Vsum = torch.empty(bh, max(nC, 1), d, dtype=dt, device=K.device)[:, :nC] if Vsum is None else Vsum
    O = torch.empty_like(Q) if O is None else O
    lse = torch.empty(bh, T, dtype=torch.float32, device=Q.device) if lse is None else lse
    rp = _rope_params(rope_base, rotary_dim, style)
    check(lib.eva_attn_prefill_rope(ctypes.byref(cfg), ctypes.byref(rp), _ptr(Q), _ptr(K), _ptr(V), _ptr(eps),
                                    _ptr(Ksum if nC else None), _ptr(Vsum if nC else None), _ptr(O), _ptr(lse),
                                    (N.EVA_SUMMARIES_PROVIDED if summaries_provided else 0) |
                                    (N.EVA_ROPE_K_ROTATED if k_rotated else 0), _stream(Q.device)))
    return O, lse, Ksum, Vsum


def eva_rope(cfg: EvaConfig, X: torch.Tensor, rope_base: float = 10000.0, pos0: int = 0,
             inverse: bool = False, out: Optional[torch.Tensor] = None, rotary_dim: Optional[int] = None,
             style: str = "interleaved", pos: Optional[torch.Tensor] = None) -> torch.Tensor:
    """RoPE (R18/R19) of rows X [bh, T, d]: row t of unit u at position (pos[u] if pos is given,
    a CUDA int64 tensor [bh], else pos0) + t; inverse: the transposed rotation (the gradient
    through RoPE)."""
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    _need(X, "X", (bh, T, d), dt)
    out = torch.empty_like(X) if out is None else out
    _need(out, "out", (bh, T, d), dt)
    if pos is not None:
        _need(pos, "pos", (bh,), torch.int64)
    rp = _rope_params(rope_base, rotary_dim, style)
    check(lib.eva_rope_ex(ctypes.byref(cfg), ctypes.byref(rp), _ptr(X), _ptr(out), int(pos0), _ptr(pos),
                          int(bool(inverse)), _stream(X.device)))
    return out


def eva_summarize_proj(cfg: EvaConfig, K: torch.Tensor, V: torch.Tensor, Pk: torch.Tensor,
                       eps: Optional[torch.Tensor] = None, Ksum: Optional[torch.Tensor] = None,
                       Vsum: Optional[torch.Tensor] = None):
    """Chunk summaries with the learned summary-key projection k~ = Pk[h] mean(k)
    (NEXT row 4, reading R17).  Pk: fp32 CUDA [H, d, d] row-major."""
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    nC = T // cfg.chunk
    _need(K, "K", (bh, T, d), dt)
    _need(V, "V", (bh, T, d), dt)
    _need(Pk, "Pk", (cfg.H, d, d), torch.float32)
    if eps is not None:
        _need(eps, "eps", (bh, nC, d), torch.float32)
    Ksum = torch.empty(bh, nC, d, dtype=dt, device=K.device) if Ksum is None else Ksum
    Vsum = torch.empty(bh, nC, d, dtype=dt, device=K.device) if Vsum is None else Vsum
    check(lib.eva_summarize_proj(ctypes.byref(cfg), _ptr(K), _ptr(V), _ptr(eps), _ptr(Pk), _ptr(Ksum),
                                 _ptr(Vsum), _stream(K.device)))
    return Ksum, Vsum


def eva_attn_prefill(cfg: EvaConfig, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, *,
                     eps: Optional[torch.Tensor] = None, Ksum: Optional[torch.Tensor] = None,
                     Vsum: Optional[torch.Tensor] = None, summaries_provided: bool = False,
                     want_lse: bool = True, simt: bool = False, O: Optional[torch.Tensor] = None,
                     lse: Optional[torch.Tensor] = None, kernel: Optional[str] = None,
                     overlap: bool = False):
    """FlashEVA chunk-causal prefill.  Returns (O, lse, Ksum, Vsum).

    kernel: None or "separate" (EVA_SUMMARIES_SEPARATE: summarize launch + tcgen05 kernel),
    "fused" (EVA_SUMMARIES_FUSED: in-kernel summaries, one launch; an error where they do not
    apply) or "simt" (the fp32-capable SIMT kernel, separate summaries)."""
    if kernel == "simt":
        simt = True
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    nC = T // cfg.chunk
    for t, nm in ((Q, "Q"), (K, "K"), (V, "V")):
        _need(t, nm, (bh, T, d), dt)
    if summaries_provided:
        if Ksum is None or Vsum is None:
            raise ValueError("summaries_provided needs Ksum and Vsum")
    if Ksum is None:
        Ksum = torch.empty(bh, max(nC, 1), d, dtype=dt, device=Q.device)[:, :nC]
    if Vsum is None:
        Vsum = torch.empty(bh, max(nC, 1), d, dtype=dt, device=Q.device)[:, :nC]
    if nC:
        _need(Ksum, "Ksum", (bh, nC, d), dt)
        _need(Vsum, "Vsum", (bh, nC, d), dt)
    if eps is not None:
        _need(eps, "eps", (bh, nC, d), torch.float32)
    O = torch.empty_like(Q) if O is None else O
    _need(O, "O", (bh, T, d), dt)
    if want_lse and lse is None:
        lse = torch.empty(bh, T, dtype=torch.float32, device=Q.device)
    flags = (N.EVA_SUMMARIES_PROVIDED if summaries_provided else 0) | (N.EVA_PREFILL_SIMT if simt else 0)
    if not summaries_provided:
        flags |= {None: 0, "simt": 0, "fused": N.EVA_SUMMARIES_FUSED,
                  "separate": N.EVA_SUMMARIES_SEPARATE}[kernel]
    elif kernel not in (None, "simt", "separate"):
        raise ValueError(f"kernel={kernel!r} with summaries_provided")
    if overlap:  # the previous launch on this stream is the eva_summarize writing Ksum/Vsum
        flags |= N.EVA_PREFILL_OVERLAP
    check(lib.eva_attn_prefill(ctypes.byref(cfg), _ptr(Q), _ptr(K), _ptr(V), _ptr(Ksum), _ptr(Vsum),
                               _ptr(eps), _ptr(O), _ptr(lse if want_lse else None), flags,
                               _stream(Q.device)))
    return O, (lse if want_lse else None), Ksum, Vsum


def eva_prefill_reserve(cfg: EvaConfig, device="cuda") -> None:
    """Allocate the library's fused-summary workspace for cfg's shape on the current stream of
    `device` (call before capturing eva_attn_prefill into a CUDA graph)."""
    check(lib.eva_prefill_reserve(ctypes.byref(cfg), _stream(torch.device(device))))


def eva_summarize_range(cfg: EvaConfig, chunk0: int, K: torch.Tensor, V: torch.Tensor,
                        eps: Optional[torch.Tensor] = None, Ksum: Optional[torch.Tensor] = None,
                        Vsum: Optional[torch.Tensor] = None):
    """Summaries of the complete chunks of rows that start at absolute chunk `chunk0`
    (K, V [bh, cfg.T, d]) -> Ksum, Vsum [bh, cfg.T // C, d] for chunks chunk0 + c."""
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    nC = T // cfg.chunk
    _need(K, "K", (bh, T, d), dt)
    _need(V, "V", (bh, T, d), dt)
    if eps is not None:
        _need(eps, "eps", (bh, nC, d), torch.float32)
    Ksum = torch.empty(bh, nC, d, dtype=dt, device=K.device) if Ksum is None else Ksum
    Vsum = torch.empty(bh, nC, d, dtype=dt, device=K.device) if Vsum is None else Vsum
    check(lib.eva_summarize_range(ctypes.byref(cfg), chunk0, _ptr(K), _ptr(V), _ptr(eps), _ptr(Ksum),
                                  _ptr(Vsum), _stream(K.device)))
    return Ksum, Vsum


def eva_summarize_range_bcast(cfg: EvaConfig, chunk0: int, K: torch.Tensor, V: torch.Tensor,
                              dst_ksum_ptrs: torch.Tensor, dst_vsum_ptrs: torch.Tensor, dst_rows: int,
                              eps: Optional[torch.Tensor] = None) -> None:
    """Summaries of chunks [chunk0, chunk0 + cfg.T // C) stored to row chunk0 + c of every
    destination: dst_*_ptrs are int64 CUDA tensors of device addresses of [bh, dst_rows, d]
    buffers (e.g. symmetric-memory peer pointers)."""
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    _need(K, "K", (bh, T, d), dt)
    _need(V, "V", (bh, T, d), dt)
    n = dst_ksum_ptrs.numel()
    for t, nm in ((dst_ksum_ptrs, "dst_ksum_ptrs"), (dst_vsum_ptrs, "dst_vsum_ptrs")):
        _need(t, nm, (n,), torch.int64)
    if eps is not None:
        _need(eps, "eps", (bh, T // cfg.chunk, d), torch.float32)
    check(lib.eva_summarize_range_bcast(ctypes.byref(cfg), chunk0, _ptr(K), _ptr(V), _ptr(eps),
                                        _ptr(dst_ksum_ptrs), _ptr(dst_vsum_ptrs), n, dst_rows,
                                        _stream(K.device)))


def eva_attn_prefill_range(cfg: EvaConfig, q0: int, k0: int, Q: torch.Tensor, K: torch.Tensor,
                           V: torch.Tensor, Ksum: torch.Tensor, Vsum: torch.Tensor, *,
                           want_lse: bool = True, simt: bool = False,
                           O: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None):
    """Prefill of the queries at positions [q0, q0 + Q.shape[1]) given keys/values for
    positions [k0, k0 + K.shape[1]) and the summaries of chunks [0, Ksum.shape[1]).
    Returns (O, lse)."""
    dt, bh, d = _tdtype(cfg), cfg.bh_count, cfg.d_head
    nq, nkv, ns = Q.shape[1], K.shape[1], Ksum.shape[1]
    _need(Q, "Q", (bh, nq, d), dt)
    _need(K, "K", (bh, nkv, d), dt)
    _need(V, "V", (bh, nkv, d), dt)
    if ns:
        _need(Ksum, "Ksum", (bh, ns, d), dt)
        _need(Vsum, "Vsum", (bh, ns, d), dt)
    O = torch.empty_like(Q) if O is None else O
    _need(O, "O", (bh, nq, d), dt)
    if want_lse and lse is None:
        lse = torch.empty(bh, nq, dtype=torch.float32, device=Q.device)
    check(lib.eva_attn_prefill_range(ctypes.byref(cfg), q0, nq, k0, nkv, _ptr(Q), _ptr(K), _ptr(V),
                                     _ptr(Ksum if ns else None), _ptr(Vsum if ns else None), ns, _ptr(O),
                                     _ptr(lse if want_lse else None), N.EVA_PREFILL_SIMT if simt else 0,
                                     _stream(Q.device)))
    return O, (lse if want_lse else None)


class HostPrefill:
    """eva_attn_prefill_host with its pipeline (2 side streams + events) and the device
    staging buffers it copies through (torch-owned, reused across calls).

    After a call, .Q/.K/.V/.O/.Ksum/.Vsum are the device copies (for eva_cache_load)."""

    def __init__(self, cfg: EvaConfig, max_slices: int = 8, device="cuda", want_lse: bool = False):
        dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
        nC = T // cfg.chunk
        self.cfg, self.device = cfg, torch.device(device)
        self.Q, self.K, self.V, self.O = (torch.empty(bh, T, d, dtype=dt, device=device) for _ in range(4))
        self.Ksum = torch.empty(bh, max(nC, 1), d, dtype=dt, device=device)[:, :nC]
        self.Vsum = torch.empty(bh, max(nC, 1), d, dtype=dt, device=device)[:, :nC]
        self.lse = torch.empty(bh, T, dtype=torch.float32, device=device) if want_lse else None
        self.max_slices = max_slices
        h = ctypes.c_void_p()
        check(lib.eva_pipeline_create(max_slices, ctypes.byref(h)))
        self._pipe = h

    def __del__(self):
        if getattr(self, "_pipe", None) is not None and self._pipe.value:
            lib.eva_pipeline_destroy(self._pipe)
            self._pipe = None

    def __call__(self, hQ: torch.Tensor, hK: torch.Tensor, hV: torch.Tensor, hO: torch.Tensor,
                 hlse: Optional[torch.Tensor] = None, eps: Optional[torch.Tensor] = None,
                 n_slices: Optional[int] = None, kernel: Optional[str] = None):
        cfg = self.cfg
        dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
        for t, nm in ((hQ, "hQ"), (hK, "hK"), (hV, "hV"), (hO, "hO")):
            if t.is_cuda or not t.is_contiguous() or t.dtype != dt or tuple(t.shape) != (bh, T, d):
                raise ValueError(f"{nm} must be a contiguous host tensor [{bh}, {T}, {d}] of {dt}")
        if hlse is not None:
            if self.lse is None:
                raise ValueError("HostPrefill(want_lse=True) is needed for hlse")
            if hlse.is_cuda or tuple(hlse.shape) != (bh, T) or hlse.dtype != torch.float32:
                raise ValueError("hlse must be a host fp32 tensor [bh, T]")
        if eps is not None:
            _need(eps, "eps", (bh, T // cfg.chunk, d), torch.float32)
        flags = {None: 0, "simt": N.EVA_PREFILL_SIMT, "fused": N.EVA_SUMMARIES_FUSED,
                 "separate": N.EVA_SUMMARIES_SEPARATE}[kernel]
        check(lib.eva_attn_prefill_host(self._pipe, ctypes.byref(cfg), _ptr(hQ), _ptr(hK), _ptr(hV),
                                        _ptr(hO), _ptr(hlse), _ptr(self.Q), _ptr(self.K), _ptr(self.V),
                                        _ptr(self.Ksum), _ptr(self.Vsum), _ptr(self.O), _ptr(self.lse),
                                        _ptr(eps), flags, n_slices or self.max_slices,
                                        _stream(self.device)))
        return hO


def eva_attn_prefill_host(cfg: EvaConfig, hQ, hK, hV, hO, **kw):
    """One-shot eva_attn_prefill_host (allocates a HostPrefill; keep one for repeated calls)."""
    return HostPrefill(cfg, device=kw.pop("device", "cuda"))(hQ, hK, hV, hO, **kw)


def eva_backward_workspace_bytes(cfg: EvaConfig) -> int:
    return int(lib.eva_backward_workspace_bytes(ctypes.byref(cfg)))


def eva_attn_backward(cfg: EvaConfig, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                      Ksum: torch.Tensor, Vsum: torch.Tensor, O: torch.Tensor, lse: torch.Tensor,
                      dO: torch.Tensor, *, eps: Optional[torch.Tensor] = None,
                      workspace: Optional[torch.Tensor] = None, dQ: Optional[torch.Tensor] = None,
                      dK: Optional[torch.Tensor] = None, dV: Optional[torch.Tensor] = None,
                      Pk: Optional[torch.Tensor] = None, dPk: Optional[torch.Tensor] = None):
    """Gradient of the prefill for L = sum(dO * O).  Returns (dQ, dK, dV), or (dQ, dK, dV, dPk)
    when the summaries came from eva_summarize_proj with the projection Pk [H, d, d] fp32
    (eva_attn_backward_proj, R17; dPk: this call's units' sum per head).

    Ksum/Vsum/O/lse/eps are what eva_attn_prefill used and produced.  workspace: a
    uint8 CUDA tensor of at least eva_backward_workspace_bytes(cfg) (with Pk:
    eva_backward_proj_workspace_bytes) bytes, allocated here when None."""
    dt, bh, T, d = _tdtype(cfg), cfg.bh_count, cfg.T, cfg.d_head
    nC = T // cfg.chunk
    for t, nm in ((Q, "Q"), (K, "K"), (V, "V"), (O, "O"), (dO, "dO")):
        _need(t, nm, (bh, T, d), dt)
    _need(lse, "lse", (bh, T), torch.float32)
    if nC:
        _need(Ksum, "Ksum", (bh, nC, d), dt)
        _need(Vsum, "Vsum", (bh, nC, d), dt)
    if eps is not None:
        _need(eps, "eps", (bh, nC, d), torch.float32)
    dQ = torch.empty_like(Q) if dQ is None else dQ
    dK = torch.empty_like(K) if dK is None else dK
    dV = torch.empty_like(V) if dV is None else dV
    for t, nm in ((dQ, "dQ"), (dK, "dK"), (dV, "dV")):
        _need(t, nm, (bh, T, d), dt)
    if Pk is not None:
        _need(Pk, "Pk", (cfg.H, d, d), torch.float32)
        dPk = torch.empty_like(Pk) if dPk is None else dPk
        _need(dPk, "dPk", (cfg.H, d, d), torch.float32)
        nbytes = int(lib.eva_backward_proj_workspace_bytes(ctypes.byref(cfg)))
    else:
        nbytes = eva_backward_workspace_bytes(cfg)
    if workspace is None:
        workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=Q.device)
    if Pk is not None:
        check(lib.eva_attn_backward_proj(ctypes.byref(cfg), _ptr(Pk), _ptr(Q), _ptr(K), _ptr(V), _ptr(Ksum),
                                         _ptr(Vsum), _ptr(O), _ptr(lse), _ptr(dO), _ptr(eps), _ptr(dQ), _ptr(dK),
                                         _ptr(dV), _ptr(dPk), _ptr(workspace), workspace.numel(),
                                         _stream(Q.device)))
        return dQ, dK, dV, dPk
    check(lib.eva_attn_backward(ctypes.byref(cfg), _ptr(Q), _ptr(K), _ptr(V), _ptr(Ksum), _ptr(Vsum),
                                _ptr(O), _ptr(lse), _ptr(dO), _ptr(eps), _ptr(dQ), _ptr(dK), _ptr(dV),
                                _ptr(workspace), workspace.numel(), _stream(Q.device)))
    return dQ, dK, dV


class DecodeCache:
    """Compressed decode cache: ring [bh, W, d] x2 + summaries [bh, cap, d] x2 (torch-owned)."""

    def __init__(self, cfg: EvaConfig, cap_chunks: int, device="cuda"):
        dt, bh, W, d = _tdtype(cfg), cfg.bh_count, cfg.window, cfg.d_head
        self.ring_k = torch.zeros(bh, W, d, dtype=dt, device=device)
        self.ring_v = torch.zeros(bh, W, d, dtype=dt, device=device)
        self.sum_k = torch.zeros(bh, max(cap_chunks, 1), d, dtype=dt, device=device)
        self.sum_v = torch.zeros(bh, max(cap_chunks, 1), d, dtype=dt, device=device)
        self.c = EvaCache()
        self.c.cfg = cfg
        self.c.pos = 0
        self.c.cap_chunks = cap_chunks
        self.c.ring_k, self.c.ring_v = self.ring_k.data_ptr(), self.ring_v.data_ptr()
        self.c.sum_k, self.c.sum_v = self.sum_k.data_ptr(), self.sum_v.data_ptr()
        self.device = torch.device(device)
        self._ws = None

    @property
    def pos(self) -> int:
        return int(self.c.pos)

    @property
    def cfg(self) -> EvaConfig:
        return self.c.cfg

    def workspace_bytes(self) -> int:
        return int(lib.eva_decode_workspace_bytes(ctypes.byref(self.c)))

    def eva_cache_append(self, K_new: torch.Tensor, V_new: torch.Tensor,
                         eps: Optional[torch.Tensor] = None) -> None:
        """Append n_new tokens per unit: K_new, V_new [bh, n_new, d]."""
        cfg = self.c.cfg
        dt, bh, d = _tdtype(cfg), cfg.bh_count, cfg.d_head
        if K_new.dim() == 2:
            K_new, V_new = K_new.unsqueeze(1), V_new.unsqueeze(1)
        n_new = K_new.shape[1]
        _need(K_new, "K_new", (bh, n_new, d), dt)
        _need(V_new, "V_new", (bh, n_new, d), dt)
        if eps is not None:
            _need(eps, "eps", (bh, self.c.cap_chunks, d), torch.float32)
        check(lib.eva_cache_append(ctypes.byref(self.c), _ptr(K_new), _ptr(V_new), n_new, _ptr(eps),
                                   _stream(self.device)))

    append = eva_cache_append

    def eva_cache_load(self, K: torch.Tensor, V: torch.Tensor, Ksum: Optional[torch.Tensor] = None,
                       Vsum: Optional[torch.Tensor] = None) -> None:
        """Prefill hand-off into an empty cache with already-computed summaries."""
        cfg = self.c.cfg
        dt, bh, d = _tdtype(cfg), cfg.bh_count, cfg.d_head
        n = K.shape[1]
        nC = n // cfg.chunk
        _need(K, "K", (bh, n, d), dt)
        _need(V, "V", (bh, n, d), dt)
        if nC:
            _need(Ksum, "Ksum", (bh, nC, d), dt)
            _need(Vsum, "Vsum", (bh, nC, d), dt)
        check(lib.eva_cache_load(ctypes.byref(self.c), _ptr(K), _ptr(V), _ptr(Ksum if nC else None),
                                 _ptr(Vsum if nC else None), n, _stream(self.device)))

    load = eva_cache_load

    def eva_attn_decode(self, q: torch.Tensor, O: Optional[torch.Tensor] = None,
                        lse: Optional[torch.Tensor] = None, want_lse: bool = True):
        """One query per unit at position pos-1: q [bh, d] -> (o [bh, d], lse [bh])."""
        cfg = self.c.cfg
        dt, bh, d = _tdtype(cfg), cfg.bh_count, cfg.d_head
        _need(q, "q", (bh, d), dt)
        O = torch.empty_like(q) if O is None else O
        if want_lse and lse is None:
            lse = torch.empty(bh, dtype=torch.float32, device=q.device)
        nbytes = self.workspace_bytes()
        if nbytes and (self._ws is None or self._ws.numel() * 4 < nbytes):
            self._ws = torch.zeros((nbytes + 3) // 4 * 2, dtype=torch.float32, device=q.device)
        ws = self._ws if nbytes else None
        check(lib.eva_attn_decode(ctypes.byref(self.c), _ptr(q), _ptr(O),
                                  _ptr(lse if want_lse else None), _ptr(ws),
                                  0 if ws is None else ws.numel() * 4, _stream(q.device)))
        return O, (lse if want_lse else None)

    decode = eva_attn_decode

    def eva_decode_step(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                        eps: Optional[torch.Tensor] = None, O: Optional[torch.Tensor] = None,
                        lse: Optional[torch.Tensor] = None, want_lse: bool = True):
        """Append (k, v) and attend q at that position in one launch: q, k, v [bh, d]."""
        cfg = self.c.cfg
        dt, bh, d = _tdtype(cfg), cfg.bh_count, cfg.d_head
        for t, nm in ((q, "q"), (k, "k"), (v, "v")):
            _need(t, nm, (bh, d), dt)
        if eps is not None:
            _need(eps, "eps", (bh, self.c.cap_chunks, d), torch.float32)
        O = torch.empty_like(q) if O is None else O
        if want_lse and lse is None:
            lse = torch.empty(bh, dtype=torch.float32, device=q.device)
        self.c.pos += 1
        nbytes = self.workspace_bytes()
        self.c.pos -= 1
        if nbytes and (self._ws is None or self._ws.numel() * 4 < nbytes):
            self._ws = torch.zeros((nbytes + 3) // 4 * 2, dtype=torch.float32, device=q.device)
        ws = self._ws if nbytes else None
        check(lib.eva_decode_step(ctypes.byref(self.c), _ptr(q), _ptr(k), _ptr(v), _ptr(eps), _ptr(O),
                                  _ptr(lse if want_lse else None), _ptr(ws),
                                  0 if ws is None else ws.numel() * 4, _stream(q.device)))
        return O, (lse if want_lse else None)

    step = eva_decode_step

    def eva_decode_step_ragged(self, pos: torch.Tensor, q: torch.Tensor, k: torch.Tensor,
                               v: torch.Tensor, eps: Optional[torch.Tensor] = None,
                               O: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None,
                               want_lse: bool = True, rope: Optional[dict] = None):
        """Per-unit positions: pos int64 CUDA [bh] (advanced in place); append (k, v) at pos[u]
        and attend q at that position, q, k, v [bh, d].  self.pos is not used.  rope: None, or
        dict(rope_base=..., rotary_dim=..., style=...) -- q and k are un-rotated and the kernel
        applies RoPE at pos[u] in the same launch (eva_decode_step_ragged_rope)."""
        cfg = self.c.cfg
        dt, bh, d = _tdtype(cfg), cfg.bh_count, cfg.d_head
        _need(pos, "pos", (bh,), torch.int64)
        for t, nm in ((q, "q"), (k, "k"), (v, "v")):
            _need(t, nm, (bh, d), dt)
        if eps is not None:
            _need(eps, "eps", (bh, self.c.cap_chunks, d), torch.float32)
        O = torch.empty_like(q) if O is None else O
        if want_lse and lse is None:
            lse = torch.empty(bh, dtype=torch.float32, device=q.device)
        nbytes = int(lib.eva_decode_ragged_workspace_bytes(ctypes.byref(self.c)))
        # its own zero-filled scratch: the split count (and so the merge-counter offset) differs
        # from the uniform decode's
        if nbytes and (getattr(self, "_ws_ragged", None) is None or self._ws_ragged.numel() * 4 < nbytes):
            self._ws_ragged = torch.zeros((nbytes + 3) // 4, dtype=torch.float32, device=q.device)
        ws = self._ws_ragged if nbytes else None
        if rope is not None:
            rp = _rope_params(rope.get("rope_base", 10000.0), rope.get("rotary_dim"),
                              rope.get("style", "interleaved"))
            check(lib.eva_decode_step_ragged_rope(ctypes.byref(self.c), _ptr(pos), ctypes.byref(rp), _ptr(q), _ptr(k),
                                                  _ptr(v), _ptr(eps), _ptr(O), _ptr(lse if want_lse else None),
                                                  _ptr(ws), 0 if ws is None else ws.numel() * 4, _stream(q.device)))
            return O, (lse if want_lse else None)
        check(lib.eva_decode_step_ragged(ctypes.byref(self.c), _ptr(pos), _ptr(q), _ptr(k), _ptr(v), _ptr(eps),
                                         _ptr(O), _ptr(lse if want_lse else None), _ptr(ws),
                                         0 if ws is None else ws.numel() * 4, _stream(q.device)))
        return O, (lse if want_lse else None)


def eva_mask_ranges(cfg: EvaConfig, n_begin: int, count: int, device="cuda"):
    lo = torch.empty(count, dtype=torch.int64, device=device)
    ns = torch.empty(count, dtype=torch.int64, device=device)
    check(lib.eva_mask_ranges(ctypes.byref(cfg), n_begin, count, _ptr(lo), _ptr(ns),
                              _stream(torch.device(device))))
    return lo, ns


def eva_philox(blocks: torch.Tensor) -> torch.Tensor:
    """blocks: integer [n, 6] (ctr0..3, key0, key1) -> Philox4x32-10 words as int64 [n, 4]."""
    x = blocks.to(torch.int64) & 0xFFFFFFFF
    x = torch.where(x >= 2 ** 31, x - 2 ** 32, x).to(torch.int32).contiguous().cuda()
    out = torch.empty(x.shape[0], 4, dtype=torch.int32, device=x.device)
    check(lib.eva_philox(_ptr(x), _ptr(out), x.shape[0], _stream(x.device)))
    return out.to(torch.int64) & 0xFFFFFFFF


def eva_cache_append(cache: "DecodeCache", K_new: torch.Tensor, V_new: torch.Tensor,
                     eps: Optional[torch.Tensor] = None) -> None:
    """C-ABI-named alias of DecodeCache.eva_cache_append."""
    cache.eva_cache_append(K_new, V_new, eps)


def eva_cache_load(cache: "DecodeCache", K, V, Ksum=None, Vsum=None) -> None:
    """C-ABI-named alias of DecodeCache.eva_cache_load."""
    cache.eva_cache_load(K, V, Ksum, Vsum)


def eva_attn_decode(cache: "DecodeCache", q: torch.Tensor, **kw):
    """C-ABI-named alias of DecodeCache.eva_attn_decode."""
    return cache.eva_attn_decode(q, **kw)


def eva_draw_eps(cfg: EvaConfig, device="cuda") -> torch.Tensor:
    nC = cfg.T // cfg.chunk
    eps = torch.empty(cfg.bh_count, max(nC, 1), cfg.d_head, dtype=torch.float32, device=device)
    check(lib.eva_draw_eps(ctypes.byref(cfg), _ptr(eps), _stream(torch.device(device))))
    return eps[:, :nC]
