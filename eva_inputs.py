"""Seeded synthetic inputs for the FlashEVA hot path (shared by tests, bench and smoke).

This module holds NO arithmetic of the method: it only draws i.i.d. normal
tensors with torch generators keyed by (seed, global unit index), so that a
(batch, head) shard generated on any rank equals the same slice of the
single-GPU input.  Both the CUDA path and the oracle consume what it returns.

Input recipe: Q, K, V ~ N(0, 1) i.i.d. per element, layout
[BH, T, d] contiguous, rounded to the path's dtype (bf16 or fp32); optional
caller-supplied eps ~ N(0, 1) of shape [BH, nC, d] in fp32.
"""
from __future__ import annotations

import torch

_UNIT_STRIDE = 1_000_003


def _gen(seed: int, unit: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * _UNIT_STRIDE + unit) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def normal_units(n_tensors: int, bh_begin: int, bh_count: int, rows: int, d: int,
                 dtype=torch.float32, seed: int = 0, device="cpu", std: float = 1.0):
    """n_tensors tensors of shape [bh_count, rows, d], unit u drawn from its own stream."""
    outs = [torch.empty(bh_count, rows, d, dtype=dtype, device=device) for _ in range(n_tensors)]
    for i in range(bh_count):
        g = _gen(seed, bh_begin + i, device)
        x = torch.randn(n_tensors, rows, d, generator=g, device=device, dtype=torch.float32)
        if std != 1.0:
            x.mul_(std)
        for t in range(n_tensors):
            outs[t][i].copy_(x[t])
    return outs


def qkv(bh_begin: int, bh_count: int, T: int, d: int, dtype=torch.bfloat16, seed: int = 0,
        device="cpu", std: float = 1.0):
    """Q, K, V of shape [bh_count, T, d] for global units [bh_begin, bh_begin + bh_count)."""
    return tuple(normal_units(3, bh_begin, bh_count, T, d, dtype, seed, device, std))


def eps(bh_begin: int, bh_count: int, nC: int, d: int, seed: int = 7, device="cpu"):
    """Caller-supplied eps ~ N(0, I) [bh_count, nC, d] fp32 (alternative to in-kernel Philox)."""
    return normal_units(1, bh_begin, bh_count, max(nC, 0), d, torch.float32, seed + 99991,
                        device)[0]


def decode_tokens(bh_begin: int, bh_count: int, steps: int, d: int, dtype=torch.bfloat16,
                  seed: int = 3, device="cpu"):
    """q, k, v for `steps` generated tokens: [steps, bh_count, d] each."""
    q, k, v = normal_units(3, bh_begin, bh_count, steps, d, dtype, seed, device)
    return q.transpose(0, 1).contiguous(), k.transpose(0, 1).contiguous(), \
        v.transpose(0, 1).contiguous()
