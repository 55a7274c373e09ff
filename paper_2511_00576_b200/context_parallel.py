"""Context-parallel (sequence-sharded) FlashEVA prefill.

The paper positions EVA against ring attention for long contexts; FlashEVA makes a
sequence split cheap because each query sees only (a) its exact local window (a
halo of < W positions before a shard) and (b) one summary per earlier chunk, and the
summaries are query-independent (S = 1) and tiny (one key/value row per C tokens).
So a rank that owns positions [q0, q1) of every unit needs exactly ONE exchange step:

  1. summaries of its own complete chunks          eva_summarize_range    (kernel)
  2. all-gather of the summaries of every rank      NCCL all_gather        (collective)
     + the halo [lo(q0), q0) of K and V from the previous rank   NCCL send/recv
  3. attention of its queries                       eva_attn_prefill_range (kernel)

Compare ring attention, which circulates every rank's full K/V (world - 1 steps).  Per
unit the exchange moves n_chunks*d*2 summary elements (all-gather) and <= 2*(W - 1)*d halo
elements; the attention itself is unchanged (same kernels, same tiles: with shard bounds on
multiples of 128 the result is bitwise equal to the single-GPU prefill).

Host-side integer bookkeeping only; every arithmetic step runs in libeva's kernels.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

import torch

from . import api
from ._native import EVA_WINDOW_SLIDING


@dataclass(frozen=True)
class SeqShard:
    rank: int
    q0: int    # first owned position
    q1: int    # one past the last owned position
    k0: int    # first key/value position the shard's queries see (halo start, lo(q0))


def window_start(n: int, C: int, W: int, mode: int) -> int:
    """lo(n) of the chunk-causal mask (include/eva.h, reading R7)."""
    if mode == EVA_WINDOW_SLIDING:
        return max(0, n // C - W // C + 1) * C
    return (n // W) * W


def block_cost(b0: int, b1: int, C: int, W: int, mode: int) -> int:
    """Key tiles the prefill kernel walks for the 128-query tiles in [b0, b1) (summary prefix
    tiles + local span tiles of 64 keys, plus ~2 tiles of fixed cost per query tile)."""
    cost = 0
    for n0 in range(b0, b1, 128):
        nl = min(n0 + 127, b1 - 1)
        lo = window_start(n0, C, W, mode)
        ns_last = (nl // C - W // C + 1) if mode == EVA_WINDOW_SLIDING else (nl // W) * W // C
        cost += -(-max(0, ns_last) // 64) + -(-(nl - lo + 1) // 64) + 2
    return cost


def seq_shards(T: int, world: int, C: int, W: int, mode: int = EVA_WINDOW_SLIDING,
               align: int = 128, balance: bool = True) -> List[SeqShard]:
    """Split positions [0, T) into `world` contiguous shards whose bounds are multiples of
    lcm(align, C) (so every interior chunk has one owner and the tensor-core tiles line up
    with the unsharded run).  balance=False gives equal lengths; balance=True equalises the
    kernel's work instead (a query at position n reads ~n/C summaries, so later shards are
    shorter).  Every shard but the first must reach back over the next shard's halo so
    that the halo comes from the previous rank alone."""
    if world < 1 or T < 1:
        raise ValueError("world >= 1 and T >= 1 required")
    g = align * C // math.gcd(align, C)
    units = -(-T // g)
    if units < world:
        raise ValueError(f"T={T} has only {units} blocks of {g} positions for {world} ranks")
    if balance:
        cost = [block_cost(i * g, min(T, (i + 1) * g), C, W, mode) for i in range(units)]
        pre = [0]
        for c in cost:
            pre.append(pre[-1] + c)
        cuts = [0]
        for r in range(1, world):
            target = pre[-1] * r / world
            i = min(range(cuts[-1] + 1, units - (world - r) + 1), key=lambda k: abs(pre[k] - target))
            cuts.append(i)
        cuts.append(units)
    else:
        base, extra = divmod(units, world)
        cuts = [0]
        for r in range(world):
            cuts.append(cuts[-1] + base + (1 if r < extra else 0))
    out = []
    for r in range(world):
        q0, q1 = cuts[r] * g, min(T, cuts[r + 1] * g)
        out.append(SeqShard(r, q0, q1, window_start(q0, C, W, mode)))
    for s in out[1:]:
        prev = out[s.rank - 1]
        if s.k0 < prev.q0:
            raise ValueError(f"shard {s.rank - 1} ({prev.q1 - prev.q0} positions) is shorter than the "
                             f"halo of shard {s.rank} ({s.q0 - s.k0}); use fewer ranks")
    return out


def exchange(Ksum: torch.Tensor, Vsum: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
             shards: List[SeqShard], rank: int, C: int, group=None,
             summaries: bool = True) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    """The one exchange step.  Ksum/Vsum [bh, c_r, d]: this rank's chunk summaries; K/V
    [bh, q1 - q0, d]: its keys/values.  Returns (Ksum_all, Vsum_all) [bh, sum c_r, d] (every
    rank's summaries in chunk order) and the halo (K_halo, V_halo) [bh, q0 - k0, d] received
    from rank - 1 (rank r sends rows [k0_{r+1} - q0_r, ...) of its K/V to rank r + 1)."""
    import torch.distributed as dist
    world = len(shards)
    me = shards[rank]
    bh, d = K.shape[0], K.shape[2]
    counts = [(s.q1 - s.q0) // C for s in shards]  # complete chunks owned by each rank
    if Ksum.shape[1] != counts[rank]:
        raise ValueError(f"rank {rank} has {Ksum.shape[1]} summaries, expected {counts[rank]}")
    mx = max(max(counts), 1)
    Ksum_all = Vsum_all = None
    if summaries:
        # (2a) all-gather of the summaries (padded to the largest count)
        send = torch.zeros(2, bh, mx, d, dtype=Ksum.dtype, device=Ksum.device)
        send[0, :, :counts[rank]] = Ksum
        send[1, :, :counts[rank]] = Vsum
        recv = torch.empty((world * 2,) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        dist.all_gather_into_tensor(recv, send, group=group)
        recv = recv.view((world,) + tuple(send.shape))
        Ksum_all = torch.cat([recv[r, 0, :, :counts[r]] for r in range(world)], dim=1).contiguous()
        Vsum_all = torch.cat([recv[r, 1, :, :counts[r]] for r in range(world)], dim=1).contiguous()
    # (2b) halo from the previous rank, to the next rank
    ops = []
    nxt = shards[rank + 1] if rank + 1 < world else None
    if nxt is not None and nxt.q0 > nxt.k0:
        lo = nxt.k0 - me.q0
        halo_out = torch.cat([K[:, lo:], V[:, lo:]], dim=1).contiguous()
        ops.append(dist.P2POp(dist.isend, halo_out, _peer(rank + 1, group), group))
    hl = me.q0 - me.k0
    halo_in = torch.empty(bh, 2 * hl, d, dtype=K.dtype, device=K.device)
    if rank > 0 and hl > 0:
        ops.append(dist.P2POp(dist.irecv, halo_in, _peer(rank - 1, group), group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return Ksum_all, Vsum_all, halo_in[:, :hl], halo_in[:, hl:]


class PeerSummaries:
    """The global summary list as symmetric memory: every rank holds [2, bh, n_chunks, d]
    (K~ and beta^) and knows every peer's address, so eva_summarize_range_bcast stores each
    rank's summaries straight into all ranks' copies over NVLink (the summarise and the
    all-gather are one kernel); a device-side barrier then orders the readers."""

    def __init__(self, bh: int, n_chunks: int, d: int, dtype, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.buf = symm.empty((2, bh, max(n_chunks, 1), d), dtype=dtype, device=device)
        gname = (group or dist.group.WORLD).group_name
        self.handle = symm.rendezvous(self.buf, gname)
        half = bh * max(n_chunks, 1) * d * self.buf.element_size()
        ptrs = [int(p) for p in self.handle.buffer_ptrs]
        self.ptr_k = torch.tensor(ptrs, dtype=torch.int64, device=device)
        self.ptr_v = torch.tensor([p + half for p in ptrs], dtype=torch.int64, device=device)
        self.n_chunks = n_chunks

    def barrier(self):
        self.handle.barrier(channel=0)


def exchange_p2p(cfg, K: torch.Tensor, V: torch.Tensor, shards: List[SeqShard], rank: int,
                 peers: PeerSummaries, group=None):
    """The exchange with the summary all-gather fused into the summarising kernel (NVLink
    stores into every rank's symmetric buffer); the halo still moves by NCCL send/recv."""
    me = shards[rank]
    sub = api.make_config(cfg.B, cfg.H, me.q1 - me.q0, cfg.d_head, cfg.chunk, cfg.window,
                          bh_begin=cfg.bh_begin, bh_count=cfg.bh_count, mode=cfg.mode,
                          dtype=api._tdtype(cfg), scale=cfg.scale, lam=cfg.lambda_, clip=cfg.clip,
                          seed=cfg.seed, layer=cfg.layer, omega_mode=cfg.omega_mode,
                          summary_bias=cfg.summary_bias)
    # Write-after-read guard: the previous cp_prefill on these PeerSummaries (last layer or
    # iteration) reads every copy in place, and a faster rank's stores below would land in a
    # slower rank's copy while its prefill still reads it.  The device-side barrier is stream
    # ordered, so every rank's earlier prefill has completed once all ranks pass it.
    peers.barrier()
    api.eva_summarize_range_bcast(sub, me.q0 // cfg.chunk, K, V, peers.ptr_k, peers.ptr_v,
                                  peers.n_chunks)
    peers.barrier()  # every rank's summaries have landed in every copy
    _, _, Kh, Vh = exchange(K.new_zeros(K.shape[0], (me.q1 - me.q0) // cfg.chunk, K.shape[2]),
                            V.new_zeros(V.shape[0], (me.q1 - me.q0) // cfg.chunk, V.shape[2]),
                            K, V, shards, rank, cfg.chunk, group, summaries=False)
    return peers.buf[0, :, :peers.n_chunks], peers.buf[1, :, :peers.n_chunks], Kh, Vh


def _peer(r: int, group) -> int:
    import torch.distributed as dist
    return r if group is None else dist.get_global_rank(group, r)


def cp_prefill(cfg, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, shards: List[SeqShard],
               rank: int, group=None, simt: bool = False, want_lse: bool = True,
               peers: Optional[PeerSummaries] = None):
    """Context-parallel prefill on this rank: Q/K/V [bh, q1 - q0, d] of this rank's shard of
    a sequence of cfg.T positions.  Returns (O, lse) for the shard.  With `peers` (symmetric
    memory for T // C summaries) the summary all-gather is fused into the summarising kernel."""
    me = shards[rank]
    if peers is not None:
        Ks_all, Vs_all, Kh, Vh = exchange_p2p(cfg, K, V, shards, rank, peers, group)
        Kc = torch.cat([Kh, K], dim=1) if Kh.shape[1] else K
        Vc = torch.cat([Vh, V], dim=1) if Vh.shape[1] else V
        return api.eva_attn_prefill_range(cfg, me.q0, me.k0, Q, Kc, Vc, Ks_all.contiguous(),
                                          Vs_all.contiguous(), want_lse=want_lse, simt=simt)
    n = me.q1 - me.q0
    sub = api.make_config(cfg.B, cfg.H, n, cfg.d_head, cfg.chunk, cfg.window, bh_begin=cfg.bh_begin,
                          bh_count=cfg.bh_count, mode=cfg.mode, dtype=api._tdtype(cfg), scale=cfg.scale,
                          lam=cfg.lambda_, clip=cfg.clip, seed=cfg.seed, layer=cfg.layer,
                          omega_mode=cfg.omega_mode, summary_bias=cfg.summary_bias)
    Ks, Vs = api.eva_summarize_range(sub, me.q0 // cfg.chunk, K, V)                   # (1)
    Ks_all, Vs_all, Kh, Vh = exchange(Ks, Vs, K, V, shards, rank, cfg.chunk, group)             # (2)
    Kc = torch.cat([Kh, K], dim=1) if Kh.shape[1] else K
    Vc = torch.cat([Vh, V], dim=1) if Vh.shape[1] else V
    return api.eva_attn_prefill_range(cfg, me.q0, me.k0, Q, Kc, Vc, Ks_all, Vs_all,      # (3)
                                      want_lse=want_lse, simt=simt)
