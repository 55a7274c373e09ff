"""Context-parallel prefill (paper_2511_00576_b200/context_parallel.py).

CPU: the shard/halo bookkeeping against the oracle's mask, and the one exchange step
(summary all-gather + halo send/recv) in real gloo process groups of 2 and 3 ranks.
GPU: every rank's eva_summarize_range + eva_attn_prefill_range, run one after another on one
device with the exchange done by slicing, must reproduce the single-call prefill -- bitwise
when the shard bounds are multiples of 128 (same tiles), within the tolerance otherwise --
and the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import eva_inputs
import oracle


def _cp():
    from paper_2511_00576_b200 import context_parallel
    return context_parallel


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("T,world,C,W", [(8192, 4, 64, 256), (1000, 3, 16, 64), (4096, 8, 32, 128),
                                         (640, 2, 128, 128), (2048, 2, 64, 512)])
def test_seq_shards_cover_align_and_halo(T, world, C, W, mode):
    cp = _cp()
    sh = cp.seq_shards(T, world, C, W, mode)
    assert sh[0].q0 == 0 and sh[-1].q1 == T
    for a, b in zip(sh, sh[1:]):
        assert a.q1 == b.q0
    for s in sh:
        assert s.q0 % 128 == 0 and s.q0 % C == 0
        lo, nsum = oracle.mask(s.q0, C, W, mode)       # independent mask implementation
        assert s.k0 == lo and s.q0 - s.k0 < W
        # every query of the shard sees keys only from [k0, its own position]
        for n in (s.q0, (s.q0 + s.q1) // 2, s.q1 - 1):
            assert oracle.mask(n, C, W, mode)[0] >= s.k0
        if s.rank:
            assert s.k0 >= sh[s.rank - 1].q0          # halo comes from the previous rank only


def test_seq_shards_rejects_short_shards():
    cp = _cp()
    with pytest.raises(ValueError):
        cp.seq_shards(256, 4, 64, 256)      # 2 blocks of 128 for 4 ranks
    with pytest.raises(ValueError):
        cp.seq_shards(512, 4, 64, 512)      # 128-position shards, 448-position halo


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, T, C, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cp = _cp()
        bh, d = 3, 8
        sh = cp.seq_shards(T, world, C, W)
        me = sh[rank]
        g = torch.Generator().manual_seed(11)
        K = torch.randn(bh, T, d, generator=g)
        V = torch.randn(bh, T, d, generator=g)
        S = torch.randn(2, bh, T // C, d, generator=g)       # stand-in summaries, chunk order
        c0, c1 = me.q0 // C, me.q1 // C
        Ks_all, Vs_all, Kh, Vh = cp.exchange(S[0, :, c0:c1].contiguous(), S[1, :, c0:c1].contiguous(),
                                             K[:, me.q0:me.q1].contiguous(), V[:, me.q0:me.q1].contiguous(),
                                             sh, rank, C)
        ok = (torch.equal(Ks_all, S[0]) and torch.equal(Vs_all, S[1])
              and torch.equal(Kh, K[:, me.k0:me.q0]) and torch.equal(Vh, V[:, me.k0:me.q0]))
        q.put((rank, bool(ok), Kh.shape[1]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T,C,W", [(2, 1000, 16, 64), (3, 1536, 64, 256)])
def test_gloo_exchange_gathers_summaries_and_halo(world, T, C, W):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, T, C, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    res = {}
    while not q.empty():
        r, ok, hl = q.get()
        res[r] = (ok, hl)
    assert sorted(res) == list(range(world))
    assert all(ok for ok, _ in res.values())
    assert res[0][1] == 0 and all(res[r][1] > 0 for r in range(1, world))


# ----------------------------------------------------------------------------- GPU
def _emulated_cp(eva, cfg, Q, K, V, shards, simt):
    """Every rank's kernels on one device; the exchange is done by slicing (the gloo test
    covers the collective)."""
    C = cfg.chunk
    sums = []
    for s in shards:
        sub = eva.make_config(cfg.B, cfg.H, s.q1 - s.q0, cfg.d_head, C, cfg.window, mode=cfg.mode,
                              dtype=Q.dtype)
        sums.append(eva.eva_summarize_range(sub, s.q0 // C, K[:, s.q0:s.q1].contiguous(),
                                            V[:, s.q0:s.q1].contiguous()))
    Ks = torch.cat([a for a, _ in sums], dim=1).contiguous()
    Vs = torch.cat([b for _, b in sums], dim=1).contiguous()
    outs = []
    for s in shards:
        O, lse = eva.eva_attn_prefill_range(cfg, s.q0, s.k0, Q[:, s.q0:s.q1].contiguous(),
                                            K[:, s.k0:s.q1].contiguous(), V[:, s.k0:s.q1].contiguous(),
                                            Ks, Vs, simt=simt)
        outs.append((O, lse))
    return Ks, Vs, torch.cat([o for o, _ in outs], dim=1), torch.cat([l for _, l in outs], dim=1)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["sliding", "block"])
@pytest.mark.parametrize("dtype,d,simt", [(torch.bfloat16, 128, False), (torch.bfloat16, 64, False),
                                          (torch.float32, 64, True), (torch.bfloat16, 64, True)])
@pytest.mark.parametrize("T,world,C,W", [(2048, 4, 64, 256), (1000, 3, 16, 64)])
def test_cp_equals_single_call_bitwise(cuda_device, mode, dtype, d, simt, T, world, C, W):
    import paper_2511_00576_b200 as eva
    cp = _cp()
    mode_i = 0 if mode == "sliding" else 1
    B, H = 1, 3
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode, dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=21, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, simt=simt)
    Ks, Vs, O2, lse2 = _emulated_cp(eva, cfg, Q, K, V, cp.seq_shards(T, world, C, W, mode_i), simt)
    torch.cuda.synchronize()
    assert torch.equal(Ks, ks) and torch.equal(Vs, vs)
    assert torch.equal(O2, O) and torch.equal(lse2, lse)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,simt,tol", [(torch.bfloat16, False, 2e-2), (torch.float32, True, 1e-4)])
def test_cp_unaligned_shards_match_oracle(cuda_device, dtype, simt, tol):
    """Shard bounds on chunk multiples that are not multiples of 128: different tiles,
    so compared with the oracle within the north_star tolerance."""
    import paper_2511_00576_b200 as eva
    from paper_2511_00576_b200.context_parallel import SeqShard
    B, H, T, d, C, W = 1, 2, 700, 64, 32, 96
    cfg = eva.make_config(B, H, T, d, C, W, dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=22, device="cuda")
    bounds = [0, 224, 480, 700]
    lo = [oracle.mask(q0, C, W, 0)[0] for q0 in bounds[:-1]]
    shards = [SeqShard(r, bounds[r], bounds[r + 1], lo[r]) for r in range(3)]
    Ks, Vs, O2, lse2 = _emulated_cp(eva, cfg, Q, K, V, shards, simt)
    torch.cuda.synchronize()
    f64 = lambda t: t.float().cpu().double().numpy()
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, T // C, d)
    rk, rv = oracle.summarize_batch(f64(K), f64(V), E, C)
    rO, rl = oracle.prefill_batch(f64(Q), f64(K), f64(V), rk, rv, C, W, 0, cfg.scale)
    assert np.abs(f64(Ks) - rk).max() <= tol and np.abs(f64(Vs) - rv).max() <= tol
    assert np.abs(f64(O2) - rO).max() <= tol and np.abs(f64(lse2) - rl).max() <= tol


@pytest.mark.gpu
def test_prefill_range_validation(cuda_device):
    import paper_2511_00576_b200 as eva
    cfg = eva.make_config(1, 1, 1024, 64, 64, 256)
    Q = torch.zeros(1, 128, 64, dtype=torch.bfloat16, device="cuda")
    K = torch.zeros(1, 320, 64, dtype=torch.bfloat16, device="cuda")
    S = torch.zeros(1, 16, 64, dtype=torch.bfloat16, device="cuda")
    # q0 = 512: lo(512) = 320 -> k0 must be <= 320; keys must reach 639
    eva.eva_attn_prefill_range(cfg, 512, 320, Q, K, K, S, S)
    with pytest.raises(eva.EvaError, match="halo"):
        eva.eva_attn_prefill_range(cfg, 512, 384, Q, K[:, :256].contiguous(), K[:, :256].contiguous(), S, S)
    with pytest.raises(eva.EvaError, match="keys end"):
        eva.eva_attn_prefill_range(cfg, 512, 320, Q, K[:, :300].contiguous(), K[:, :300].contiguous(), S, S)
    with pytest.raises(eva.EvaError, match="n_sum"):
        eva.eva_attn_prefill_range(cfg, 512, 320, Q, K, K, S[:, :2].contiguous(), S[:, :2].contiguous())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,d", [(torch.bfloat16, 128), (torch.float32, 64)])
def test_summarize_bcast_writes_every_destination(cuda_device, dtype, d):
    """The fused summarise + all-gather kernel: three emulated ranks each summarise their shard
    and store it into all three destination buffers (stand-ins for NVLink peer buffers);
    every buffer ends up bitwise equal to the single-call summaries."""
    import paper_2511_00576_b200 as eva
    cp = _cp()
    B, H, T, C, W = 1, 3, 1536, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W, dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=41, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    nC = T // C
    bufs = [torch.full((2, B * H, nC, d), float("nan"), dtype=dtype, device="cuda") for _ in range(3)]
    pk = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    pv = torch.tensor([b[1].data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    for s in cp.seq_shards(T, 3, C, W):
        sub = eva.make_config(B, H, s.q1 - s.q0, d, C, W, dtype=dtype)
        eva.eva_summarize_range_bcast(sub, s.q0 // C, K[:, s.q0:s.q1].contiguous(), V[:, s.q0:s.q1].contiguous(),
                                      pk, pv, nC)
    torch.cuda.synchronize()
    for b in bufs:
        assert torch.equal(b[0], ks) and torch.equal(b[1], vs)
    with pytest.raises(eva.EvaError, match="INVALID_ARG"):   # destination rows too few
        eva.eva_summarize_range_bcast(cfg, 0, K, V, pk, pv, nC - 1)


def _symm_cp_worker(q):
    """One process, world size 1, NCCL + symmetric memory: the P2P exchange path end to end."""
    import paper_2511_00576_b200 as eva
    cp = _cp()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        B, H, T, d, C, W = 1, 2, 1024, 128, 64, 256
        cfg = eva.make_config(B, H, T, d, C, W)
        Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=42, device="cuda")
        O, lse, _, _ = eva.eva_attn_prefill(cfg, Q, K, V)
        try:
            peers = cp.PeerSummaries(B * H, T // C, d, torch.bfloat16, "cuda")
        except Exception as e:  # symmetric memory unavailable on this box
            q.put(("skip", repr(e)[:200]))
            return
        sh = cp.seq_shards(T, 1, C, W)
        O2, lse2 = cp.cp_prefill(cfg, Q, K, V, sh, 0, peers=peers)
        torch.cuda.synchronize()
        q.put(("ok", bool(torch.equal(O2, O) and torch.equal(lse2, lse))))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_cp_prefill_symmetric_memory_world1(cuda_device):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_symm_cp_worker, args=(q,))
    p.start()
    p.join(timeout=300)
    assert p.exitcode == 0
    kind, val = q.get(timeout=5)
    if kind == "skip":
        pytest.skip(f"symmetric memory unavailable: {val}")
    assert val is True
