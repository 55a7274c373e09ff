"""Multi-process (gloo, world_size 2, CPU) tests of the (b,h)-sharding bookkeeping that
bench.py and the multi-GPU driver use.  No kernel runs here; the GPU side of the N>1
path is the same per-rank C-ABI call on a contiguous unit shard."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _load_parallel():
    # import the pure-Python module without loading libeva.so (no GPU on the build host)
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location(
        "eva_parallel", os.path.join(root, "paper_2511_00576_b200", "parallel.py"))
    mod = importlib.util.module_from_spec(spec)
    import sys
    sys.modules["eva_parallel"] = mod
    spec.loader.exec_module(mod)
    return mod


def test_shard_units_cover_exactly():
    P = _load_parallel()
    for total in (0, 1, 7, 16, 256, 8192):
        for world in (1, 2, 3, 4, 8):
            sh = P.shard_units(total, world)
            assert [s.rank for s in sh] == list(range(world))
            covered = [u for s in sh for u in range(s.bh_begin, s.bh_begin + s.bh_count)]
            assert covered == list(range(total))
            assert max(s.bh_count for s in sh) - min(s.bh_count for s in sh) <= 1


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = _load_parallel()
        import eva_inputs
        B, H, T, d = 3, 3, 40, 8           # 9 units over 2 ranks: shards of 5 and 4
        sh = P.shard_units(B * H, world)
        me = sh[rank]
        # rank-local generation keyed by global unit == slice of the global input
        q_loc, _, _ = eva_inputs.qkv(me.bh_begin, me.bh_count, T, d, torch.float32, seed=5)
        q_all, _, _ = eva_inputs.qkv(0, B * H, T, d, torch.float32, seed=5)
        assert torch.equal(q_loc, q_all[me.bh_begin:me.bh_begin + me.bh_count])
        # gather of per-rank slabs rebuilds the global tensor in unit order
        g = P.gather_units(q_loc * 2, sh)
        # scatter from rank 0 hands every rank its slab
        s = P.scatter_units(q_all if rank == 0 else None, sh, (T, d), torch.float32, "cpu")
        ok_scatter = torch.equal(s, q_loc)
        # device-time reduction is a max over ranks
        t = P.max_over_ranks(1.0 + rank)
        if rank == 0:
            q.put(("gather", bool(torch.equal(g, q_all * 2))))
        q.put(("scatter%d" % rank, ok_scatter))
        q.put(("max%d" % rank, t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_gather_scatter_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = {}
    while not q.empty():
        k, v = q.get()
        res[k] = v
    assert res["gather"] is True
    assert res["scatter0"] is True and res["scatter1"] is True
    assert res["max0"] == 2.0 and res["max1"] == 2.0
