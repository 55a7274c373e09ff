"""Ragged decode (per-unit positions) against the fp64 oracle's
streaming cache (oracle.Cache, pinned in test_oracle*.py): units hold prompts of different
lengths, then advance one token per call at their own positions."""
import ctypes

import numpy as np
import pytest
import torch

import eva_inputs
import oracle

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


@pytest.fixture(scope="module")
def eva(cuda_device):
    import paper_2511_00576_b200 as eva
    return eva


def f64(t):
    return t.detach().float().cpu().double().numpy()


def _unit_view(eva, cache, u):
    """A one-unit eva_cache aliasing unit u's slices of the cache buffers."""
    from paper_2511_00576_b200 import _native as N
    cfg = cache.c.cfg
    v = N.EvaCache()
    v.cfg = eva.make_config(cfg.B, cfg.H, 0, cfg.d_head, cfg.chunk, cfg.window, mode=cfg.mode,
                            dtype=torch.bfloat16 if cfg.dtype == N.EVA_BF16 else torch.float32,
                            seed=cfg.seed, bh_begin=cfg.bh_begin + u, bh_count=1, scale=cfg.scale)
    v.pos = 0
    v.cap_chunks = cache.c.cap_chunks
    v.ring_k, v.ring_v = cache.ring_k[u].data_ptr(), cache.ring_v[u].data_ptr()
    v.sum_k, v.sum_v = cache.sum_k[u].data_ptr(), cache.sum_v[u].data_ptr()
    return v


@pytest.mark.parametrize("mode", ["sliding", "block"])
@pytest.mark.parametrize("dtype,d,C,W", [(torch.float32, 32, 8, 24), (torch.bfloat16, 128, 16, 64),
                                         (torch.bfloat16, 64, 64, 128)])
def test_ragged_decode_parity(eva, mode, dtype, d, C, W):
    from paper_2511_00576_b200 import _native as N
    BH, steps = 4, 70
    prompt = [0, 5, C * 3 - 1, 2 * W + 7]        # empty, short, about to complete a chunk, long
    cap = (max(prompt) + steps) // C + 1
    cfg = eva.make_config(1, BH, 0, d, C, W, mode=mode, dtype=dtype, seed=21)
    cache = eva.DecodeCache(cfg, cap, device="cuda")
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    orc = [oracle.Cache(d, C, W, m, cap=cap, scale=cfg.scale) for _ in range(BH)]
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, BH, cap + 1, d)
    T_all = max(prompt) + steps
    q, k, v = eva_inputs.decode_tokens(0, BH, T_all, d, dtype, seed=22, device="cuda")
    # ragged prompts through one-unit views of the cache
    for u, n in enumerate(prompt):
        if n == 0:
            continue
        view = _unit_view(eva, cache, u)
        kk = k[:n, u].unsqueeze(0).contiguous()
        vv = v[:n, u].unsqueeze(0).contiguous()
        N.check(N.lib.eva_cache_append(ctypes.byref(view), kk.data_ptr(), vv.data_ptr(), n, None, None))
        for t in range(n):
            assert orc[u].append(f64(k[t, u]), f64(v[t, u]), E[u, t // C]) == 0
    pos = torch.tensor(prompt, dtype=torch.int64, device="cuda")
    worst = 0.0
    for s in range(steps):
        idx = [prompt[u] + s for u in range(BH)]
        qs = torch.stack([q[idx[u], u] for u in range(BH)]).contiguous()
        ks = torch.stack([k[idx[u], u] for u in range(BH)]).contiguous()
        vs = torch.stack([v[idx[u], u] for u in range(BH)]).contiguous()
        o, lse = cache.eva_decode_step_ragged(pos, qs, ks, vs)
        of, lf = f64(o), f64(lse)
        for u in range(BH):
            assert orc[u].append(f64(ks[u]), f64(vs[u]), E[u, idx[u] // C]) == 0
            ro, rl = orc[u].decode(f64(qs[u]))
            worst = max(worst, np.max(np.abs(of[u] - ro)), abs(lf[u] - rl))
    assert worst <= TOL[dtype], worst
    assert pos.tolist() == [p + steps for p in prompt]
    for u in range(BH):   # every unit's summaries equal the oracle's
        rks, rvs = orc[u].summaries()
        n = rks.shape[0]
        assert np.max(np.abs(f64(cache.sum_k[u, :n]) - rks), initial=0.0) <= TOL[dtype]
        assert np.max(np.abs(f64(cache.sum_v[u, :n]) - rvs), initial=0.0) <= TOL[dtype]


def test_ragged_uniform_equals_decode_step(eva):
    """With equal positions the ragged step gives the uniform step's outputs."""
    BH, d, C, W, T0 = 3, 64, 16, 32, 45
    cfg = eva.make_config(1, BH, 0, d, C, W, seed=3)
    a = eva.DecodeCache(cfg, 10, device="cuda")
    b = eva.DecodeCache(cfg, 10, device="cuda")
    q, k, v = eva_inputs.decode_tokens(0, BH, T0 + 20, d, torch.bfloat16, seed=4, device="cuda")
    a.eva_cache_append(k[:T0].transpose(0, 1).contiguous(), v[:T0].transpose(0, 1).contiguous())
    b.eva_cache_append(k[:T0].transpose(0, 1).contiguous(), v[:T0].transpose(0, 1).contiguous())
    pos = torch.full((BH,), T0, dtype=torch.int64, device="cuda")
    for t in range(T0, T0 + 20):
        oa, la = a.eva_decode_step(q[t], k[t], v[t])
        ob, lb = b.eva_decode_step_ragged(pos, q[t], k[t], v[t])
        torch.cuda.synchronize()
        assert torch.allclose(oa.float(), ob.float(), rtol=0, atol=2e-2)
        assert torch.allclose(la, lb, rtol=0, atol=1e-3)


def test_ragged_two_launch_form_parity():
    """The append-kernel + decode pair (EVA_RAGGED_TWO_LAUNCH, read once per process) runs the
    parity cases in a child pytest."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, EVA_RAGGED_TWO_LAUNCH="1")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-x", "-k",
                        "test_ragged_decode_parity or test_ragged_uniform", "-p", "no:cacheprovider"],
                       env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("style", ["interleaved", "neox"])
def test_ragged_decode_with_per_unit_rope(eva, style):
    """A ragged serving batch with RoPE (R18/R19): every step rotates the new q and k at each
    unit's own position with eva_rope(pos=the same device array the ragged step advances), then
    eva_decode_step_ragged; against the oracle cache fed the fp64-rotated (stored-precision) k, q."""
    dtype, d, C, W, rd = torch.bfloat16, 64, 16, 64, 32
    BH, steps = 4, 40
    prompt = [0, 9, C * 2 - 1, W + 3]
    cap = (max(prompt) + steps) // C + 1
    cfg = eva.make_config(1, BH, 0, d, C, W, dtype=dtype, seed=23)
    cache = eva.DecodeCache(cfg, cap, device="cuda")
    orc = [oracle.Cache(d, C, W, oracle.SLIDING, cap=cap, scale=cfg.scale) for _ in range(BH)]
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, BH, cap + 1, d)
    st = oracle.ROPE_NEOX if style == "neox" else oracle.ROPE_INTERLEAVED
    q, k, v = eva_inputs.decode_tokens(0, BH, max(prompt) + steps, d, dtype, seed=24, device="cuda")
    from paper_2511_00576_b200 import _native as N
    one = eva.make_config(1, BH, 1, d, C, W, dtype=dtype, seed=23)
    for u, n in enumerate(prompt):   # prompts: rotated keys at positions 0..n-1
        if n == 0:
            continue
        kr = torch.stack([eva.eva_rope(eva.make_config(1, 1, n, d, C, W, dtype=dtype),
                                       k[:n, u].unsqueeze(0).contiguous(), rotary_dim=rd, style=style)[0]])
        view = _unit_view(eva, cache, u)
        N.check(N.lib.eva_cache_append(ctypes.byref(view), kr.data_ptr(), v[:n, u].unsqueeze(0).contiguous().data_ptr(),
                                       n, None, None))
        for t in range(n):
            kt = oracle.rope_ex(f64(k[t, u])[None], [t], rotary_dim=rd, style=st)
            kt = torch.from_numpy(kt).to(dtype).double().numpy()[0]
            assert orc[u].append(kt, f64(v[t, u]), E[u, t // C]) == 0
    pos = torch.tensor(prompt, dtype=torch.int64, device="cuda")
    worst = 0.0
    for s in range(steps):
        idx = [prompt[u] + s for u in range(BH)]
        qs = torch.stack([q[idx[u], u] for u in range(BH)]).unsqueeze(1).contiguous()
        ks = torch.stack([k[idx[u], u] for u in range(BH)]).unsqueeze(1).contiguous()
        vs = torch.stack([v[idx[u], u] for u in range(BH)]).contiguous()
        qr = eva.eva_rope(one, qs, rotary_dim=rd, style=style, pos=pos)[:, 0].contiguous()
        kr = eva.eva_rope(one, ks, rotary_dim=rd, style=style, pos=pos)[:, 0].contiguous()
        o, lse = cache.eva_decode_step_ragged(pos, qr, kr, vs)
        of = f64(o)
        for u in range(BH):
            kt = torch.from_numpy(oracle.rope_ex(f64(ks[u]), [idx[u]], rotary_dim=rd, style=st)).to(dtype).double().numpy()[0]
            qt = torch.from_numpy(oracle.rope_ex(f64(qs[u]), [idx[u]], rotary_dim=rd, style=st)).to(dtype).double().numpy()[0]
            assert orc[u].append(kt, f64(vs[u]), E[u, idx[u] // C]) == 0
            ro, rl = orc[u].decode(qt)
            worst = max(worst, np.max(np.abs(of[u] - ro)))
    assert worst <= 2e-2, worst
    assert pos.tolist() == [p + steps for p in prompt]


@pytest.mark.parametrize("style", ["interleaved", "neox"])
@pytest.mark.parametrize("dtype,d,rd,C,W", [(torch.bfloat16, 64, 32, 16, 64), (torch.bfloat16, 128, 128, 64, 128),
                                            (torch.float32, 32, 16, 8, 24)])
def test_ragged_decode_rope_folded(eva, style, dtype, d, rd, C, W):
    """RoPE folded into the one-launch ragged step (eva_decode_step_ragged_rope): q and k_new
    un-rotated in, rotated in registers at each unit's position.  Against the oracle cache fed the
    fp64-rotated keys (stored in dtype, R18) and the fp64-rotated query, and against the two-pass
    form (eva_rope at pos, then eva_decode_step_ragged) on a second cache."""
    BH, steps = 4, 2 * C + 5
    prompt = [0, 9, C * 2 - 1, W + 3]
    cap = (max(prompt) + steps) // C + 1
    cfg = eva.make_config(1, BH, 0, d, C, W, dtype=dtype, seed=25)
    caches = [eva.DecodeCache(cfg, cap, device="cuda") for _ in range(2)]
    orc = [oracle.Cache(d, C, W, oracle.SLIDING, cap=cap, scale=cfg.scale) for _ in range(BH)]
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, BH, cap + 1, d)
    st = oracle.ROPE_NEOX if style == "neox" else oracle.ROPE_INTERLEAVED
    q, k, v = eva_inputs.decode_tokens(0, BH, max(prompt) + steps, d, dtype, seed=26, device="cuda")
    from paper_2511_00576_b200 import _native as N
    one = eva.make_config(1, BH, 1, d, C, W, dtype=dtype, seed=25)
    for u, n in enumerate(prompt):
        if n == 0:
            continue
        kr = eva.eva_rope(eva.make_config(1, 1, n, d, C, W, dtype=dtype), k[:n, u].unsqueeze(0).contiguous(),
                          rotary_dim=rd, style=style)
        for cache in caches:
            view = _unit_view(eva, cache, u)
            N.check(N.lib.eva_cache_append(ctypes.byref(view), kr.data_ptr(),
                                           v[:n, u].unsqueeze(0).contiguous().data_ptr(), n, None, None))
        for t in range(n):
            kt = torch.from_numpy(oracle.rope_ex(f64(k[t, u])[None], [t], rotary_dim=rd, style=st)).to(dtype)
            assert orc[u].append(kt.double().numpy()[0], f64(v[t, u]), E[u, t // C]) == 0
    pos = [torch.tensor(prompt, dtype=torch.int64, device="cuda") for _ in range(2)]
    rope = dict(rope_base=10000.0, rotary_dim=rd, style=style)
    worst, worst2 = 0.0, 0.0
    tol = TOL[dtype]
    for s in range(steps):
        idx = [prompt[u] + s for u in range(BH)]
        qs = torch.stack([q[idx[u], u] for u in range(BH)]).contiguous()
        ks = torch.stack([k[idx[u], u] for u in range(BH)]).contiguous()
        vs = torch.stack([v[idx[u], u] for u in range(BH)]).contiguous()
        o, lse = caches[0].eva_decode_step_ragged(pos[0], qs, ks, vs, rope=rope)
        qr = eva.eva_rope(one, qs.unsqueeze(1).contiguous(), rotary_dim=rd, style=style, pos=pos[1])[:, 0].contiguous()
        kr = eva.eva_rope(one, ks.unsqueeze(1).contiguous(), rotary_dim=rd, style=style, pos=pos[1])[:, 0].contiguous()
        o2, _ = caches[1].eva_decode_step_ragged(pos[1], qr, kr, vs)
        of = f64(o)
        worst2 = max(worst2, (o.float() - o2.float()).abs().max().item())
        for u in range(BH):
            kt = torch.from_numpy(oracle.rope_ex(f64(ks[u])[None], [idx[u]], rotary_dim=rd, style=st)).to(dtype)
            qt = oracle.rope_ex(f64(qs[u])[None], [idx[u]], rotary_dim=rd, style=st)[0]
            assert orc[u].append(kt.double().numpy()[0], f64(vs[u]), E[u, idx[u] // C]) == 0
            ro, rl = orc[u].decode(qt)
            worst = max(worst, np.max(np.abs(of[u] - ro)), abs(float(lse[u]) - rl))
    assert worst <= tol, worst
    assert worst2 <= tol, worst2
    assert pos[0].tolist() == pos[1].tolist() == [p + steps for p in prompt]
    # the rotated keys in the ring and the summaries agree with the two-pass cache
    for a, b in ((caches[0].ring_k, caches[1].ring_k), (caches[0].sum_k, caches[1].sum_k),
                 (caches[0].sum_v, caches[1].sum_v)):
        assert (a.float() - b.float()).abs().max().item() <= tol


def test_ragged_decode_rope_validation(eva):
    cfg = eva.make_config(1, 2, 0, 128, 16, 64)
    cache = eva.DecodeCache(cfg, 4, device="cuda")
    pos = torch.zeros(2, dtype=torch.int64, device="cuda")
    z = torch.zeros(2, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):   # rd / 16 = 3: no shuffle partner
        cache.eva_decode_step_ragged(pos, z, z, z, rope=dict(rotary_dim=48, style="neox"))
    with pytest.raises(eva.EvaError, match="INVALID_ARG"):
        cache.eva_decode_step_ragged(pos, z, z, z, rope=dict(rope_base=0.5))
