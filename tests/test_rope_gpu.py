"""GPU parity of eva_rope_summarize (the fused RoPE producer, NEXT row 4 part, DESIGN.md
R18) against oracle.rope (pinned in test_oracle_rope.py) + oracle.summarize, and of the
prefill on its outputs against the oracle prefill on the fp64-rotated inputs."""
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


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("B,H,T,d,C,W", [(1, 2, 200, 16, 16, 32), (1, 2, 515, 64, 64, 128),
                                         (1, 1, 700, 128, 64, 256), (1, 1, 40, 64, 64, 128),
                                         (2, 1, 1000, 32, 8, 24)])
def test_rope_summarize_parity(eva, dtype, B, H, T, d, C, W):
    base = 10000.0
    cfg = eva.make_config(B, H, T, d, C, W, dtype=dtype, seed=9)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=10, device="cuda")
    Qr, Kr, ks, vs = eva.eva_rope_summarize(cfg, Q, K, V, rope_base=base)
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Qr, Kr, V, Ksum=ks, Vsum=vs, summaries_provided=True)
    torch.cuda.synchronize()
    nC = T // C
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, nC, d)
    tol = TOL[dtype]
    def stored(x):  # R18: the producer stores RoPE(Q), RoPE(K) in cfg.dtype (RNE) and
        # summarises / attends those stored values -- applied here to the oracle's own output
        return torch.from_numpy(x).to(dtype).double().numpy()

    for u in range(B * H):
        rq = oracle.rope(f64(Q[u]), base)
        rk = oracle.rope(f64(K[u]), base)
        assert np.max(np.abs(f64(Qr[u]) - rq)) <= tol
        assert np.max(np.abs(f64(Kr[u]) - rk)) <= tol
        rq, rk = stored(rq), stored(rk)
        sk, sv = oracle.summarize(rk, f64(V[u]), E[u], C)
        if nC:
            assert np.max(np.abs(f64(ks[u]) - sk)) <= tol
            assert np.max(np.abs(f64(vs[u]) - sv)) <= tol
        ro, rl = oracle.prefill(rq, rk, f64(V[u]), sk, sv, C, W, oracle.SLIDING, cfg.scale)
        assert np.max(np.abs(f64(O[u]) - ro)) <= tol
        assert np.max(np.abs(f64(lse[u]) - rl)) <= tol


def test_rope_summarize_validation(eva):
    cfg = eva.make_config(1, 1, 64, 64, 16, 32)
    X = torch.zeros(1, 64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="INVALID_ARG"):
        eva.eva_rope_summarize(cfg, X, X, X, rope_base=0.5)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d,T,pos0", [(16, 50, 0), (64, 300, 0), (128, 1, 4097)])
def test_rope_and_inverse(eva, dtype, d, T, pos0):
    """eva_rope vs oracle.rope; the inverse is the transpose: rows against oracle.rope at the
    negated position (R(-a) = R(a)^T per pair), and inverse(rope(X)) = X."""
    cfg = eva.make_config(1, 2, T, d, 1, 1, dtype=dtype)
    (X,) = eva_inputs.normal_units(1, 0, 2, T, d, dtype, seed=31, device="cuda")
    Y = eva.eva_rope(cfg, X, pos0=pos0)
    Z = eva.eva_rope(cfg, X, pos0=pos0, inverse=True)
    back = eva.eva_rope(cfg, Y, pos0=pos0, inverse=True)
    torch.cuda.synchronize()
    tol = TOL[dtype]
    for u in range(2):
        assert np.max(np.abs(f64(Y[u]) - oracle.rope(f64(X[u]), pos0=pos0))) <= tol
        want_inv = np.concatenate([oracle.rope(f64(X[u, t:t + 1]), pos0=-(pos0 + t)) for t in range(T)])
        assert np.max(np.abs(f64(Z[u]) - want_inv)) <= tol
    assert np.max(np.abs(f64(back) - f64(X))) <= 2 * tol


def test_rope_in_place(eva):
    cfg = eva.make_config(1, 1, 64, 64, 1, 1)
    (X,) = eva_inputs.normal_units(1, 0, 1, 64, 64, torch.bfloat16, seed=32, device="cuda")
    want = eva.eva_rope(cfg, X, pos0=5)
    eva.eva_rope(cfg, X, pos0=5, out=X)
    torch.cuda.synchronize()
    assert torch.equal(X, want)


def test_training_chain_with_rope(eva):
    """Forward through the fused RoPE producer, eva_attn_backward on the rotated inputs, then
    the transposed rotation: dQ, dK, dV of L = sum(dO * O(rope(Q), rope(K), V)) against the
    oracle's backward on its own rotated (stored-precision) inputs followed by R^T per row."""
    B, H, T, d, C, W = 1, 2, 300, 64, 16, 64
    cfg = eva.make_config(B, H, T, d, C, W, seed=12)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=13, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=14, device="cuda")
    Qr, Kr, ks, vs = eva.eva_rope_summarize(cfg, Q, K, V)
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Qr, Kr, V, Ksum=ks, Vsum=vs, summaries_provided=True)
    dQr, dKr, dV = eva.eva_attn_backward(cfg, Qr, Kr, V, ks, vs, O, lse, dO)
    dQ = eva.eva_rope(cfg, dQr, inverse=True)
    dK = eva.eva_rope(cfg, dKr, inverse=True)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, T // C, d)
    for u in range(B * H):
        rq = torch.from_numpy(oracle.rope(f64(Q[u]))).to(torch.bfloat16).double().numpy()
        rk = torch.from_numpy(oracle.rope(f64(K[u]))).to(torch.bfloat16).double().numpy()
        gq, gk, gv = oracle.backward(rq, rk, f64(V[u]), E[u], f64(dO[u]), C, W, oracle.SLIDING, cfg.scale)
        # R^T per row = the rotation at the negated position
        gq = np.concatenate([oracle.rope(gq[t:t + 1], pos0=-t) for t in range(T)])
        gk = np.concatenate([oracle.rope(gk[t:t + 1], pos0=-t) for t in range(T)])
        for name, got, want in (("dQ", dQ[u], gq), ("dK", dK[u], gk), ("dV", dV[u], gv)):
            err = np.max(np.abs(f64(got) - want))
            assert err <= 2e-2 * max(1.0, np.max(np.abs(want))), (name, u, err)


# ------------------------------------------------------------------ R19: rotary_dim, half-split,
# per-unit device positions (the ragged decode batch), against oracle.rope_ex
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d,rd", [(64, 16), (64, 64), (128, 32), (128, 128), (32, 16)])
@pytest.mark.parametrize("style", ["interleaved", "neox"])
@pytest.mark.parametrize("inverse", [False, True])
def test_rope_ex_parity(eva, dtype, d, rd, style, inverse):
    BH, T = 5, 37
    cfg = eva.make_config(1, BH, T, d, 16, 32, dtype=dtype)
    (X,) = eva_inputs.normal_units(1, 0, BH, T, d, dtype, seed=41, device="cuda")
    pos = torch.tensor([0, 7, 4096, 123457, 2 ** 31 + 5], dtype=torch.int64, device="cuda")
    Y = eva.eva_rope(cfg, X, rope_base=500.0, rotary_dim=rd, style=style, pos=pos, inverse=inverse)
    torch.cuda.synchronize()
    st = oracle.ROPE_NEOX if style == "neox" else oracle.ROPE_INTERLEAVED
    worst = 0.0
    for u in range(BH):
        p = int(pos[u]) + np.arange(T)
        want = oracle.rope_ex(f64(X[u]), p, base=500.0, rotary_dim=rd, style=st, inverse=inverse)
        worst = max(worst, np.max(np.abs(f64(Y[u]) - want)))
        # pass-through channels are copied exactly
        assert torch.equal(Y[u, :, rd:], X[u, :, rd:])
    # bf16 output rounding: 2^-8 of |y| <= a few units; fp32 angle reduction at 2^31
    assert worst <= (2e-2 if dtype == torch.bfloat16 else 2e-4), worst
    # scalar pos0 path: the same as a pos array of equal positions
    Y0 = eva.eva_rope(cfg, X, rope_base=500.0, rotary_dim=rd, style=style, pos0=4096, inverse=inverse)
    Y1 = eva.eva_rope(cfg, X, rope_base=500.0, rotary_dim=rd, style=style,
                      pos=torch.full((BH,), 4096, dtype=torch.int64, device="cuda"), inverse=inverse)
    assert torch.equal(Y0, Y1)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d,rd,style", [(64, 16, "neox"), (128, 128, "neox"), (128, 32, "interleaved"),
                                        (64, 32, "neox")])
def test_rope_summarize_ex_parity(eva, dtype, d, rd, style):
    """The fused producer with rotary_dim / half-split pairs (partner pieces exchanged between
    lanes): Qr, Kr, the summaries of the rotated keys and the prefill on them vs the oracle."""
    B, H, T, C, W = 1, 3, 300, 32, 64
    cfg = eva.make_config(B, H, T, d, C, W, dtype=dtype, seed=19)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=20, device="cuda")
    Qr, Kr, ks, vs = eva.eva_rope_summarize(cfg, Q, K, V, rope_base=10000.0, rotary_dim=rd, style=style)
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Qr, Kr, V, Ksum=ks, Vsum=vs, summaries_provided=True)
    torch.cuda.synchronize()
    st = oracle.ROPE_NEOX if style == "neox" else oracle.ROPE_INTERLEAVED
    nC = T // C
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, nC, d)
    tol = TOL[dtype]
    for u in range(B * H):
        p = np.arange(T)
        rq = oracle.rope_ex(f64(Q[u]), p, rotary_dim=rd, style=st)
        rk = oracle.rope_ex(f64(K[u]), p, rotary_dim=rd, style=st)
        assert np.max(np.abs(f64(Qr[u]) - rq)) <= tol
        assert np.max(np.abs(f64(Kr[u]) - rk)) <= tol
        rq = torch.from_numpy(rq).to(dtype).double().numpy()
        rk = torch.from_numpy(rk).to(dtype).double().numpy()
        sk, sv = oracle.summarize(rk, f64(V[u]), E[u], C)
        assert np.max(np.abs(f64(ks[u]) - sk)) <= tol
        assert np.max(np.abs(f64(vs[u]) - sv)) <= tol
        ro, rl = oracle.prefill(rq, rk, f64(V[u]), sk, sv, C, W, oracle.SLIDING, cfg.scale)
        assert np.max(np.abs(f64(O[u]) - ro)) <= tol


def test_rope_ex_validation(eva):
    cfg = eva.make_config(1, 1, 8, 64, 16, 32)
    X = torch.zeros(1, 8, 64, dtype=torch.bfloat16, device="cuda")
    for kw in (dict(rotary_dim=24), dict(rotary_dim=80), dict(rotary_dim=8), dict(style=2)):
        with pytest.raises((eva.EvaError, KeyError, ValueError)):
            eva.eva_rope(cfg, X, **kw)
    cfg = eva.make_config(1, 1, 96, 128, 32, 64)
    Z = torch.zeros(1, 96, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):   # rd / 16 = 3: no butterfly partner
        eva.eva_rope_summarize(cfg, Z, Z, Z, rotary_dim=48, style="neox")


# ------------------------------------------------------------------ RoPE inside the tensor-core
# prefill (eva_attn_prefill_rope): the kernel rotates the landed Q / local-K tiles in shared
# memory; compared with the oracle on the fp64-rotated inputs rounded to bf16 (R18: the rotated
# values the MMA reads are bf16), and with the two-pass path (rope-summarize + prefill).
@pytest.mark.parametrize("B,H,T,d,C,W,rd,style,mode", [
    (1, 2, 515, 64, 64, 128, 64, "interleaved", 0),
    (1, 2, 515, 64, 64, 128, 16, "neox", 0),
    (1, 1, 700, 128, 64, 256, 128, "interleaved", 0),
    (1, 1, 700, 128, 64, 256, 128, "neox", 0),
    (2, 1, 1000, 128, 32, 96, 32, "interleaved", 1),
    (1, 2, 640, 64, 16, 64, 32, "neox", 1),
    (1, 1, 100, 64, 64, 128, 64, "interleaved", 0),
    (1, 3, 40, 128, 64, 128, 128, "neox", 0),      # T < C: no summaries, one partial tile
    (1, 1, 600, 128, 128, 256, 64, "interleaved", 0),   # C = 128 (the bulk RoPE summariser's largest chunk)
    (1, 2, 520, 64, 32, 64, 16, "neox", 1),        # rotary_dim 16: one half-split piece pair per row
])
def test_prefill_rope_in_kernel_parity(eva, B, H, T, d, C, W, rd, style, mode):
    base = 10000.0
    cfg = eva.make_config(B, H, T, d, C, W, seed=23, mode=mode)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=24, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill_rope(cfg, Q, K, V, rope_base=base, rotary_dim=rd, style=style)
    # the two-pass path on the same inputs
    Qr, Kr, ks2, vs2 = eva.eva_rope_summarize(cfg, Q, K, V, rope_base=base, rotary_dim=rd, style=style)
    O2, lse2, _, _ = eva.eva_attn_prefill(cfg, Qr, Kr, V, Ksum=ks2, Vsum=vs2, summaries_provided=True)
    # summaries provided: the same call on the summaries the first call computed
    O3, lse3, _, _ = eva.eva_attn_prefill_rope(cfg, Q, K, V, rope_base=base, rotary_dim=rd, style=style,
                                               Ksum=ks.clone(), Vsum=vs.clone(), summaries_provided=True)
    torch.cuda.synchronize()
    # the bulk summariser rotates the landed keys with its own recurrence: same values up to
    # the bf16 rounding of a rotated key
    if T // C:
        assert (ks.float() - ks2.float()).abs().max().item() <= 2e-2
        assert (vs.float() - vs2.float()).abs().max().item() <= 2e-2
    assert torch.equal(O, O3) and torch.equal(lse, lse3)
    assert (O.float() - O2.float()).abs().max().item() <= 2e-2
    st = oracle.ROPE_NEOX if style == "neox" else oracle.ROPE_INTERLEAVED
    nC = T // C
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, nC, d)
    omode = oracle.SLIDING if mode == 0 else oracle.BLOCK
    for u in range(B * H):
        p = np.arange(T)
        rq = torch.from_numpy(oracle.rope_ex(f64(Q[u]), p, base=base, rotary_dim=rd, style=st)).to(torch.bfloat16)
        rk = torch.from_numpy(oracle.rope_ex(f64(K[u]), p, base=base, rotary_dim=rd, style=st)).to(torch.bfloat16)
        rq, rk = rq.double().numpy(), rk.double().numpy()
        sk, sv = oracle.summarize(rk, f64(V[u]), E[u], C)
        if nC:
            assert np.max(np.abs(f64(ks[u]) - sk)) <= 2e-2
        ro, rl = oracle.prefill(rq, rk, f64(V[u]), sk, sv, C, W, omode, cfg.scale)
        assert np.max(np.abs(f64(O[u]) - ro)) <= 2e-2
        assert np.max(np.abs(f64(lse[u]) - rl)) <= 2e-2


def test_prefill_rope_in_kernel_long_positions(eva):
    """configs[2]'s per-unit shape (T = 8192, d = 128, C = 64, W = 256) on 2 units: positions up
    to 8191 exercise the rotation recurrence over whole tiles; sampled query rows vs the oracle."""
    B, H, T, d, C, W = 1, 2, 8192, 128, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W, seed=29)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=30, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill_rope(cfg, Q, K, V, rope_base=10000.0)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, T // C, d)
    rows = np.array([0, 1, 127, 128, 4095, 4096, 6000, 8064, 8191])
    for u in range(B * H):
        p = np.arange(T)
        rq = torch.from_numpy(oracle.rope_ex(f64(Q[u]), p, base=10000.0)).to(torch.bfloat16).double().numpy()
        rk = torch.from_numpy(oracle.rope_ex(f64(K[u]), p, base=10000.0)).to(torch.bfloat16).double().numpy()
        sk, sv = oracle.summarize(rk, f64(V[u]), E[u], C)
        ro, rl = oracle.prefill(rq, rk, f64(V[u]), sk, sv, C, W, oracle.SLIDING, cfg.scale)
        assert np.max(np.abs(f64(O[u])[rows] - ro[rows])) <= 2e-2
        assert np.max(np.abs(f64(O[u]) - ro)) <= 2e-2


def test_prefill_rope_in_kernel_validation(eva):
    cfg = eva.make_config(1, 1, 256, 64, 16, 32, dtype=torch.float32)
    Z = torch.zeros(1, 256, 64, dtype=torch.float32, device="cuda")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):   # the tensor-core path is bf16
        eva.eva_attn_prefill_rope(cfg, Z, Z, Z)
    cfg = eva.make_config(1, 1, 256, 128, 16, 32)
    Z = torch.zeros(1, 256, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):   # rotary_dim not a power of two
        eva.eva_attn_prefill_rope(cfg, Z, Z, Z, rotary_dim=96)
    cfg = eva.make_config(1, 1, 256, 32, 16, 32)
    Z = torch.zeros(1, 256, 32, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):   # d = 32: no tensor-core kernel
        eva.eva_attn_prefill_rope(cfg, Z, Z, Z)


@pytest.mark.parametrize("mode,bias,T", [("noncausal", 0.0, 512), ("sliding", 0.7, 700), ("block", -0.4, 576)])
def test_prefill_rope_in_kernel_variants(eva, mode, bias, T):
    """In-kernel RoPE with the non-causal partition (R15) and the summary-logit bias (R16):
    against oracle_prefill_ext on the bf16-stored fp64-rotated inputs."""
    B, H, d, C, W = 1, 2, 128, 64, 128
    m = {"sliding": 0, "block": 1, "noncausal": 2}[mode]
    cfg = eva.make_config(B, H, T, d, C, W, seed=31, mode=mode, summary_bias=bias)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=32, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill_rope(cfg, Q, K, V, rope_base=10000.0, rotary_dim=64, style="neox")
    torch.cuda.synchronize()
    nC = T // C
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, nC, d)
    p = np.arange(T)
    rq = np.stack([torch.from_numpy(oracle.rope_ex(f64(Q[u]), p, rotary_dim=64, style=oracle.ROPE_NEOX))
                   .to(torch.bfloat16).double().numpy() for u in range(B * H)])
    rk = np.stack([torch.from_numpy(oracle.rope_ex(f64(K[u]), p, rotary_dim=64, style=oracle.ROPE_NEOX))
                   .to(torch.bfloat16).double().numpy() for u in range(B * H)])
    sk, sv = oracle.summarize_batch(rk, f64(V), E, C)
    assert np.max(np.abs(f64(ks) - sk)) <= 2e-2
    ro, rl = oracle.prefill_ext_batch(rq, rk, f64(V), f64(ks), f64(vs), C, W, m, cfg.scale, bias)
    assert np.max(np.abs(f64(O) - ro)) <= 2e-2
    assert np.max(np.abs(f64(lse) - rl)) <= 2e-2


def test_ragged_rope_ignores_two_launch_switch():
    """EVA_RAGGED_TWO_LAUNCH=1 selects the two-launch ragged form; RoPE is folded into the
    one-launch form only, so the RoPE step must still run (and equal the default process's)."""
    import os
    import subprocess
    import sys
    code = (
        "import torch, eva_inputs, paper_2511_00576_b200 as eva\n"
        "cfg = eva.make_config(1, 4, 0, 64, 16, 64)\n"
        "c = eva.DecodeCache(cfg, 8, device='cuda')\n"
        "pos = torch.tensor([0, 3, 15, 40], dtype=torch.int64, device='cuda')\n"
        "q, k, v = eva_inputs.decode_tokens(0, 4, 20, 64, torch.bfloat16, seed=3, device='cuda')\n"
        "outs = []\n"
        "for i in range(20):\n"
        "    o, _ = c.eva_decode_step_ragged(pos, q[i], k[i], v[i], rope=dict(rotary_dim=32, style='neox'))\n"
        "    outs.append(o.float().cpu())\n"
        "torch.save(torch.stack(outs), '/tmp/eva_rr_%s.pt' % __import__('os').environ.get('EVA_RAGGED_TWO_LAUNCH', '0'))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for flag in ("0", "1"):
        env = dict(os.environ, EVA_RAGGED_TWO_LAUNCH=flag, PYTHONPATH=root)
        r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
    a, b = torch.load("/tmp/eva_rr_0.pt"), torch.load("/tmp/eva_rr_1.pt")
    assert torch.equal(a, b)


@pytest.mark.parametrize("d,rd,style,mode", [(128, 128, "interleaved", "sliding"), (64, 32, "neox", "block"),
                                             (128, 64, "neox", "noncausal")])
def test_prefill_rope_k_prerotated(eva, d, rd, style, mode):
    """EVA_ROPE_K_ROTATED: K comes in rotated (eva_rope's output), the kernel rotates Q only and
    the summaries are the plain summariser's on the rotated keys.  Against the oracle on the
    bf16-stored rotated inputs, and against the full in-kernel path."""
    B, H, T, C, W = 1, 2, 768, 64, 128
    m = {"sliding": 0, "block": 1, "noncausal": 2}[mode]
    cfg = eva.make_config(B, H, T, d, C, W, seed=33, mode=mode)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=34, device="cuda")
    Kr = eva.eva_rope(cfg, K, rotary_dim=rd, style=style)
    O, lse, ks, vs = eva.eva_attn_prefill_rope(cfg, Q, Kr, V, rotary_dim=rd, style=style, k_rotated=True)
    O2, lse2, ks2, vs2 = eva.eva_attn_prefill_rope(cfg, Q, K, V, rotary_dim=rd, style=style)
    torch.cuda.synchronize()
    assert (O.float() - O2.float()).abs().max().item() <= 2e-2
    assert (ks.float() - ks2.float()).abs().max().item() <= 2e-2
    st = oracle.ROPE_NEOX if style == "neox" else oracle.ROPE_INTERLEAVED
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, T // C, d)
    p = np.arange(T)
    rq = np.stack([torch.from_numpy(oracle.rope_ex(f64(Q[u]), p, rotary_dim=rd, style=st))
                   .to(torch.bfloat16).double().numpy() for u in range(B * H)])
    rk = np.stack([torch.from_numpy(oracle.rope_ex(f64(K[u]), p, rotary_dim=rd, style=st))
                   .to(torch.bfloat16).double().numpy() for u in range(B * H)])
    sk, sv = oracle.summarize_batch(rk, f64(V), E, C)
    assert np.max(np.abs(f64(ks) - sk)) <= 2e-2
    ro, rl = oracle.prefill_ext_batch(rq, rk, f64(V), f64(ks), f64(vs), C, W, m, cfg.scale)
    assert np.max(np.abs(f64(O) - ro)) <= 2e-2
    assert np.max(np.abs(f64(lse) - rl)) <= 2e-2


@pytest.mark.parametrize("style", ["interleaved", "neox"])
def test_rope_prefill_to_decode_handoff(eva, style):
    """The RoPE serving path end to end: RoPE(K) once (eva_rope), the prefill rotating Q only
    (EVA_ROPE_K_ROTATED), the cache loaded with the rotated keys and the prefill's summaries, then
    decode tokens with RoPE folded into the ragged step -- against the oracle's streaming cache on
    the bf16-stored rotated keys (R18) and the fp64-rotated queries."""
    B, H, T, d, C, W, rd = 1, 2, 300, 64, 16, 64, 32
    BH, steps = B * H, 20
    cfg = eva.make_config(B, H, T, d, C, W, seed=41)
    Q, K, V = eva_inputs.qkv(0, BH, T, d, torch.bfloat16, seed=42, device="cuda")
    Kr = eva.eva_rope(cfg, K, rotary_dim=rd, style=style)
    O, lse, ks, vs = eva.eva_attn_prefill_rope(cfg, Q, Kr, V, rotary_dim=rd, style=style, k_rotated=True)
    cap = (T + steps) // C + 1
    cache = eva.DecodeCache(cfg, cap, device="cuda")
    cache.eva_cache_load(Kr, V, ks, vs)
    q, k, v = eva_inputs.decode_tokens(0, BH, steps, d, torch.bfloat16, seed=43, device="cuda")
    pos = torch.full((BH,), T, dtype=torch.int64, device="cuda")
    outs = []
    for i in range(steps):
        o, l = cache.eva_decode_step_ragged(pos, q[i], k[i], v[i], rope=dict(rotary_dim=rd, style=style))
        outs.append((o.clone(), l.clone()))
    torch.cuda.synchronize()
    st = oracle.ROPE_NEOX if style == "neox" else oracle.ROPE_INTERLEAVED
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, BH, cap + 1, d)
    worst = 0.0
    for u in range(BH):
        orc = oracle.Cache(d, C, W, oracle.SLIDING, cap=cap, scale=cfg.scale)
        rk = torch.from_numpy(oracle.rope_ex(f64(K[u]), np.arange(T), rotary_dim=rd, style=st)).to(torch.bfloat16)
        rk = rk.double().numpy()
        for t in range(T):
            assert orc.append(rk[t], f64(V[u, t]), E[u, t // C]) == 0
        # the prefill's last row equals the streaming cache's decode at position T - 1
        rq_last = oracle.rope_ex(f64(Q[u, T - 1])[None], [T - 1], rotary_dim=rd, style=st)
        rq_last = torch.from_numpy(rq_last).to(torch.bfloat16).double().numpy()[0]
        ro, _ = orc.decode(rq_last)
        worst = max(worst, np.max(np.abs(f64(O[u, T - 1]) - ro)))
        for i in range(steps):
            kt = torch.from_numpy(oracle.rope_ex(f64(k[i, u])[None], [T + i], rotary_dim=rd, style=st)).to(torch.bfloat16)
            qt = oracle.rope_ex(f64(q[i, u])[None], [T + i], rotary_dim=rd, style=st)[0]
            assert orc.append(kt.double().numpy()[0], f64(v[i, u]), E[u, (T + i) // C]) == 0
            ro, rl = orc.decode(qt)
            worst = max(worst, np.max(np.abs(f64(outs[i][0][u]) - ro)), abs(float(outs[i][1][u]) - rl))
    assert worst <= 2e-2, worst
    assert pos.tolist() == [T + steps] * BH
