"""GPU parity of eva_attn_backward (NEXT row 1) against the fp64 oracle (oracle.backward).

The oracle's gradient is pinned in tests/test_oracle_backward.py (finite
differences, autograd of the direct form, causal-softmax special cases).
Tolerance (reading R20): gradients are sums over many queries, so the bound is
the north_star tolerance on the gradient's own scale (absolute below 1):
    max |GPU - oracle| <= tol * max(1, max |oracle|),  tol = 1e-4 fp32, 2e-2 bf16.
"""
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


def _check(name, got, ref, tol):
    bound = tol * max(1.0, float(np.max(np.abs(ref))) if ref.size else 1.0)
    err = float(np.max(np.abs(got - ref))) if ref.size else 0.0
    assert err <= bound, f"{name}: max err {err:.3e} > {bound:.3e}"


CASES = [  # (B, H, T, d, C, W)
    (1, 1, 256, 16, 16, 32),      # configs[0]
    (1, 2, 300, 32, 8, 24),       # ragged T, W = 3C
    (2, 1, 515, 64, 64, 128),     # configs[1] shape family, ragged tail
    (1, 2, 700, 128, 64, 256),    # configs[2] shape family
    (1, 1, 130, 64, 16, 16),      # W = C
    (1, 1, 40, 64, 64, 128),      # T < C: no summaries
    (1, 1, 1, 128, 4, 8),         # T = 1
    (1, 1, 96, 64, 1, 3),         # C = 1: exact causal softmax gradients
    (1, 1, 1500, 32, 4, 8),       # 375 chunks: several summary tiles and segments
    (1, 1, 2200, 128, 8, 16),     # bf16 tensor-core main pass: 3 summary key tiles, ragged tail
]


@pytest.mark.parametrize("mode", ["sliding", "block"])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_backward_parity(eva, case, mode, dtype):
    B, H, T, d, C, W = case
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode, dtype=dtype, seed=11)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=3, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, dtype, seed=4, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    dQ, dK, dV = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO)
    torch.cuda.synchronize()
    nC = T // C
    E = oracle.eps_units(cfg.seed, cfg.layer, cfg.bh_begin, cfg.bh_count, nC, d)
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    rq, rk, rv = oracle.backward_batch(f64(Q), f64(K), f64(V), E, f64(dO), C, W, m, cfg.scale)
    tol = TOL[dtype]
    _check("dQ", f64(dQ), rq, tol)
    _check("dK", f64(dK), rk, tol)
    _check("dV", f64(dV), rv, tol)


@pytest.mark.parametrize("omega_mode", [0, 1])
def test_backward_caller_eps_and_omega_readings(eva, omega_mode):
    B, H, T, d, C, W = 1, 2, 384, 64, 16, 64
    cfg = eva.make_config(B, H, T, d, C, W, dtype=torch.float32, omega_mode=omega_mode, seed=1)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.float32, seed=5, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.float32, seed=6, device="cuda")
    nC = T // C
    E = eva_inputs.eps(0, B * H, nC, d, seed=8, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, eps=E)
    dQ, dK, dV = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, eps=E)
    torch.cuda.synchronize()
    om = omega_mode
    rq, rk, rv = oracle.backward_batch(f64(Q), f64(K), f64(V), f64(E), f64(dO), C, W,
                                       oracle.SLIDING, cfg.scale, omega_mode=om)
    _check("dQ", f64(dQ), rq, 1e-4)
    _check("dK", f64(dK), rk, 1e-4)
    _check("dV", f64(dV), rv, 1e-4)


def test_backward_sharded_equals_unsharded(eva):
    """A (b, h) shard computes exactly its slice (Philox keyed by the global unit)."""
    B, H, T, d, C, W = 2, 2, 256, 64, 16, 32
    full = eva.make_config(B, H, T, d, C, W, dtype=torch.float32, seed=2)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.float32, seed=9, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.float32, seed=10, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(full, Q, K, V)
    g = eva.eva_attn_backward(full, Q, K, V, ks, vs, O, lse, dO)
    sh = eva.make_config(B, H, T, d, C, W, dtype=torch.float32, seed=2, bh_begin=1, bh_count=2)
    sl = slice(1, 3)
    gs = eva.eva_attn_backward(sh, Q[sl].contiguous(), K[sl].contiguous(), V[sl].contiguous(),
                               ks[sl].contiguous(), vs[sl].contiguous(), O[sl].contiguous(),
                               lse[sl].contiguous(), dO[sl].contiguous())
    torch.cuda.synchronize()
    for a, b in zip(g, gs):
        assert torch.allclose(a[sl], b, rtol=0, atol=1e-5)


def test_backward_workspace_reuse_is_stateless(eva):
    """A dirty workspace gives the same result (the kernels initialise what they accumulate)."""
    B, H, T, d, C, W = 1, 2, 200, 32, 8, 16
    cfg = eva.make_config(B, H, T, d, C, W, dtype=torch.float32, seed=4)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.float32, seed=12, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.float32, seed=13, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    ws = torch.full((eva.eva_backward_workspace_bytes(cfg),), 0x7F, dtype=torch.uint8, device="cuda")
    a = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws)
    a = [t.clone() for t in a]
    b = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.allclose(x, y, rtol=0, atol=1e-6)
    with pytest.raises(eva.EvaError):
        eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws[:1024])


@pytest.mark.parametrize("B,H,T,d,C,W", [(1, 4, 4096, 128, 64, 256), (2, 2, 2048, 64, 64, 128)])
def test_backward_full_size_family(eva, B, H, T, d, C, W):
    """configs[1]/[2] head dims and chunking at T in the thousands, bf16 through the
    tensor-core forward, all elements against the oracle."""
    cfg = eva.make_config(B, H, T, d, C, W, dtype=torch.bfloat16, seed=21)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=22, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=23, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    dQ, dK, dV = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, T // C, d)
    rq, rk, rv = oracle.backward_batch(f64(Q), f64(K), f64(V), E, f64(dO), C, W, oracle.SLIDING,
                                       cfg.scale)
    _check("dQ", f64(dQ), rq, 2e-2)
    _check("dK", f64(dK), rk, 2e-2)
    _check("dV", f64(dV), rv, 2e-2)


# ---- the variants (NEXT row 3): non-causal partition (R15) and the summary-logit bias (R16)
VARIANT_CASES = [  # (B, H, T, d, C, W), T % C == 0 for the non-causal partition
    (1, 1, 256, 16, 16, 32),
    (1, 2, 312, 32, 8, 24),       # W = 3C, last block ragged (312 % 24 = 0, 312 % 64 != 0)
    (2, 1, 576, 64, 64, 128),     # last block half full
    (1, 2, 704, 128, 64, 256),
    (1, 1, 128, 64, 16, 16),      # W = C
    (1, 1, 96, 64, 1, 3),         # C = 1: exact bidirectional softmax gradients
    (1, 1, 2200, 128, 8, 16),     # 275 chunks: 3 summary key tiles on the tensor-core pass
    (1, 1, 40, 64, 8, 64),        # W > T: one block, no summary visible
]


@pytest.mark.parametrize("mode,bias", [("noncausal", 0.0), ("noncausal", "lnC"),
                                       ("sliding", "lnC"), ("block", -0.5)])
@pytest.mark.parametrize("case", VARIANT_CASES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_backward_variant_parity(eva, case, mode, bias, dtype):
    B, H, T, d, C, W = case
    b = float(np.log(C)) if bias == "lnC" else bias
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode, dtype=dtype, seed=17, summary_bias=b)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=21, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, dtype, seed=22, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    dQ, dK, dV = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, cfg.layer, cfg.bh_begin, cfg.bh_count, T // C, d)
    m = {"sliding": oracle.SLIDING, "block": oracle.BLOCK, "noncausal": oracle.NONCAUSAL}[mode]
    rq, rk, rv = oracle.backward_batch(f64(Q), f64(K), f64(V), E, f64(dO), C, W, m, cfg.scale,
                                       bias=b)
    tol = TOL[dtype]
    _check("dQ", f64(dQ), rq, tol)
    _check("dK", f64(dK), rk, tol)
    _check("dV", f64(dV), rv, tol)


def test_backward_noncausal_large_sampled(eva):
    """configs[2]-like rows (d = 128, C = 64, W = 256) at T = 4096 under the non-causal
    partition with bias ln C, tensor-core pass; the oracle runs on 2 units."""
    B, H, T, d, C, W = 1, 2, 4096, 128, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W, mode="noncausal", seed=5, summary_bias=float(np.log(C)))
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=23, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=24, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    dQ, dK, dV = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, T // C, d)
    rq, rk, rv = oracle.backward_batch(f64(Q), f64(K), f64(V), E, f64(dO), C, W, oracle.NONCAUSAL,
                                       cfg.scale, bias=float(np.log(C)))
    _check("dQ", f64(dQ), rq, 2e-2)
    _check("dK", f64(dK), rk, 2e-2)
    _check("dV", f64(dV), rv, 2e-2)


@pytest.mark.parametrize("knob", ["EVA_BACKWARD_FUSED", "EVA_BACKWARD_UNFUSED", "EVA_BACKWARD_SIMT"])
def test_backward_alternate_paths_parity(knob):
    """Schedules chosen by size or by a knob read once per process run in a child pytest with
    the knob set: the fused tensor-core schedule (chain rule in the local tiles' drain; the
    default only from 2^25 elements on) on EVERY bf16 parity and variant case, the one-launch
    schedule with the fp32 dK/dV workspace + finalize (EVA_BACKWARD_UNFUSED) and the SIMT
    main pass for bf16 (EVA_BACKWARD_SIMT) on a subset."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, **{knob: "1"})
    if knob == "EVA_BACKWARD_FUSED":
        sel = ("test_backward_parity and dtype1 or test_backward_variant_parity and dtype1 or "
               "test_backward_bf16_omega_branch")
    else:
        sel = ("test_backward_parity and dtype1 and (case2 or case3 or case9) or "
               "test_backward_variant_parity and dtype1 and case3 or test_backward_bf16_omega_branch")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-x", "-k", sel,
                        "-p", "no:cacheprovider"], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("mode,bias", [("sliding", 0.0), ("noncausal", "lnC")])
def test_backward_large_default_schedule_sampled(eva, mode, bias):
    """configs[2]'s B, H, d, C, W at T = 1024 (2^25 elements: the fused schedule by default),
    oracle on the first and last unit."""
    B, H, T, d, C, W = 8, 32, 1024, 128, 64, 256
    b = float(np.log(C)) if bias == "lnC" else bias
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode, seed=31, summary_bias=b)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=32, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=33, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    dQ, dK, dV = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO)
    torch.cuda.synchronize()
    m = oracle.SLIDING if mode == "sliding" else oracle.NONCAUSAL
    for u in (0, B * H - 1):
        sl = slice(u, u + 1)
        E = oracle.eps_units(cfg.seed, cfg.layer, u, 1, T // C, d)
        rq, rk, rv = oracle.backward_batch(f64(Q[sl]), f64(K[sl]), f64(V[sl]), E, f64(dO[sl]), C, W, m,
                                           cfg.scale, bias=b)
        _check("dQ", f64(dQ[sl]), rq, 2e-2)
        _check("dK", f64(dK[sl]), rk, 2e-2)
        _check("dV", f64(dV[sl]), rv, 2e-2)


def test_backward_configs2_full_size_sampled(eva):
    """BASELINE configs[2] per GPU (B=8, H=32, T=8192, d=128, C=64, W=256) -- the launch the
    bench times (fused schedule) -- with the oracle on the first and last of the 256 units."""
    B, H, T, d, C, W = 8, 32, 8192, 128, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W, seed=1)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=2, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    dQ, dK, dV = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO)
    torch.cuda.synchronize()
    for u in (0, B * H - 1):
        sl = slice(u, u + 1)
        E = oracle.eps_units(cfg.seed, cfg.layer, u, 1, T // C, d)
        rq, rk, rv = oracle.backward_batch(f64(Q[sl]), f64(K[sl]), f64(V[sl]), E, f64(dO[sl]), C, W,
                                           oracle.SLIDING, cfg.scale)
        _check("dQ", f64(dQ[sl]), rq, 2e-2)
        _check("dK", f64(dK[sl]), rk, 2e-2)
        _check("dV", f64(dV[sl]), rv, 2e-2)


# ---- the Eq.15 branch of the bf16 backward (clip-gated omega; reading R14)
OMEGA_CASES = [  # (B, H, T, d, C, W, lam, clip, k_std, v_std)
    (1, 2, 1024, 64, 8, 16, 0.3, 0.3, 0.25, 4.0),
    (1, 2, 1024, 128, 8, 16, 0.3, 0.3, 0.2, 4.0),
    (1, 1, 2048, 64, 16, 32, 0.5, 0.4, 0.3, 3.0),
]


@pytest.mark.parametrize("case", OMEGA_CASES)
def test_backward_bf16_omega_branch(eva, case):
    """bf16 backward where the omega path of Eq.15 is large enough to be seen: lambda != 1,
    a clip bound that gates ~1/3 of the channels, small-norm keys (so the log-xi softmax of
    a chunk spreads over several rows and omega.k matters) and large values (large d beta).
    Sized with torch fp64 autograd of the augmented form: deleting the clip gate, replacing
    lambda by 1 in the gate, or dropping the omega path changes max|dK| by 1.4-5x the bound
    below (mutation check).  Runs on the unfused (register finalize) schedule
    here and on the fused (COEF) schedule in test_backward_alternate_paths_parity."""
    B, H, T, d, C, W, lam, clip, ks_, vs_ = case
    cfg = eva.make_config(B, H, T, d, C, W, seed=91, lam=lam, clip=clip)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.float32, seed=92, device="cuda")
    K = (K * ks_).to(torch.bfloat16)
    V = (V * vs_).to(torch.bfloat16)
    Q = Q.to(torch.bfloat16)
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=93, device="cuda")
    O, lse, ksum, vsum = eva.eva_attn_prefill(cfg, Q, K, V)
    dQ, dK, dV = eva.eva_attn_backward(cfg, Q, K, V, ksum, vsum, O, lse, dO)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, B * H, T // C, d)
    # both sides of the gate are exercised
    kt = f64(K)[:, :T // C * C].reshape(B * H, T // C, C, d).mean(axis=2)
    inside = np.abs(kt + E) <= clip
    assert 0.15 < inside.mean() < 0.85
    rq, rk, rv = oracle.backward_batch(f64(Q), f64(K), f64(V), E, f64(dO), C, W, oracle.SLIDING,
                                       cfg.scale, lam=lam, clip=clip)
    _check("dQ", f64(dQ), rq, 2e-2)
    _check("dK", f64(dK), rk, 2e-2)
    _check("dV", f64(dV), rv, 2e-2)
