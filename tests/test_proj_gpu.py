"""GPU parity of eva_summarize_proj (the learned summary-key projection, NEXT row 4 part,
DESIGN.md R17) against oracle.summarize_proj (pinned in test_oracle_proj.py), and of the
prefill that consumes its summaries against the oracle prefill on the oracle's summaries."""
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


def _proj(H, d, seed):
    g = torch.Generator().manual_seed(seed)
    P = torch.randn(H, d, d, generator=g, dtype=torch.float64) / np.sqrt(d)
    return P


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d,C,T", [(16, 16, 200), (32, 8, 100), (64, 64, 515), (128, 64, 700), (128, 16, 130)])
@pytest.mark.parametrize("philox", [True, False])
def test_summarize_proj_parity(eva, dtype, d, C, T, philox):
    B, H = 2, 3
    cfg = eva.make_config(B, H, T, d, C, 2 * C, dtype=dtype, seed=5, bh_begin=1, bh_count=4)
    _, K, V = eva_inputs.qkv(1, 4, T, d, dtype, seed=2, device="cuda")
    nC = T // C
    eps = None if philox else eva_inputs.eps(1, 4, nC, d, device="cuda")
    P = _proj(H, d, d + C)
    ks, vs = eva.eva_summarize_proj(cfg, K, V, P.float().cuda(), eps=eps)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, cfg.layer, 1, 4, nC, d) if philox else f64(eps)
    # the kernel reads the fp32 projection: the oracle gets the same fp32-rounded values
    Pf = P.float().double().numpy()
    for u in range(4):
        h = (1 + u) % H
        rk, rv = oracle.summarize_proj(f64(K[u]), f64(V[u]), E[u], Pf[h], C)
        assert np.max(np.abs(f64(ks[u]) - rk)) <= TOL[dtype], u
        assert np.max(np.abs(f64(vs[u]) - rv)) <= TOL[dtype], u


def test_identity_projection_equals_summarize(eva):
    B, H, T, d, C = 1, 2, 256, 64, 32
    cfg = eva.make_config(B, H, T, d, C, 64, dtype=torch.float32, seed=8)
    _, K, V = eva_inputs.qkv(0, 2, T, d, torch.float32, seed=3, device="cuda")
    I = torch.eye(d, device="cuda").expand(H, d, d).contiguous()
    a = eva.eva_summarize(cfg, K, V)
    b = eva.eva_summarize_proj(cfg, K, V, I)
    torch.cuda.synchronize()
    assert torch.allclose(a[0], b[0], rtol=0, atol=1e-6) and torch.allclose(a[1], b[1], rtol=0, atol=1e-6)


def test_prefill_on_projected_summaries(eva):
    """The prefill consumes the projected summaries unchanged (EVA_SUMMARIES_PROVIDED)."""
    B, H, T, d, C, W = 1, 2, 700, 128, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W, seed=6)
    Q, K, V = eva_inputs.qkv(0, 2, T, d, torch.bfloat16, seed=4, device="cuda")
    P = _proj(H, d, 77)
    ks, vs = eva.eva_summarize_proj(cfg, K, V, P.float().cuda())
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, 2, T // C, d)
    Pf = P.float().double().numpy()
    for u in range(2):
        rk, rv = oracle.summarize_proj(f64(K[u]), f64(V[u]), E[u], Pf[u % H], C)
        ro, rl = oracle.prefill(f64(Q[u]), f64(K[u]), f64(V[u]), rk, rv, C, W, oracle.SLIDING, cfg.scale)
        assert np.max(np.abs(f64(O[u]) - ro)) <= 2e-2
        assert np.max(np.abs(f64(lse[u]) - rl)) <= 2e-2


def test_summarize_proj_validation(eva):
    cfg = eva.make_config(1, 1, 64, 64, 16, 32)
    K = torch.zeros(1, 64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        eva.eva_summarize_proj(cfg, K, K, torch.zeros(1, 64, 32, device="cuda"))
    big = eva.make_config(1, 1, 8192, 128, 4096, 4096)   # chunk too long for the register summariser
    K2 = torch.zeros(1, 8192, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):
        eva.eva_summarize_proj(big, K2, K2, torch.zeros(1, 128, 128, device="cuda"))


# ---------------------------------------------------------------- backward through the projection
def _bwd_tol(ref):
    return 2e-2 * max(1.0, float(np.max(np.abs(ref))))


@pytest.mark.parametrize("d,C,T,W", [(64, 64, 515, 128), (128, 64, 700, 256), (64, 16, 300, 32), (32, 32, 260, 64)])
@pytest.mark.parametrize("fused", [False, True])
def test_backward_proj_parity(eva, d, C, T, W, fused, monkeypatch):
    """eva_attn_backward_proj (bf16) vs oracle.backward_proj (pinned by finite differences): dQ,
    dK, dV per unit and dP summed over the units of each head; lambda = 1 and eps scaled so the
    Eq.15 clip bites -- the omega path carries weight.  fused: the
    tcgen05 schedule with the chain-rule coefficients (EVA_BACKWARD_FUSED, d in {64, 128})."""
    if fused and d not in (64, 128):
        pytest.skip("the fused schedule is the tcgen05 path (d in {64, 128})")
    import subprocess, sys, os, json
    B, H = 2, 3
    cfg = eva.make_config(B, H, T, d, C, W, seed=5, bh_begin=1, bh_count=4, lam=1.0)
    Q, K, V = eva_inputs.qkv(1, 4, T, d, torch.bfloat16, seed=2, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 1, 4, T, d, torch.bfloat16, seed=3, device="cuda")
    nC = T // C
    eps = (1.5 * eva_inputs.eps(1, 4, nC, d, device="cuda")).contiguous()
    P = _proj(H, d, d + C + 1)
    Pc = P.float().cuda()
    ks, vs = eva.eva_summarize_proj(cfg, K, V, Pc, eps=eps)
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True)
    if fused and os.environ.get("EVA_BACKWARD_FUSED") != "1":
        # the schedule knob is read once per process: rerun this case in a child with it set
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                            f"{__file__}::test_backward_proj_parity[True-{d}-{C}-{T}-{W}]"],
                           env=dict(os.environ, EVA_BACKWARD_FUSED="1"), capture_output=True, text=True,
                           timeout=600, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
        return
    dQ, dK, dV, dP = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, eps=eps, Pk=Pc)
    torch.cuda.synchronize()
    Pf = P.float().double().numpy()
    E = f64(eps)
    dP_ref = np.zeros((H, d, d))
    for u in range(4):
        h = (1 + u) % H
        rq, rk, rv, rp = oracle.backward_proj(f64(Q[u]), f64(K[u]), f64(V[u]), E[u], Pf[h], f64(dO[u]), C, W,
                                              scale=cfg.scale, lam=1.0)
        dP_ref[h] += rp
        for got, want, nm in ((dQ[u], rq, "dQ"), (dK[u], rk, "dK"), (dV[u], rv, "dV")):
            err = np.max(np.abs(f64(got) - want))
            assert err <= _bwd_tol(want), (nm, u, err)
    err = np.max(np.abs(f64(dP) - dP_ref))
    assert err <= 2e-2 * max(1.0, float(np.max(np.abs(dP_ref)))), err
    # the projection path carries weight: with P replaced by I the outputs move by more than the tolerance
    if not fused:
        Ic = torch.eye(d, device="cuda").expand(H, d, d).contiguous()
        d2 = eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, eps=eps, Pk=Ic)
        assert float((d2[1].float() - dK.float()).abs().max()) > 2e-2


def test_backward_proj_rejects_unsupported(eva):
    cfg = eva.make_config(1, 1, 64, 64, 16, 32, dtype=torch.float32)
    Z = torch.zeros(1, 64, 64, device="cuda")
    P = torch.zeros(1, 64, 64, device="cuda")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):
        eva.eva_attn_backward(cfg, Z, Z, Z, Z[:, :4], Z[:, :4], Z, torch.zeros(1, 64, device="cuda"), Z, Pk=P)
