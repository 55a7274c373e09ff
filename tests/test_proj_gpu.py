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
