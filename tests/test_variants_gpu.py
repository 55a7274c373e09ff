"""GPU parity of the prefill variants (R15, R16) through
the C ABI against the fp64 oracle's oracle_prefill_ext: the non-causal partition and the
summary-logit bias, on the SIMT (fp32, bf16) and tcgen05 (bf16) kernels; the bias in the
decode kernel; and the causal-only entry points refusing the non-causal mode.
Tolerances as in test_parity_gpu.py (north_star: 1e-4 fp32, 2e-2 bf16)."""
import math

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


def _oracle(cfg, Q, K, V, mode, bias):
    E = oracle.eps_units(cfg.seed, cfg.layer, cfg.bh_begin, cfg.bh_count, cfg.T // cfg.chunk, cfg.d_head)
    rk, rv = oracle.summarize_batch(f64(K), f64(V), E, cfg.chunk)
    rO, rl = oracle.prefill_ext_batch(f64(Q), f64(K), f64(V), rk, rv, cfg.chunk, cfg.window, mode,
                                      cfg.scale, bias)
    return rk, rv, rO, rl


# (B, H, T, d, C, W): ragged T (not a multiple of W or of the 128-query tile), W smaller
# than a query tile (rows of one tile in different blocks), W larger, many summary tiles
NC_CASES = [(1, 2, 384, 64, 16, 64), (2, 1, 448, 128, 32, 96), (1, 2, 640, 64, 64, 256),
            (1, 1, 1088, 128, 8, 32), (1, 1, 96, 64, 32, 128), (1, 3, 320, 32, 16, 48)]


@pytest.mark.parametrize("case", NC_CASES)
@pytest.mark.parametrize("dtype,kernel", [(torch.float32, "simt"), (torch.bfloat16, "simt"),
                                          (torch.bfloat16, None)])
def test_noncausal_prefill_parity(eva, case, dtype, kernel):
    B, H, T, d, C, W = case
    if kernel is None and d not in (64, 128):
        pytest.skip("tensor-core kernel covers d in {64, 128}")
    cfg = eva.make_config(B, H, T, d, C, W, mode="noncausal", dtype=dtype, seed=31)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=32, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, kernel=kernel)
    torch.cuda.synchronize()
    rk, rv, rO, rl = _oracle(cfg, Q, K, V, oracle.NONCAUSAL, 0.0)
    tol = TOL[dtype]
    assert np.abs(f64(ks) - rk).max() <= tol and np.abs(f64(vs) - rv).max() <= tol
    assert np.abs(f64(O) - rO).max() <= tol, np.abs(f64(O) - rO).max()
    assert np.abs(f64(lse) - rl).max() <= tol


@pytest.mark.parametrize("dtype,simt", [(torch.float32, True), (torch.bfloat16, False)])
def test_noncausal_window_covers_sequence_is_full_softmax(eva, dtype, simt):
    T, d = 320, 64
    cfg = eva.make_config(1, 2, T, d, 64, 512, mode="noncausal", dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, 2, T, d, dtype, seed=33, device="cuda")
    O, _, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, simt=simt)
    ref = torch.nn.functional.scaled_dot_product_attention(Q.double(), K.double(), V.double(),
                                                           is_causal=False, scale=cfg.scale)
    assert (O.double() - ref).abs().max().item() <= TOL[dtype]


@pytest.mark.parametrize("mode,om", [("sliding", oracle.SLIDING), ("block", oracle.BLOCK),
                                     ("noncausal", oracle.NONCAUSAL)])
@pytest.mark.parametrize("dtype,kernel", [(torch.float32, "simt"), (torch.bfloat16, None)])
@pytest.mark.parametrize("bias", [math.log(64), -1.5])
def test_summary_bias_prefill_parity(eva, mode, om, dtype, kernel, bias):
    B, H, T, d, C, W = 1, 2, 1024, 64, 64, 128
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode, dtype=dtype, seed=34, summary_bias=bias)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=35, device="cuda")
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, kernel=kernel)
    torch.cuda.synchronize()
    _, _, rO, rl = _oracle(cfg, Q, K, V, om, bias)
    assert np.abs(f64(O) - rO).max() <= TOL[dtype]
    assert np.abs(f64(lse) - rl).max() <= TOL[dtype]
    # the bias changes the result (it is applied, not ignored)
    _, _, rO0, _ = _oracle(cfg, Q, K, V, om, 0.0)
    assert np.abs(f64(O) - rO0).max() > 2 * TOL[dtype]


@pytest.mark.parametrize("dtype,d,C,W", [(torch.float32, 32, 8, 24), (torch.bfloat16, 128, 16, 64)])
def test_summary_bias_decode_equals_prefill_rows(eva, dtype, d, C, W):
    """Streaming decode with summary_bias == the oracle's biased prefill at every position."""
    BH, T, bias = 2, 120, math.log(C)
    cfg = eva.make_config(1, BH, 0, d, C, W, dtype=dtype, seed=36, summary_bias=bias)
    cache = eva.DecodeCache(cfg, T // C, device="cuda")
    q, k, v = eva_inputs.decode_tokens(0, BH, T, d, dtype, seed=37, device="cuda")
    outs = []
    for t in range(T):
        o, _ = cache.eva_decode_step(q[t], k[t], v[t])
        outs.append(f64(o))
    torch.cuda.synchronize()
    Qs, Ks, Vs = (x.transpose(0, 1).contiguous() for x in (q, k, v))
    cfgT = eva.make_config(1, BH, T, d, C, W, dtype=dtype, seed=36, summary_bias=bias)
    _, _, rO, _ = _oracle(cfgT, Qs, Ks, Vs, oracle.SLIDING, bias)
    worst = max(np.abs(outs[t] - rO[:, t]).max() for t in range(T))
    assert worst <= TOL[dtype], worst


@pytest.mark.parametrize("dtype,simt", [(torch.float32, True), (torch.bfloat16, False)])
def test_noncausal_sharded_equals_unsharded(eva, dtype, simt):
    B, H, T, d, C, W = 2, 2, 384, 64, 32, 96
    cfg = eva.make_config(B, H, T, d, C, W, mode="noncausal", dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=38, device="cuda")
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, simt=simt)
    c2 = eva.make_config(B, H, T, d, C, W, mode="noncausal", dtype=dtype, bh_begin=1, bh_count=2)
    O2, lse2, _, _ = eva.eva_attn_prefill(c2, Q[1:3].contiguous(), K[1:3].contiguous(), V[1:3].contiguous(),
                                          simt=simt)
    assert torch.equal(O2, O[1:3]) and torch.equal(lse2, lse[1:3])


def test_noncausal_refused_by_causal_entry_points(eva):
    d = 64
    cfg = eva.make_config(1, 1, 0, d, 16, 32, mode="noncausal")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):
        cache = eva.DecodeCache(cfg, 4, device="cuda")
        x = torch.zeros(1, d, dtype=torch.bfloat16, device="cuda")
        cache.eva_cache_append(x, x)
    cfgT = eva.make_config(1, 1, 64, d, 16, 32, mode="noncausal")
    Q = torch.zeros(1, 64, d, dtype=torch.bfloat16, device="cuda")
    S = torch.zeros(1, 4, d, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):
        eva.eva_attn_prefill_range(cfgT, 0, 0, Q, Q, Q, S, S)
    bad = eva.make_config(1, 1, 70, d, 16, 32, mode="noncausal")   # T % C != 0
    Q70 = torch.zeros(1, 70, d, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="INVALID_ARG"):
        eva.eva_attn_prefill(bad, Q70, Q70, Q70)
