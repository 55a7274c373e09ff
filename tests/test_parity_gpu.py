"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle.

Tolerances (north_star): max |GPU - oracle| <= 1e-4 on the fp32
path and <= 2e-2 on the bf16 path for O, LSE, Ksum, Vsum on unit-variance
inputs; mask ranges and Philox words bit-exact.  Both sides consume the same
seeded inputs (eva_inputs) and the same eps (caller-supplied, or the two
independent Philox implementations).
"""
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


def oracle_eps_for(cfg, nC, d):
    return oracle.eps_units(cfg.seed, cfg.layer, cfg.bh_begin, cfg.bh_count, nC, d)


def run_oracle(Q, K, V, E, C, W, mode, scale):
    ks, vs = oracle.summarize_batch(f64(K), f64(V), E, C)
    O, lse = oracle.prefill_batch(f64(Q), f64(K), f64(V), ks, vs, C, W, mode, scale)
    return ks, vs, O, lse


# ----------------------------------------------------------------------------- bit-exact pieces
def test_philox_bit_exact(eva):
    rng = np.random.default_rng(0)
    blocks = rng.integers(0, 2 ** 32, size=(256, 6), dtype=np.uint64).astype(np.int64)
    blocks[0] = 0
    blocks[1] = 0xFFFFFFFF
    out = eva.eva_philox(torch.from_numpy(blocks)).cpu().numpy()
    for i in range(blocks.shape[0]):
        b = [int(x) for x in blocks[i]]
        assert [int(x) for x in out[i]] == oracle.philox4x32_10(b[:4], b[4:])


@pytest.mark.parametrize("d", [16, 64, 128])
def test_draw_eps_matches_oracle(eva, d):
    cfg = eva.make_config(2, 3, 640, d, 64, 128, bh_begin=1, bh_count=4, seed=0xABCDEF0123, layer=5)
    e = f64(eva.eva_draw_eps(cfg))
    ref = oracle_eps_for(cfg, 10, d)
    assert np.max(np.abs(e - ref)) < 2e-5


@pytest.mark.parametrize("mode", ["sliding", "block"])
@pytest.mark.parametrize("C,W", [(1, 1), (1, 5), (4, 4), (8, 32), (64, 256), (16, 64)])
def test_mask_ranges_bit_exact(eva, mode, C, W):
    cfg = eva.make_config(1, 1, 1, 16, C, W, mode=mode)
    lo, ns = eva.eva_mask_ranges(cfg, 0, 20000)
    lo, ns = lo.cpu().numpy(), ns.cpu().numpy()
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    for n in list(range(0, 3000)) + list(range(19000, 20000)):
        assert (lo[n], ns[n]) == oracle.mask(n, C, W, m)


# ----------------------------------------------------------------------------- summaries
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d", [16, 32, 64, 128])
@pytest.mark.parametrize("philox", [False, True])
def test_summarize_parity(eva, dtype, d, philox):
    B, H, T, C = 1, 3, 200, 16
    cfg = eva.make_config(B, H, T, d, C, 32, dtype=dtype, seed=99)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=1, device="cuda")
    nC = T // C
    eps = None if philox else eva_inputs.eps(0, B * H, nC, d, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V, eps=eps)
    E = oracle_eps_for(cfg, nC, d) if philox else f64(eps)
    rk, rv = oracle.summarize_batch(f64(K), f64(V), E, C)
    assert np.max(np.abs(f64(ks) - rk)) <= TOL[dtype]
    assert np.max(np.abs(f64(vs) - rv)) <= TOL[dtype]


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("C", [16, 32, 64, 128])
@pytest.mark.parametrize("philox", [False, True])
def test_summarize_bulk_parity(eva, d, C, philox):
    """The bf16 persistent bulk-copy summariser (d in {64, 128}, C in {16..128}): many chunks
    per CTA (more chunks than resident CTAs), a ragged tail (T % C != 0), a chunk range (c0)."""
    B, H, T = 2, 37, 40 * C + C // 2
    cfg = eva.make_config(B, H, T, d, C, 2 * C, seed=5)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=17, device="cuda")
    nC = T // C
    eps = None if philox else eva_inputs.eps(0, B * H, nC, d, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V, eps=eps)
    E = oracle_eps_for(cfg, nC, d) if philox else f64(eps)
    rk, rv = oracle.summarize_batch(f64(K), f64(V), E, C)
    assert np.max(np.abs(f64(ks) - rk)) <= 2e-2
    assert np.max(np.abs(f64(vs) - rv)) <= 2e-2
    # the same rows as a range starting at absolute chunk 7 (its draws)
    ks2, vs2 = eva.eva_summarize_range(cfg, 7, K, V)
    E2 = np.stack([oracle.eps(cfg.seed, cfg.layer, u, 7 + nC, d)[7:] for u in range(B * H)])
    rk2, rv2 = oracle.summarize_batch(f64(K), f64(V), E2, C)
    assert np.max(np.abs(f64(ks2) - rk2)) <= 2e-2 and np.max(np.abs(f64(vs2) - rv2)) <= 2e-2


def test_summarize_singleton_and_constant_chunks(eva):
    """C = 1 -> (k~, beta) = (k, v) exactly; a constant chunk -> its own (k, v)."""
    Q, K, V = eva_inputs.qkv(0, 2, 64, 64, torch.float32, seed=4, device="cuda")
    cfg = eva.make_config(1, 2, 64, 64, 1, 4, dtype=torch.float32)
    ks, vs = eva.eva_summarize(cfg, K, V)
    assert torch.equal(ks, K) and torch.max((vs - V).abs()).item() < 1e-6
    Kc = K[:, :1].expand(2, 64, 64).contiguous()
    Vc = V[:, :1].expand(2, 64, 64).contiguous()
    cfg = eva.make_config(1, 2, 64, 64, 16, 32, dtype=torch.float32)
    ks, vs = eva.eva_summarize(cfg, Kc, Vc)
    assert torch.max((ks - Kc[:, :4]).abs()).item() < 1e-6
    assert torch.max((vs - Vc[:, :4]).abs()).item() < 1e-5


# ----------------------------------------------------------------------------- prefill
CASES = [  # (B, H, T, d, C, W)
    (1, 1, 256, 16, 16, 32),      # configs[0]
    (1, 2, 300, 32, 8, 24),       # ragged T, W = 3C
    (2, 1, 515, 64, 64, 128),     # configs[1] shape family, ragged tail
    (1, 2, 700, 128, 64, 256),    # configs[2] shape family
    (1, 1, 130, 64, 16, 16),      # W = C: a tile consumes summaries of its own rows
    (1, 1, 40, 64, 64, 128),      # T < C: no summaries at all
    (1, 1, 1, 128, 4, 8),         # T = 1
    (1, 1, 96, 64, 1, 3),         # C = 1: exact causal softmax
    (2, 3, 1100, 64, 32, 96),     # several pair items per unit, Q tile 1 partly past T
    (1, 3, 300, 128, 16, 32),     # last pair: Q tile 1 = rows 256..299
]


def fused_applies(d, C, mode="sliding"):
    """EVA_SUMMARIES_FUSED envelope (include/eva.h): d in {64, 128}, causal, C in {16, 32, 64}."""
    return d in (64, 128) and mode != "noncausal" and C in (16, 32, 64)


@pytest.mark.parametrize("mode", ["sliding", "block"])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dtype,kernel", [(torch.float32, "simt"), (torch.bfloat16, "simt"),
                                          (torch.bfloat16, "separate"), (torch.bfloat16, "fused"),
                                          (torch.bfloat16, None)])
@pytest.mark.parametrize("caller_eps", [False, True])
def test_prefill_parity(eva, case, mode, dtype, kernel, caller_eps):
    B, H, T, d, C, W = case
    if kernel in ("separate", "fused") and d not in (64, 128):
        pytest.skip("tensor-core kernels cover d in {64, 128}; other d run the SIMT kernel")
    if kernel == "fused" and not fused_applies(d, C, mode):
        pytest.skip("outside the in-kernel summaries' envelope (test_fused_flag_rejected_outside_envelope)")
    if caller_eps and kernel not in ("fused", "simt"):
        pytest.skip("caller eps: covered on the fused and SIMT paths")
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode, dtype=dtype, seed=7)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=2, device="cuda")
    nC = T // C
    eps = eva_inputs.eps(0, B * H, nC, d, device="cuda") if caller_eps and nC else None
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, kernel=kernel, eps=eps)
    torch.cuda.synchronize()
    E = f64(eps) if eps is not None else oracle_eps_for(cfg, nC, d)
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    rk, rv, rO, rl = run_oracle(Q, K, V, E, C, W, m, cfg.scale)
    tol = TOL[dtype]
    if nC:
        assert np.max(np.abs(f64(ks) - rk)) <= tol
        assert np.max(np.abs(f64(vs) - rv)) <= tol
    err = np.max(np.abs(f64(O) - rO))
    assert err <= tol, err
    assert np.max(np.abs(f64(lse) - rl)) <= tol


@pytest.mark.parametrize("dtype,simt", [(torch.float32, True), (torch.bfloat16, False)])
def test_prefill_window_covers_sequence_is_softmax(eva, dtype, simt):
    """W >= T reduces to exact causal softmax: compare with torch SDPA in fp64."""
    T, d = 256, 64
    cfg = eva.make_config(1, 2, T, d, 64, 256, dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, 2, T, d, dtype, seed=3, device="cuda")
    O, _, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, simt=simt)
    ref = torch.nn.functional.scaled_dot_product_attention(
        Q.double(), K.double(), V.double(), is_causal=True, scale=cfg.scale)
    assert (O.double() - ref).abs().max().item() <= TOL[dtype]


@pytest.mark.parametrize("dtype,simt,kernel", [(torch.float32, True, None), (torch.bfloat16, False, None)])
def test_prefill_summaries_provided_and_poison(eva, dtype, simt, kernel):
    """Everything a query block must not see is poisoned with large finite values;
    its outputs must not move (bit-exact).  Uses EVA_SUMMARIES_PROVIDED."""
    T, d, C, W = 1024, 64, 64, 128
    cfg = eva.make_config(1, 1, T, d, C, W, dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, 1, T, d, dtype, seed=5, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, simt=simt,
                                        kernel=kernel)
    n0, n1 = 512, 639  # one 128-query block
    lo0, _ = oracle.mask(n0, C, W, 0)
    _, ns1 = oracle.mask(n1, C, W, 0)
    K2, V2, ks2, vs2 = K.clone(), V.clone(), ks.clone(), vs.clone()
    K2[:, :lo0] = 3e4
    V2[:, :lo0] = -3e4
    K2[:, n1 + 1:] = 3e4
    V2[:, n1 + 1:] = 3e4
    ks2[:, ns1:] = 3e4
    vs2[:, ns1:] = -3e4
    O2, lse2, _, _ = eva.eva_attn_prefill(cfg, Q, K2, V2, Ksum=ks2, Vsum=vs2, summaries_provided=True,
                                          simt=simt, kernel=kernel)
    assert torch.equal(O2[:, n0:n1 + 1], O[:, n0:n1 + 1])
    assert torch.equal(lse2[:, n0:n1 + 1], lse[:, n0:n1 + 1])


@pytest.mark.parametrize("mode", ["sliding", "block"])
@pytest.mark.parametrize("dtype,simt", [(torch.float32, True), (torch.bfloat16, False)])
def test_prefill_position_probe(eva, mode, dtype, simt):
    """q = k = 0: every logit is 0, xi = 1, k~ = 0, beta = chunk mean of v.  With
    v_m = (1, (m mod 64)/8) (exact in bf16) each output is the mean over exactly the
    visible set; an off-by-one in any range moves it by >= 1/8/64 > tolerance... x8."""
    T, d, C, W = 640, 64, 16, 64
    cfg = eva.make_config(1, 1, T, d, C, W, mode=mode, dtype=dtype)
    Q = torch.zeros(1, T, d, dtype=dtype, device="cuda")
    K = torch.zeros_like(Q)
    V = torch.zeros_like(Q)
    V[0, :, 0] = 1.0
    V[0, :, 1] = (torch.arange(T, device="cuda", dtype=torch.float32) % 64).to(dtype) / 8.0
    O, _, _, vs = eva.eva_attn_prefill(cfg, Q, K, V, simt=simt)
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    Of = O.float().cpu().numpy()[0]
    for n in range(T):
        lo, ns = oracle.mask(n, C, W, m)
        vals = [((c * C) % 64 + (C - 1) / 2) / 8.0 for c in range(ns)] + \
            [(x % 64) / 8.0 for x in range(lo, n + 1)]
        assert abs(Of[n, 0] - 1.0) < 1e-2
        assert abs(Of[n, 1] - np.mean(vals)) <= 2e-2 * max(1.0, abs(np.mean(vals)) / 8), n


def test_prefill_detects_beta_perturbation(eva):
    """SPEC fault injection: a 1e-3 perturbation of one beta must fail the
    suite: the Vsum gate (1e-4) trips, and exactly the rows that see that summary move."""
    T, d, C, W = 512, 32, 16, 32
    cfg = eva.make_config(1, 1, T, d, C, W, dtype=torch.float32)
    Q, K, V = eva_inputs.qkv(0, 1, T, d, torch.float32, seed=6, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    O0, _, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, simt=True)
    E = oracle_eps_for(cfg, T // C, d)
    rk, rv = oracle.summarize_batch(f64(K), f64(V), E, C)
    assert np.max(np.abs(f64(vs) - rv)) <= 1e-4
    vs[0, 3] += 1e-3
    assert np.max(np.abs(f64(vs) - rv)) > 1e-4  # the parity gate on Vsum now fails
    O1, _, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, simt=True)
    moved = (O1 != O0).any(dim=-1)[0].cpu().numpy()
    sees = np.array([oracle.mask(n, C, W, 0)[1] > 3 for n in range(T)])
    assert np.array_equal(moved, sees)


@pytest.mark.parametrize("dtype,simt,kernel", [(torch.float32, True, None), (torch.bfloat16, False, "separate"),
                                               (torch.bfloat16, False, "fused")])
def test_sharded_equals_unsharded(eva, dtype, simt, kernel):
    """(b,h) shards computed separately are bitwise equal to the full run (RNG keyed by global unit)."""
    B, H, T, d, C, W = 2, 3, 384, 64, 32, 64
    cfg = eva.make_config(B, H, T, d, C, W, dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=8, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, simt=simt, kernel=kernel)
    for b0, cnt in ((0, 2), (2, 3), (5, 1)):
        c2 = eva.make_config(B, H, T, d, C, W, dtype=dtype, bh_begin=b0, bh_count=cnt)
        q, k, v = eva_inputs.qkv(b0, cnt, T, d, dtype, seed=8, device="cuda")
        O2, lse2, ks2, vs2 = eva.eva_attn_prefill(c2, q, k, v, simt=simt, kernel=kernel)
        assert torch.equal(O2, O[b0:b0 + cnt]) and torch.equal(lse2, lse[b0:b0 + cnt])
        assert torch.equal(ks2, ks[b0:b0 + cnt]) and torch.equal(vs2, vs[b0:b0 + cnt])


@pytest.mark.parametrize("dtype,kernel,n_slices", [(torch.bfloat16, None, 1), (torch.bfloat16, None, 4),
                                                    (torch.bfloat16, None, 7), (torch.float32, "simt", 3)])
def test_prefill_host_pipeline_equals_device_call(eva, dtype, kernel, n_slices):
    """eva_attn_prefill_host (H2D / kernels / D2H pipelined over unit slices) is bitwise
    equal to one eva_attn_prefill over all units, and leaves the device copies in place."""
    B, H, T, d, C, W = 2, 3, 320, 64, 32, 64
    cfg = eva.make_config(B, H, T, d, C, W, bh_begin=0, dtype=dtype)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, dtype, seed=12, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, simt=kernel == "simt")
    hQ, hK, hV = (x.cpu().pin_memory() for x in (Q, K, V))
    hO = torch.full((B * H, T, d), float("nan"), dtype=dtype).pin_memory()
    hl = torch.full((B * H, T), float("nan")).pin_memory()
    hp = eva.HostPrefill(cfg, max_slices=8, device="cuda", want_lse=True)
    hp(hQ, hK, hV, hO, hlse=hl, n_slices=n_slices, kernel=kernel)
    torch.cuda.synchronize()
    assert torch.equal(hO, O.cpu()) and torch.equal(hl, lse.cpu())
    assert torch.equal(hp.Ksum, ks) and torch.equal(hp.Vsum, vs) and torch.equal(hp.K, K)
    with pytest.raises(eva.EvaError, match="INVALID_ARG"):
        hp(hQ, hK, hV, hO, n_slices=9)


@pytest.mark.parametrize("d", [64, 128])
def test_prefill_overlap_flag_equals_plain_call(eva, d):
    """EVA_PREFILL_OVERLAP (prefill launched right after the eva_summarize producing its
    summaries, local tiles started before that kernel completes): deterministic (the same bits
    eagerly, repeatedly and inside a CUDA graph) and equal to the plain call up to the tile
    order (the plain call walks the summary tiles first)."""
    B, H, T, C, W = 2, 4, 1536, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=14, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    O, lse, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True)
    ks2, vs2 = torch.zeros_like(ks), torch.zeros_like(vs)
    O2, lse2 = torch.zeros_like(O), torch.zeros_like(lse)
    ref = None
    for _ in range(3):
        ks2.zero_(); vs2.zero_()
        eva.eva_summarize(cfg, K, V, Ksum=ks2, Vsum=vs2)
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks2, Vsum=vs2, summaries_provided=True, O=O2, lse=lse2,
                             overlap=True)
        torch.cuda.synchronize()
        if ref is None:
            ref = (O2.clone(), lse2.clone())
            assert (O2.float() - O.float()).abs().max().item() <= 2e-2
            assert (lse2 - lse).abs().max().item() <= 1e-3
        assert torch.equal(O2, ref[0]) and torch.equal(lse2, ref[1])
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g):
            eva.eva_summarize(cfg, K, V, Ksum=ks2, Vsum=vs2)
            eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks2, Vsum=vs2, summaries_provided=True, O=O2,
                                 lse=lse2, overlap=True)
    for _ in range(3):
        ks2.zero_(); vs2.zero_(); O2.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(O2, ref[0]) and torch.equal(lse2, ref[1])


def test_errors_are_reported_not_silent(eva):
    cfg = eva.make_config(1, 1, 64, 64, 16, 40)  # W % C != 0
    Q = torch.zeros(1, 64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(eva.EvaError, match="INVALID_ARG"):
        eva.eva_attn_prefill(cfg, Q, Q, Q)
    cfg = eva.make_config(1, 1, 64, 64, 16, 32, samples=4)
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):
        eva.eva_attn_prefill(cfg, Q, Q, Q)


# ----------------------------------------------------------------------------- decode
@pytest.mark.parametrize("mode", ["sliding", "block"])
@pytest.mark.parametrize("dtype,d,C,W", [(torch.float32, 32, 8, 24), (torch.bfloat16, 128, 16, 64),
                                         (torch.bfloat16, 64, 4, 4), (torch.float32, 16, 1, 3)])
def test_decode_streaming_parity(eva, mode, dtype, d, C, W):
    """Token-by-token append + decode == oracle streaming cache at every step."""
    BH, T = 3, 150
    cfg = eva.make_config(1, BH, 0, d, C, W, mode=mode, dtype=dtype, seed=11)
    cap = T // C
    cache = eva.DecodeCache(cfg, cap, device="cuda")
    q, k, v = eva_inputs.decode_tokens(0, BH, T, d, dtype, seed=12, device="cuda")
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    orc = [oracle.Cache(d, C, W, m, cap=cap, scale=cfg.scale) for _ in range(BH)]
    E = oracle_eps_for(cfg, cap + 1, d)
    worst = 0.0
    for t in range(T):
        cache.eva_cache_append(k[t], v[t])
        o, lse = cache.eva_attn_decode(q[t])
        of, lf = f64(o), f64(lse)
        for u in range(BH):
            assert orc[u].append(f64(k[t, u]), f64(v[t, u]), E[u, t // C]) == 0
            ro, rl = orc[u].decode(f64(q[t, u]))
            worst = max(worst, np.max(np.abs(of[u] - ro)), abs(lf[u] - rl))
    assert worst <= TOL[dtype], worst
    # the cache's summaries equal the oracle's
    rks, rvs = orc[1].summaries()
    n = cache.pos // C
    assert np.max(np.abs(f64(cache.sum_k[1, :n]) - rks)) <= TOL[dtype]
    assert np.max(np.abs(f64(cache.sum_v[1, :n]) - rvs)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_prefill_handoff_then_decode(eva, dtype):
    """append(n_new = T) after a prompt, then token-by-token: each decoded row equals
    the prefill row of the extended sequence."""
    BH, T0, G, d, C, W = 2, 1000, 70, 64, 64, 128
    T = T0 + G
    cfg = eva.make_config(1, BH, T, d, C, W, dtype=dtype, seed=21)
    Q, K, V = eva_inputs.qkv(0, BH, T, d, dtype, seed=22, device="cuda")
    O_full, lse_full, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, simt=True)
    cache = eva.DecodeCache(cfg, T // C + 1, device="cuda")
    cache.eva_cache_append(K[:, :T0].contiguous(), V[:, :T0].contiguous())
    o, lse = cache.eva_attn_decode(Q[:, T0 - 1].contiguous())
    outs = [o]
    for t in range(T0, T):
        cache.eva_cache_append(K[:, t].contiguous(), V[:, t].contiguous())
        o, lse = cache.eva_attn_decode(Q[:, t].contiguous())
        outs.append(o)
    dec = torch.stack(outs, 1)
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    assert (dec.float() - O_full[:, T0 - 1:].float()).abs().max().item() <= tol


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_cache_load_equals_append(eva, dtype):
    """eva_cache_load with the prefill's summaries == eva_cache_append(n_new = T): same ring,
    same summaries (bitwise), and the decode continues identically."""
    BH, T, d, C, W = 3, 777, 64, 32, 96
    cfg = eva.make_config(1, BH, T, d, C, W, dtype=dtype, seed=31)
    Q, K, V = eva_inputs.qkv(0, BH, T, d, dtype, seed=32, device="cuda")
    _, _, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, simt=True)
    a = eva.DecodeCache(cfg, T // C + 4, device="cuda")
    b = eva.DecodeCache(cfg, T // C + 4, device="cuda")
    a.eva_cache_append(K, V)
    b.eva_cache_load(K, V, ks, vs)
    assert a.pos == b.pos == T
    assert torch.equal(a.ring_k, b.ring_k) and torch.equal(a.ring_v, b.ring_v)
    nC = T // C
    assert torch.equal(a.sum_k[:, :nC], b.sum_k[:, :nC]) and torch.equal(a.sum_v[:, :nC], b.sum_v[:, :nC])
    q, k, v = eva_inputs.decode_tokens(0, BH, 80, d, dtype, seed=33, device="cuda")
    for t in range(80):
        a.eva_cache_append(k[t], v[t])
        b.eva_cache_append(k[t], v[t])
        oa, la = a.eva_attn_decode(q[t])
        ob, lb = b.eva_attn_decode(q[t])
        assert torch.equal(oa, ob) and torch.equal(la, lb)


@pytest.mark.parametrize("BH,ctx", [(1, 5000), (2, 20000), (64, 3000)])
def test_decode_split_k_parity(eva, BH, ctx):
    """Long compressed contexts at small batch use split-K with the in-kernel last-CTA merge;
    the cache (filled through eva_cache_load) decodes like the oracle row."""
    d, C, W = 128, 64, 256
    T = ctx
    cfg = eva.make_config(1, BH, T, d, C, W, dtype=torch.bfloat16, seed=41)
    Q, K, V = eva_inputs.qkv(0, BH, T, d, torch.bfloat16, seed=42, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    cache = eva.DecodeCache(cfg, T // C + 2, device="cuda")
    cache.eva_cache_load(K[:, :T - 1].contiguous(), V[:, :T - 1].contiguous(), ks[:, :(T - 1) // C].contiguous(),
                         vs[:, :(T - 1) // C].contiguous())
    cache.eva_cache_append(K[:, T - 1].contiguous(), V[:, T - 1].contiguous())
    assert cache.workspace_bytes() > 0 or BH * 8 >= 148 * 8
    for rep in range(2):  # the merge counters must be left at zero
        o, lse = cache.eva_attn_decode(Q[:, T - 1].contiguous())
        for u in range(BH):
            E = oracle.eps(cfg.seed, cfg.layer, u, T // C, d)
            rk, rv = oracle.summarize(f64(K[u]), f64(V[u]), E, C)
            _, rO, rl = oracle.prefill_rows(f64(Q[u]), f64(K[u]), f64(V[u]), rk, rv, [T - 1], C, W, 0, cfg.scale)
            assert np.max(np.abs(f64(o[u]) - rO[0])) <= 2e-2
            assert abs(float(lse[u]) - rl[0]) <= 2e-2


@pytest.mark.parametrize("dtype,d,C,W,mode", [(torch.bfloat16, 128, 16, 64, "sliding"),
                                              (torch.float32, 64, 8, 8, "block"),
                                              (torch.bfloat16, 64, 64, 128, "sliding")])
def test_fused_decode_step_equals_append_then_decode(eva, dtype, d, C, W, mode):
    """eva_decode_step == eva_cache_append(1) + eva_attn_decode, bit for bit (outputs and cache),
    across chunk completions, with in-kernel Philox and with caller eps."""
    T0, G = 300, 150
    for use_eps, BH in ((False, 5), (True, 5), (False, 1030)):  # 1030 units: two-launch path
        cfg = eva.make_config(1, BH, 0, d, C, W, mode=mode, dtype=dtype, seed=51)
        cap = (T0 + G) // C + 1
        a = eva.DecodeCache(cfg, cap, device="cuda")
        b = eva.DecodeCache(cfg, cap, device="cuda")
        eps = eva_inputs.eps(0, BH, cap, d, device="cuda") if use_eps else None
        q, k, v = eva_inputs.decode_tokens(0, BH, T0 + G, d, dtype, seed=52, device="cuda")
        a.eva_cache_append(k[:T0].transpose(0, 1).contiguous(), v[:T0].transpose(0, 1).contiguous(), eps)
        b.eva_cache_append(k[:T0].transpose(0, 1).contiguous(), v[:T0].transpose(0, 1).contiguous(), eps)
        for t in range(T0, T0 + G):
            a.eva_cache_append(k[t], v[t], eps)
            oa, la = a.eva_attn_decode(q[t])
            ob, lb = b.eva_decode_step(q[t], k[t], v[t], eps)
            assert torch.equal(oa, ob) and torch.equal(la, lb), t
        assert a.pos == b.pos
        assert torch.equal(a.ring_k, b.ring_k) and torch.equal(a.ring_v, b.ring_v)
        assert torch.equal(a.sum_k, b.sum_k) and torch.equal(a.sum_v, b.sum_v)


def test_decode_poisoned_stale_ring_slots(eva):
    """Stale / invisible ring slots and unused summary rows are poisoned; output unchanged."""
    BH, d, C, W, T = 2, 64, 16, 64, 300
    cfg = eva.make_config(1, BH, 0, d, C, W, dtype=torch.bfloat16)
    cache = eva.DecodeCache(cfg, 32, device="cuda")
    q, k, v = eva_inputs.decode_tokens(0, BH, T, d, torch.bfloat16, seed=13, device="cuda")
    for t in range(T):
        cache.eva_cache_append(k[t], v[t])
    o, lse = cache.eva_attn_decode(q[T - 1])
    n = T - 1
    lo, ns = oracle.mask(n, C, W, 0)
    for p in range(n - W + 1, lo):  # still in the ring but not visible
        cache.ring_k[:, p % W] = 3e4
        cache.ring_v[:, p % W] = 3e4
    cache.sum_k[:, ns:] = 3e4
    cache.sum_v[:, ns:] = -3e4
    o2, lse2 = cache.eva_attn_decode(q[T - 1])
    assert torch.equal(o, o2) and torch.equal(lse, lse2)


def test_decode_capacity_error(eva):
    cfg = eva.make_config(1, 1, 0, 64, 16, 32)
    cache = eva.DecodeCache(cfg, 1, device="cuda")
    x = torch.zeros(1, 31, 64, dtype=torch.bfloat16, device="cuda")
    cache.eva_cache_append(x, x)
    with pytest.raises(eva.EvaError, match="CAPACITY"):
        cache.eva_cache_append(x[:, :1], x[:, :1])


# ----------------------------------------------------------------------------- full-size sampled parity
@pytest.mark.parametrize("kernel", ["fused", "separate"])
@pytest.mark.parametrize("B,H,T,d,C,W", [(1, 16, 2048, 64, 64, 128), (1, 4, 8192, 128, 64, 256),
                                         (8, 32, 8192, 128, 64, 256)])
def test_full_size_sampled_parity(eva, B, H, T, d, C, W, kernel):
    """BASELINE configs[1] (full) and configs[2] (4 of its 256 units, same kernel launch
    shape per unit) on the bf16 tensor-core path; oracle on sampled rows."""
    cfg = eva.make_config(B, H, T, d, C, W, dtype=torch.bfloat16)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, kernel=kernel)
    nC = T // C
    rng = np.random.default_rng(1)
    for u in sorted({0, B * H // 2 + 1, B * H - 1}):
        E = oracle.eps(cfg.seed, cfg.layer, u, nC, d)
        rk, rv = oracle.summarize(f64(K[u]), f64(V[u]), E, C)
        assert np.max(np.abs(f64(ks[u]) - rk)) <= 2e-2
        assert np.max(np.abs(f64(vs[u]) - rv)) <= 2e-2
        rows = np.unique(np.concatenate([rng.integers(0, T, 200), [0, 1, C - 1, C, W - 1, W, T - 1]]))
        rows, rO, rl = oracle.prefill_rows(f64(Q[u]), f64(K[u]), f64(V[u]), rk, rv, rows, C, W, 0,
                                           cfg.scale)
        assert np.max(np.abs(f64(O[u])[rows] - rO)) <= 2e-2
        assert np.max(np.abs(f64(lse[u])[rows] - rl)) <= 2e-2


# ----------------------------------------------------------------------------- configs[4] sweep shapes
@pytest.mark.parametrize("T,C,W", [(4096, 32, 128), (16384, 32, 512), (32768, 128, 128), (65536, 64, 512),
                                   (131072, 128, 512)])
def test_long_context_sweep_sampled_parity(eva, T, C, W):
    """BASELINE configs[4] shapes (H=32, d=128 per unit; 2 units run, same launch shape per
    unit): summaries of sampled chunks and outputs of sampled rows vs the oracle."""
    d, units = 128, 2
    cfg = eva.make_config(1, units, T, d, C, W, dtype=torch.bfloat16, seed=5)
    Q, K, V = eva_inputs.qkv(0, units, T, d, torch.bfloat16, seed=9, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    nC = T // C
    rng = np.random.default_rng(T + C + W)
    for u in range(units):
        E = oracle.eps(cfg.seed, cfg.layer, u, nC, d)
        Kf, Vf = f64(K[u]), f64(V[u])
        rk, rv = oracle.summarize(Kf, Vf, E, C)
        assert np.max(np.abs(f64(ks[u]) - rk)) <= 2e-2
        assert np.max(np.abs(f64(vs[u]) - rv)) <= 2e-2
        rows = np.unique(np.concatenate([rng.integers(0, T, 48), [0, W - 1, W, T // 2, T - 1]]))
        rows, rO, rl = oracle.prefill_rows(f64(Q[u]), Kf, Vf, rk, rv, rows, C, W, 0, cfg.scale)
        assert np.max(np.abs(f64(O[u])[rows] - rO)) <= 2e-2
        assert np.max(np.abs(f64(lse[u])[rows] - rl)) <= 2e-2


# ----------------------------------------------------------------------------- fused summaries
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("mode", ["sliding", "block"])
def test_fused_equals_separate(eva, d, mode):
    """EVA_SUMMARIES_FUSED vs EVA_SUMMARIES_SEPARATE on the same inputs: the summaries agree to
    one bf16 rounding step (fp32 summation order differs), and the attention of the fused call
    equals the separate kernel run on the fused call's own summaries up to the tile walk order."""
    B, H, T, C, W = 3, 7, 1000, 32, 128
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=31, device="cuda")
    O1, l1, ks1, vs1 = eva.eva_attn_prefill(cfg, Q, K, V, kernel="fused")
    O2, l2, ks2, vs2 = eva.eva_attn_prefill(cfg, Q, K, V, kernel="separate")
    O3, l3, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks1, Vsum=vs1, summaries_provided=True)
    torch.cuda.synchronize()
    # one bf16 rounding step of the value, plus fp32 summation-order noise near zero
    ulp = lambda x: x.float().abs() * 2.0 ** -7 + 1e-5
    assert bool(((ks1.float() - ks2.float()).abs() <= ulp(ks2)).all())
    assert bool(((vs1.float() - vs2.float()).abs() <= ulp(vs2)).all())
    # the same math in another tile order: within two bf16 rounding steps of the output
    assert bool(((O1.float() - O3.float()).abs() <= 2.0 ** -6 * O3.float().abs().clamp_min(1.0)).all())
    assert (l1 - l3).abs().max().item() <= 1e-3


def test_fused_deterministic_across_launches_shapes_and_graphs(eva):
    """The fused launch's workspace (ticket, done counter, epoch, ready flags) is reused across
    launches of different shapes and inside a CUDA graph: the results stay bitwise identical
    (no stale flag is ever taken for a fresh one, the counters are left consistent)."""
    shapes = [(1, 16, 2048, 64, 64, 128), (2, 5, 777, 128, 16, 64), (1, 16, 2048, 64, 64, 128),
              (4, 3, 300, 64, 16, 16), (2, 5, 777, 128, 16, 64)]
    first = {}
    for rep in range(2):
        for sh in shapes:
            B, H, T, d, C, W = sh
            cfg = eva.make_config(B, H, T, d, C, W)
            Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=sum(sh), device="cuda")
            out = eva.eva_attn_prefill(cfg, Q, K, V, kernel="fused")
            torch.cuda.synchronize()
            if sh not in first:
                first[sh] = [t.clone() for t in out]
            for a, b in zip(out, first[sh]):
                assert torch.equal(a, b), sh
    B, H, T, d, C, W = shapes[1]
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=sum(shapes[1]), device="cuda")
    O, lse = torch.zeros_like(Q), torch.zeros(B * H, T, device="cuda")
    ks = torch.zeros(B * H, T // C, d, dtype=torch.bfloat16, device="cuda")
    vs = torch.zeros_like(ks)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        eva.eva_prefill_reserve(cfg)  # on the capture stream: torch.cuda.graph(stream=s) below
        with torch.cuda.graph(g, stream=s):
            eva.eva_attn_prefill(cfg, Q, K, V, kernel="fused", O=O, lse=lse, Ksum=ks, Vsum=vs)
    for _ in range(5):
        O.zero_(); ks.zero_(); vs.zero_()
        g.replay()
        torch.cuda.synchronize()
        ref = first[shapes[1]]
        assert torch.equal(O, ref[0]) and torch.equal(lse, ref[1])
        assert torch.equal(ks, ref[2]) and torch.equal(vs, ref[3])


def test_fused_flag_rejected_outside_envelope(eva):
    """EVA_SUMMARIES_FUSED where it does not apply is an error, not a silent fallback; flags 0
    there runs the separate launches and matches the oracle (test_prefill_parity)."""
    Q = torch.zeros(2, 256, 64, dtype=torch.bfloat16, device="cuda")
    for kw in (dict(chunk=128, window=256), dict(chunk=8, window=16), dict(chunk=16, window=32, mode="noncausal")):
        cfg = eva.make_config(1, 2, 256, 64, kw["chunk"], kw["window"], mode=kw.get("mode", "sliding"))
        with pytest.raises(eva.EvaError, match="UNSUPPORTED"):
            eva.eva_attn_prefill(cfg, Q, Q, Q, kernel="fused")
    cfg = eva.make_config(1, 2, 256, 64, 16, 32, dtype=torch.float32)
    with pytest.raises(eva.EvaError, match="UNSUPPORTED"):
        eva.eva_attn_prefill(cfg, Q.float(), Q.float(), Q.float(), kernel="fused")


def test_fused_many_waves_sampled_parity(eva):
    """Many more query tiles than resident CTAs (ticket order, flags awaited across waves), a
    ragged tail and W = C (a tile reads the summaries of its own rows): oracle on sampled units."""
    B, H, T, d, C, W = 4, 64, 1100, 64, 16, 16
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=77, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, kernel="fused")
    nC = T // C
    for u in (0, 101, B * H - 1):
        E = oracle.eps(cfg.seed, cfg.layer, u, nC, d)
        rk, rv = oracle.summarize(f64(K[u]), f64(V[u]), E, C)
        assert np.max(np.abs(f64(ks[u]) - rk)) <= 2e-2
        assert np.max(np.abs(f64(vs[u]) - rv)) <= 2e-2
        rows = np.arange(T)
        rows, rO, rl = oracle.prefill_rows(f64(Q[u]), f64(K[u]), f64(V[u]), rk, rv, rows, C, W, 0, cfg.scale)
        assert np.max(np.abs(f64(O[u])[rows] - rO)) <= 2e-2
        assert np.max(np.abs(f64(lse[u])[rows] - rl)) <= 2e-2


def test_cache_load_with_summaries_in_place(eva):
    """The summaries written straight into the decode cache (eva_summarize on cache.sum_k /
    sum_v, cap_chunks == nC) and eva_cache_load copying only the ring: the same cache as the
    copying hand-off, and the same decode."""
    BH, T, d, C, W = 4, 1024, 128, 64, 256
    dtype = torch.bfloat16
    cfg = eva.make_config(1, BH, T, d, C, W, dtype=dtype, seed=51)
    Q, K, V = eva_inputs.qkv(0, BH, T, d, dtype, seed=52, device="cuda")
    nC = T // C
    a = eva.DecodeCache(cfg, nC, device="cuda")
    b = eva.DecodeCache(cfg, nC, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    a.eva_cache_load(K, V, ks, vs)
    eva.eva_summarize(cfg, K, V, Ksum=b.sum_k, Vsum=b.sum_v)   # in place
    b.eva_cache_load(K, V, b.sum_k, b.sum_v)                   # ring only
    torch.cuda.synchronize()
    assert a.pos == b.pos == T
    for x, y in ((a.ring_k, b.ring_k), (a.ring_v, b.ring_v), (a.sum_k, b.sum_k), (a.sum_v, b.sum_v)):
        assert torch.equal(x, y)
    q, k, v = eva_inputs.decode_tokens(0, BH, 8, d, dtype, seed=53, device="cuda")
    for t in range(8):
        oa, la = a.eva_decode_step(q[t], k[t], v[t])
        ob, lb = b.eva_decode_step(q[t], k[t], v[t])
        assert torch.equal(oa, ob) and torch.equal(la, lb)
    # aliasing only one of the two, or with a cache larger than nC, is rejected
    c = eva.DecodeCache(cfg, nC, device="cuda")
    with pytest.raises(eva.EvaError, match="INVALID_ARG"):
        c.eva_cache_load(K, V, c.sum_k, vs)
    from paper_2511_00576_b200 import _native as N
    import ctypes
    e = eva.DecodeCache(cfg, nC + 2, device="cuda")
    st = N.lib.eva_cache_load(ctypes.byref(e.c), K.data_ptr(), V.data_ptr(), e.sum_k.data_ptr(), e.sum_v.data_ptr(),
                              T, None)
    assert st == N.EVA_ERR_INVALID_ARG and b"cap_chunks" in N.lib.eva_last_error()
