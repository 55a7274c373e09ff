"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Each pin is chosen so that a plausible mistake in the oracle (a dropped term,
wrong sign or index, transposed operand, missing clip or lambda, off-by-one
in the window) fails at least one of them.  None of these tests touches the
CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from bruteforce import eva_direct, exact_causal_softmax, partition_sets, summary_direct

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------- Philox
def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox_kat.json)."""
    for v in _gold("philox_kat.json")["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert oracle.philox4x32_10(ctr, key) == [int(x, 16) for x in v["out"]]


def test_eps_is_standard_normal():
    """Box-Muller output is N(0,1): moments and a KS test over 2^18 draws."""
    from scipy import stats
    e = np.concatenate([oracle.eps(1234, 0, bh, 256, 128).ravel() for bh in range(8)])
    assert abs(e.mean()) < 4 / math.sqrt(e.size)
    assert abs(e.var() - 1.0) < 0.01
    assert stats.kstest(e, "norm").pvalue > 1e-3
    # the four lanes of one Philox block are not correlated with each other
    x = oracle.eps(5, 1, 3, 4096, 4)
    cc = np.corrcoef(x.T)
    assert np.max(np.abs(cc - np.eye(4))) < 0.06


def test_eps_streams_are_distinct_and_deterministic():
    a = oracle.eps(1234, 0, 5, 16, 64)
    assert np.array_equal(a, oracle.eps(1234, 0, 5, 16, 64))
    for other in (oracle.eps(1235, 0, 5, 16, 64), oracle.eps(1234, 1, 5, 16, 64),
                  oracle.eps(1234, 0, 6, 16, 64)):
        assert np.max(np.abs(a - other)) > 0.5
    # a chunk's draw does not depend on how many chunks are drawn (counter-based)
    assert np.array_equal(oracle.eps(1234, 0, 5, 3, 64), a[:3])
    # d not a multiple of 4: leading components agree with the d=8 draw
    assert np.array_equal(oracle.eps(9, 0, 0, 2, 6), oracle.eps(9, 0, 0, 2, 8)[:, :6])


def test_box_muller_lane_mapping():
    """eps[c][4i+j] comes from Philox block (i, c, bh, layer): check via the KAT'd block."""
    seed, layer, bh = 0x1234_5678_9ABC_DEF0, 3, 11
    e = oracle.eps(seed, layer, bh, 3, 8)
    x = oracle.philox4x32_10([1, 2, bh, layer], [seed & 0xFFFFFFFF, seed >> 32])
    u = [((w >> 8) + 0.5) / 2 ** 24 for w in x]
    r = math.sqrt(-2 * math.log(u[0]))
    assert abs(e[2, 4] - r * math.cos(2 * math.pi * u[1])) < 1e-12
    assert abs(e[2, 5] - r * math.sin(2 * math.pi * u[1])) < 1e-12


# --------------------------------------------------------------------------- partition
def test_partition_spec_examples():
    g = _gold("worked_examples.json")
    for key in ("partition_block_n5", "partition_sliding_n11"):
        ex = g[key]
        mode = oracle.SLIDING if ex["mode"] == "sliding" else oracle.BLOCK
        lo, ns = oracle.mask(ex["n"], ex["C"], ex["W"], mode)
        assert list(range(lo, ex["n"] + 1)) == ex["E"]
        assert [list(range(c * ex["C"], (c + 1) * ex["C"])) for c in range(ns)] == ex["chunks"]


@pytest.mark.parametrize("mode", ["sliding", "block"])
def test_partition_exact_cover_vs_set_enumeration(mode):
    """Range form == SPEC set form, and E(n) U chunks = {0..n} disjoint."""
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    for C in (1, 2, 4, 8, 16):
        for R in (1, 2, 3, 4, 8):
            W = R * C
            for n in range(0, 700):
                E, chunks = partition_sets(n, C, W, mode)
                lo, ns = oracle.mask(n, C, W, m)
                assert (lo, ns) == (E[0], len(chunks))
                cover = sorted(E + [x for ch in chunks for x in ch])
                assert cover == list(range(n + 1))
                assert n in E and len(E) <= W


def test_window_size_bounds():
    """Sliding: W-C+1 <= |E(n)| <= W once n >= W-1; block: |E| = n mod W + 1."""
    C, W = 16, 64
    for n in range(W - 1, 2000):
        lo, _ = oracle.mask(n, C, W, oracle.SLIDING)
        assert W - C + 1 <= n - lo + 1 <= W
        lo, _ = oracle.mask(n, C, W, oracle.BLOCK)
        assert n - lo + 1 == n % W + 1


def test_cache_entry_closed_form():
    """W + (T-W)/C entries at the last position (paper setting P:141)."""
    for case in _gold("worked_examples.json")["cache_report"]["cases"]:
        n = case["T"] - 1
        lo, ns = oracle.mask(n, case["C"], case["W"], oracle.SLIDING)
        assert (n - lo + 1) + ns == case["eva"]
        lo, ns = oracle.mask(n, case["C"], case["W"], oracle.BLOCK)
        assert (n - lo + 1) + ns == case["eva"]


# --------------------------------------------------------------------------- summaries
@pytest.mark.parametrize("key", ["summary_d1", "summary_d1_clip_bites", "summary_d1_negative_clip"])
def test_summary_worked_examples(key):
    ex = _gold("worked_examples.json")[key]
    ks, vs, om = oracle.summarize(ex["K"], ex["V"], ex["eps"], ex["C"], ex["lambda"], ex["clip"],
                                  return_omega=True)
    assert np.allclose(ks, ex["k_tilde"], atol=1e-15)
    assert np.allclose(om, ex["omega"], atol=1e-15)
    assert np.allclose(vs, ex["beta"], atol=1e-14)


def test_summary_constant_and_singleton_chunks():
    rng = np.random.default_rng(0)
    d = 16
    k, v = rng.normal(size=d), rng.normal(size=d)
    E = rng.normal(size=(1, d))
    ks, vs = oracle.summarize(np.tile(k, (8, 1)), np.tile(v, (8, 1)), E, 8)
    assert np.allclose(ks[0], k, atol=1e-14) and np.allclose(vs[0], v, atol=1e-14)
    K, V = rng.normal(size=(5, d)), rng.normal(size=(5, d))
    ks, vs = oracle.summarize(K, V, rng.normal(size=(5, d)), 1)
    assert np.array_equal(ks, K) and np.allclose(vs, V, atol=1e-15)


def test_summary_envelope_omega_bound_and_linear_domain():
    """beta inside the chunk's value envelope; |omega| <= lambda;
    log-domain softmax == linear-domain xi ratio at small magnitudes."""
    rng = np.random.default_rng(1)
    for C, d in ((4, 3), (8, 8), (16, 5)):
        T = 3 * C
        K = 0.4 * rng.normal(size=(T, d))
        V = rng.normal(size=(T, d))
        E = rng.normal(size=(T // C, d)) * 3
        ks, vs, om = oracle.summarize(K, V, E, C, return_omega=True)
        assert np.all(np.abs(om) <= 0.1 + 1e-15)
        for c in range(T // C):
            Vc = V[c * C:(c + 1) * C]
            assert np.all(vs[c] <= Vc.max(0) + 1e-12) and np.all(vs[c] >= Vc.min(0) - 1e-12)
            kt, omega, beta = summary_direct(K[c * C:(c + 1) * C], Vc, E[c])
            assert np.allclose(ks[c], kt, atol=1e-14)
            assert np.allclose(om[c], omega, atol=1e-15)
            assert np.allclose(vs[c], beta, atol=1e-12)
    # zero noise and zero mean key -> omega = 0 -> beta = softmax(-|k|^2/2)-weighted values
    K = np.array([[1.0, -1.0], [-1.0, 1.0], [2.0, 0.0], [-2.0, 0.0]])
    V = np.array([[1.0, 0.0], [0.0, 1.0], [5.0, 5.0], [7.0, 7.0]])
    ks, vs, om = oracle.summarize(K, V, np.zeros((1, 2)), 4, return_omega=True)
    assert np.all(om == 0) and np.all(ks == 0)
    w = np.exp(-0.5 * (K ** 2).sum(1))
    assert np.allclose(vs[0], (w[:, None] * V).sum(0) / w.sum(), atol=1e-14)


def test_summary_alternative_omega_reading():
    """omega_mode 1 (reading R3 alternative): omega = k~ + lambda*clip(eps)."""
    ex = _gold("worked_examples.json")["summary_d1_clip_bites"]
    _, _, om = oracle.summarize(ex["K"], ex["V"], ex["eps"], 2, omega_mode=1, return_omega=True)
    assert abs(om[0, 0] - (0.5 + 0.1)) < 1e-15


# --------------------------------------------------------------------------- prefill
def test_prefill_worked_T3():
    ex = _gold("worked_examples.json")["prefill_T3"]
    Q, K, V = (np.array(ex[k]) for k in ("Q", "K", "V"))
    ks, vs = oracle.summarize(K, V, ex["eps"], ex["C"])
    O, _ = oracle.prefill(Q, K, V, ks, vs, ex["C"], ex["W"], oracle.SLIDING, ex["scale"])
    assert np.allclose(O, ex["O"], atol=1e-14)


@pytest.mark.parametrize("mode", [oracle.SLIDING, oracle.BLOCK])
def test_prefill_window_covers_sequence_is_exact_softmax(mode):
    """W >= T: no summaries, Eq.12 == Eq.1 causal: library pin via torch SDPA fp64."""
    rng = np.random.default_rng(2)
    T, d, C = 96, 32, 8
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    scale = 1 / math.sqrt(d)
    ks, vs = oracle.summarize(K, V, rng.normal(size=(T // C, d)), C)
    O, lse = oracle.prefill(Q, K, V, ks, vs, C, 128, mode, scale)
    ref = torch.nn.functional.scaled_dot_product_attention(
        *(torch.from_numpy(x)[None, None] for x in (Q, K, V)), is_causal=True, scale=scale)[0, 0]
    assert np.max(np.abs(O - ref.numpy())) < 1e-12
    logits = scale * Q @ K.T
    logits[np.triu_indices(T, 1)] = -np.inf
    lse_ref = np.log(np.exp(logits - logits.max(1, keepdims=True)).sum(1)) + logits.max(1)
    assert np.max(np.abs(lse - lse_ref)) < 1e-12


@pytest.mark.parametrize("mode", [oracle.SLIDING, oracle.BLOCK])
def test_prefill_chunk1_is_exact_softmax(mode):
    """C = 1: k~ = k, beta = v, Z exact -> exact causal softmax for any W and eps."""
    rng = np.random.default_rng(3)
    T, d = 70, 8
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    ks, vs = oracle.summarize(K, V, 5 * rng.normal(size=(T, d)), 1)
    for W in (1, 3, 16):
        O, _ = oracle.prefill(Q, K, V, ks, vs, 1, W, mode, 0.7)
        assert np.max(np.abs(O - exact_causal_softmax(Q, K, V, 0.7))) < 1e-12


@pytest.mark.parametrize("mode", ["sliding", "block"])
def test_prefill_equals_direct_eq9_bruteforce(mode):
    """Augmented-softmax form (Eq.12-14) == direct Eq.9/10 form, independent code."""
    rng = np.random.default_rng(4)
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    for trial in range(30):
        C = int(rng.choice([1, 2, 3, 4]))
        W = C * int(rng.integers(1, 4))
        T = int(rng.integers(1, 40))
        d = int(rng.integers(1, 7))
        Q, K, V = (0.6 * rng.normal(size=(T, d)) for _ in range(3))
        E = rng.normal(size=(max(T // C, 1), d))
        scale = float(rng.uniform(0.3, 1.5))
        ks, vs = oracle.summarize(K, V, E[: T // C], C)
        O, _ = oracle.prefill(Q, K, V, ks, vs, C, W, m, scale)
        ref = eva_direct(Q, K, V, E, C, W, mode, scale)
        assert np.max(np.abs(O - ref)) < 1e-12, (trial, C, W, T, d)


def test_prefill_row_stochastic_and_mask_fuzz():
    """Weights sum to 1 (V = 1 -> O = 1); rows outside the visible set do not matter."""
    rng = np.random.default_rng(5)
    T, d, C, W = 200, 16, 8, 32
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    ks, vs = oracle.summarize(K, V, rng.normal(size=(T // C, d)), C)
    O1, _ = oracle.prefill(Q, K, np.ones_like(V), ks, np.ones_like(vs), C, W, 0, 0.25)
    assert np.max(np.abs(O1 - 1)) < 1e-13
    O, lse = oracle.prefill(Q, K, V, ks, vs, C, W, 0, 0.25)
    n = 150
    lo, ns = oracle.mask(n, C, W, 0)
    K2, V2, ks2, vs2 = K.copy(), V.copy(), ks.copy(), vs.copy()
    K2[:lo] = 30.0
    V2[:lo] = -30.0
    K2[n + 1:] = 30.0
    V2[n + 1:] = 30.0
    ks2[ns:] = 30.0
    vs2[ns:] = 30.0
    O2, lse2 = oracle.prefill(Q, K2, V2, ks2, vs2, C, W, 0, 0.25)
    assert np.array_equal(O2[n], O[n]) and lse2[n] == lse[n]


def test_prefill_detects_beta_perturbation():
    """SPEC fault injection: a 1e-3 perturbation of one beta is visible."""
    rng = np.random.default_rng(6)
    T, d, C, W = 128, 8, 8, 16
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    ks, vs = oracle.summarize(K, V, rng.normal(size=(T // C, d)), C)
    O, _ = oracle.prefill(Q, K, V, ks, vs, C, W, 0, 1.0)
    vs[3, 2] += 1e-3
    O2, _ = oracle.prefill(Q, K, V, ks, vs, C, W, 0, 1.0)
    assert np.max(np.abs(O2 - O)) > 1e-6
    # and rows that cannot see chunk 3 are untouched
    for n in range(T):
        if oracle.mask(n, C, W, 0)[1] <= 3:
            assert np.array_equal(O[n], O2[n])


def test_prefill_rows_matches_full():
    rng = np.random.default_rng(7)
    T, d, C, W = 300, 16, 16, 48
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    ks, vs = oracle.summarize(K, V, rng.normal(size=(T // C, d)), C)
    O, lse = oracle.prefill(Q, K, V, ks, vs, C, W, 1, 0.3)
    rows, Or, lr = oracle.prefill_rows(Q, K, V, ks, vs, [299, 0, 17, 160], C, W, 1, 0.3)
    assert np.array_equal(Or, O[rows]) and np.array_equal(lr, lse[rows])


def test_batch_drivers_match_per_unit():
    rng = np.random.default_rng(8)
    BH, T, d, C, W = 3, 64, 8, 4, 16
    Q, K, V = (rng.normal(size=(BH, T, d)) for _ in range(3))
    E = rng.normal(size=(BH, T // C, d))
    ks, vs = oracle.summarize_batch(K, V, E, C)
    O, lse = oracle.prefill_batch(Q, K, V, ks, vs, C, W, 0, 0.5)
    for u in range(BH):
        k1, v1 = oracle.summarize(K[u], V[u], E[u], C)
        o1, l1 = oracle.prefill(Q[u], K[u], V[u], k1, v1, C, W, 0, 0.5)
        assert np.array_equal(k1, ks[u]) and np.array_equal(v1, vs[u])
        assert np.array_equal(o1, O[u]) and np.array_equal(l1, lse[u])


# --------------------------------------------------------------------------- decode
@pytest.mark.parametrize("mode,C,W", [(oracle.SLIDING, 4, 12), (oracle.BLOCK, 4, 8),
                                      (oracle.SLIDING, 8, 8), (oracle.SLIDING, 16, 64)])
def test_decode_streaming_equals_prefill(mode, C, W):
    """Streaming row n == full recompute row n at every step."""
    rng = np.random.default_rng(9)
    T, d = 300, 8
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    E = rng.normal(size=(T // C + 1, d))
    ks, vs = oracle.summarize(K, V, E[: T // C], C)
    O, lse = oracle.prefill(Q, K, V, ks, vs, C, W, mode, 0.5)
    cache = oracle.Cache(d, C, W, mode, cap=T // C, scale=0.5)
    for n in range(T):
        assert cache.append(K[n], V[n], E[n // C]) == 0
        o, l = cache.decode(Q[n])
        assert np.max(np.abs(o - O[n])) < 1e-12 and abs(l - lse[n]) < 1e-12
    cks, cvs = cache.summaries()
    assert np.array_equal(cks, ks) and np.array_equal(cvs, vs)


def test_decode_chunk1_is_exact_softmax_and_capacity():
    rng = np.random.default_rng(10)
    T, d = 40, 4
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    ref = exact_causal_softmax(Q, K, V, 1.0)
    cache = oracle.Cache(d, 1, 3, oracle.SLIDING, cap=T)
    for n in range(T):
        cache.append(K[n], V[n], rng.normal(size=d))
        o, _ = cache.decode(Q[n])
        assert np.max(np.abs(o - ref[n])) < 1e-12
    small = oracle.Cache(d, 2, 2, oracle.SLIDING, cap=1)
    z = np.zeros(d)
    assert small.append(z, z, z) == 0 and small.append(z, z, z) == 0
    assert small.append(z, z, z) == 0
    assert small.append(z, z, z) == 3  # second summary exceeds cap = 1
