"""Pins of the oracle's prefill variants (R15, R16):
the non-causal partition and the summary-logit bias (the |P_c| multiplicity that
Eq.10, omits).  Each pin is independent of the oracle's code: torch SDPA, a two-loop
softmax, the brute-force set enumeration of tests/bruteforce.py, or a closed form."""
import math

import numpy as np
import pytest
import torch

import oracle
from bruteforce import eva_direct, exact_causal_softmax, exact_softmax


def _one(x):
    return x[None]


def test_noncausal_window_covers_sequence_is_full_softmax():
    """W >= T: one block, no summaries -> Eq.1 without the causal restriction (SDPA fp64)."""
    rng = np.random.default_rng(20)
    T, d, C = 96, 16, 8
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    ks, vs = oracle.summarize(K, V, rng.normal(size=(T // C, d)), C)
    O, lse = oracle.prefill_ext_batch(_one(Q), _one(K), _one(V), _one(ks), _one(vs), C, 128,
                                      oracle.NONCAUSAL, 0.3)
    ref = torch.nn.functional.scaled_dot_product_attention(
        *(torch.from_numpy(x)[None, None] for x in (Q, K, V)), is_causal=False, scale=0.3)[0, 0]
    assert np.max(np.abs(O[0] - ref.numpy())) < 1e-12
    lg = 0.3 * Q @ K.T
    assert np.max(np.abs(lse[0] - (np.log(np.exp(lg - lg.max(1, keepdims=True)).sum(1)) + lg.max(1)))) < 1e-12


def test_noncausal_chunk1_is_full_softmax():
    """C = 1: every summary is its token (k~ = k, beta = v) -> full softmax for any W, eps."""
    rng = np.random.default_rng(21)
    T, d = 60, 8
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    ks, vs = oracle.summarize(K, V, 4 * rng.normal(size=(T, d)), 1)
    for W in (1, 4, 7, 64):
        O, _ = oracle.prefill_ext_batch(_one(Q), _one(K), _one(V), _one(ks), _one(vs), 1, W,
                                        oracle.NONCAUSAL, 0.9)
        assert np.max(np.abs(O[0] - exact_softmax(Q, K, V, 0.9))) < 1e-12


def test_noncausal_equals_direct_eq9_bruteforce():
    """Augmented form == direct Eq.9/10 with the non-causal partition as explicit sets."""
    rng = np.random.default_rng(22)
    for trial in range(30):
        C = int(rng.choice([1, 2, 3, 4]))
        W = C * int(rng.integers(1, 4))
        T = C * int(rng.integers(1, 12))
        d = int(rng.integers(1, 7))
        Q, K, V = (0.6 * rng.normal(size=(T, d)) for _ in range(3))
        E = rng.normal(size=(T // C, d))
        scale = float(rng.uniform(0.3, 1.5))
        ks, vs = oracle.summarize(K, V, E, C)
        O, _ = oracle.prefill_ext_batch(_one(Q), _one(K), _one(V), _one(ks), _one(vs), C, W,
                                        oracle.NONCAUSAL, scale)
        ref = eva_direct(Q, K, V, E, C, W, f"noncausal:{T}", scale)
        assert np.max(np.abs(O[0] - ref)) < 1e-12, (trial, C, W, T, d)


@pytest.mark.parametrize("mode", ["sliding", "block"])
def test_bias_equals_direct_with_multiplicity(mode):
    """bias b on every summary logit == each chunk's Z-term counted e^b times (brute force)."""
    rng = np.random.default_rng(23)
    m = oracle.SLIDING if mode == "sliding" else oracle.BLOCK
    for trial in range(20):
        C = int(rng.choice([2, 3, 4]))
        W = C * int(rng.integers(1, 3))
        T = int(rng.integers(C, 36))
        d = int(rng.integers(1, 6))
        Q, K, V = (0.6 * rng.normal(size=(T, d)) for _ in range(3))
        E = rng.normal(size=(T // C, d))
        ks, vs = oracle.summarize(K, V, E, C)
        O, _ = oracle.prefill_ext_batch(_one(Q), _one(K), _one(V), _one(ks), _one(vs), C, W, m, 0.8,
                                        bias=math.log(C))
        ref = eva_direct(Q, K, V, E, C, W, mode, 0.8, multiplicity=C)
        assert np.max(np.abs(O[0] - ref)) < 1e-12, (trial, C, W, T)


@pytest.mark.parametrize("mode", [oracle.SLIDING, oracle.BLOCK, oracle.NONCAUSAL])
def test_bias_lnC_makes_constant_chunks_exact(mode):
    """Closed form: if every chunk repeats one key/value (k~ = k, beta = v), a summary with
    bias ln C stands exactly for its C identical tokens, so the output is exact softmax
    attention (causal or full); without the bias it is not."""
    rng = np.random.default_rng(24)
    T, d, C, W = 64, 8, 4, 16
    base_k, base_v = rng.normal(size=(T // C, d)), rng.normal(size=(T // C, d))
    K = np.repeat(base_k, C, axis=0)
    V = np.repeat(base_v, C, axis=0)
    Q = rng.normal(size=(T, d))
    ks, vs = oracle.summarize(K, V, rng.normal(size=(T // C, d)), C)
    assert np.max(np.abs(ks - base_k)) < 1e-14 and np.max(np.abs(vs - base_v)) < 1e-14
    ref = exact_softmax(Q, K, V, 0.5) if mode == oracle.NONCAUSAL else exact_causal_softmax(Q, K, V, 0.5)
    O, _ = oracle.prefill_ext_batch(_one(Q), _one(K), _one(V), _one(ks), _one(vs), C, W, mode, 0.5,
                                    bias=math.log(C))
    O0, _ = oracle.prefill_ext_batch(_one(Q), _one(K), _one(V), _one(ks), _one(vs), C, W, mode, 0.5)
    assert np.max(np.abs(O[0] - ref)) < 1e-12
    assert np.max(np.abs(O0[0] - ref)) > 1e-3


def test_ext_causal_bias0_matches_prefill_and_row_stochastic():
    rng = np.random.default_rng(25)
    T, d, C, W = 100, 8, 4, 12
    Q, K, V = (rng.normal(size=(T, d)) for _ in range(3))
    ks, vs = oracle.summarize(K, V, rng.normal(size=(T // C, d)), C)
    for mode in (oracle.SLIDING, oracle.BLOCK):
        O, l = oracle.prefill(Q, K, V, ks, vs, C, W, mode, 0.4)
        O2, l2 = oracle.prefill_ext_batch(_one(Q), _one(K), _one(V), _one(ks), _one(vs), C, W, mode, 0.4)
        assert np.max(np.abs(O - O2[0])) < 1e-14 and np.max(np.abs(l - l2[0])) < 1e-13
    for mode in (oracle.SLIDING, oracle.BLOCK, oracle.NONCAUSAL):
        O1, _ = oracle.prefill_ext_batch(_one(Q), _one(K), _one(np.ones_like(V)), _one(ks),
                                         _one(np.ones_like(vs)), C, W, mode, 0.4, bias=1.7)
        assert np.max(np.abs(O1 - 1)) < 1e-13
