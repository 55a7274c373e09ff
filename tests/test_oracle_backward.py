"""Pins of oracle.backward (the fp64 gradient of the FlashEVA prefill, NEXT row 1).

oracle_backward writes the chain rule out step by step (eva_oracle.c); these
pins tie it to things other than itself:
  * central finite differences of the FORWARD oracle (summarize + prefill) on
    L = sum(dO * O) -- every element of dQ, dK, dV, both window modes, both
    omega readings, with clipped and unclipped channels present;
  * torch fp64 autograd through an independent DIRECT-form EVA (explicit index
    sets, linear-domain xi ratio, Eq.9/Eq.10 term by term; tests/bruteforce.py
    style, no shared code with the oracle);
  * special cases that reduce to textbook causal softmax attention: C = 1
    (every summary is its own token) and W >= T (no summaries).
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import oracle
from bruteforce import partition_sets


def _inputs(T, d, C, seed, scale_kv=1.0):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((T, d)) * 0.5
    K = rng.standard_normal((T, d)) * scale_kv
    V = rng.standard_normal((T, d))
    E = rng.standard_normal((max(T // C, 0), d))
    G = rng.standard_normal((T, d))
    return Q, K, V, E, G


def _loss(Q, K, V, E, G, C, W, mode, scale, omega_mode):
    ks, vs = oracle.summarize(K, V, E, C, omega_mode=omega_mode)
    O, _ = oracle.prefill(Q, K, V, ks, vs, C, W, mode, scale)
    return float((O * G).sum())


@pytest.mark.parametrize("mode,omega_mode", [(oracle.SLIDING, 0), (oracle.BLOCK, 0),
                                             (oracle.SLIDING, 1)])
def test_backward_matches_finite_differences(mode, omega_mode):
    T, d, C, W, scale = 16, 4, 2, 4, 0.7
    Q, K, V, E, G = _inputs(T, d, C, 11 + mode + 3 * omega_mode)
    # both clip branches must be exercised for the pin to mean anything
    kt = K.reshape(T // C, C, d).mean(axis=1)
    inside = np.abs(kt + E) <= 1.0
    assert inside.any() and (~inside).any()
    dQ, dK, dV = oracle.backward(Q, K, V, E, G, C, W, mode, scale, omega_mode=omega_mode)
    h = 1e-6
    for X, dX in ((Q, dQ), (K, dK), (V, dV)):
        num = np.zeros_like(X)
        for idx in np.ndindex(*X.shape):
            x0 = X[idx]
            X[idx] = x0 + h
            lp = _loss(Q, K, V, E, G, C, W, mode, scale, omega_mode)
            X[idx] = x0 - h
            lm = _loss(Q, K, V, E, G, C, W, mode, scale, omega_mode)
            X[idx] = x0
            num[idx] = (lp - lm) / (2 * h)
        np.testing.assert_allclose(dX, num, rtol=0, atol=2e-7)


def _torch_direct(Q, K, V, E, C, W, mode, scale, lam=0.1, clip=1.0, multiplicity=1.0):
    """EVA by explicit sets and the linear-domain Eq.9/Eq.10 mixture, in torch.
    mode: oracle.SLIDING / oracle.BLOCK or a bruteforce.partition_sets name ("noncausal:T");
    multiplicity: the weight of each chunk's Z-term (R16: bias = ln multiplicity)."""
    T = Q.shape[0]
    rows = []
    names = {oracle.SLIDING: "sliding", oracle.BLOCK: "block"}
    for n in range(T):
        Eset, chunks = partition_sets(n, C, W, names.get(mode, mode))
        num = torch.zeros(V.shape[1], dtype=torch.float64)
        Z = torch.zeros((), dtype=torch.float64)
        for m in Eset:
            w = torch.exp(scale * (Q[n] * K[m]).sum())
            Z = Z + w
            num = num + w * V[m]
        for members in chunks:
            c = members[0] // C  # the chunk's own index (non-causal lists skip the block)
            Kc, Vc = K[members], V[members]
            kt = Kc.sum(0) / len(members)
            om = lam * torch.clamp(kt + E[c], -clip, clip)
            xi = torch.exp((Kc * om).sum(1) - 0.5 * (Kc * Kc).sum(1))
            beta = (xi[:, None] * Vc).sum(0) / xi.sum()
            w = multiplicity * torch.exp(scale * (Q[n] * kt).sum())
            Z = Z + w
            num = num + w * beta
        rows.append(num / Z)
    return torch.stack(rows)


@pytest.mark.parametrize("mode", [oracle.SLIDING, oracle.BLOCK])
@pytest.mark.parametrize("C,W", [(2, 4), (3, 6), (4, 4)])
def test_backward_matches_autograd_of_direct_form(mode, C, W):
    T, d, scale = 4 * W + C + 1, 5, 0.5
    Q, K, V, E, G = _inputs(T, d, C, 100 + C + W + mode, scale_kv=0.6)
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (Q, K, V))
    O = _torch_direct(tq, tk, tv, torch.tensor(E), C, W, mode, scale)
    (O * torch.tensor(G)).sum().backward()
    dQ, dK, dV = oracle.backward(Q, K, V, E, G, C, W, mode, scale)
    np.testing.assert_allclose(dQ, tq.grad.numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(dK, tk.grad.numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(dV, tv.grad.numpy(), rtol=0, atol=1e-11)


def _causal_softmax_grads(Q, K, V, G, scale):
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (Q, K, V))
    T = Q.shape[0]
    S = scale * tq @ tk.T
    S = S.masked_fill(torch.triu(torch.ones(T, T, dtype=torch.bool), 1), -math.inf)
    (torch.softmax(S, -1) @ tv * torch.tensor(G)).sum().backward()
    return tq.grad.numpy(), tk.grad.numpy(), tv.grad.numpy()


@pytest.mark.parametrize("mode", [oracle.SLIDING, oracle.BLOCK])
@pytest.mark.parametrize("C,W,T", [(1, 3, 13), (4, 64, 40), (8, 32, 32)])
def test_backward_special_cases_are_causal_softmax(mode, C, W, T):
    """C = 1 (singleton summaries: k~ = k, beta = v, w = 1) or W >= T (no summaries)."""
    d, scale = 6, 0.8
    Q, K, V, E, G = _inputs(T, d, C, 7 * C + T)
    got = oracle.backward(Q, K, V, E, G, C, W, mode, scale)
    want = _causal_softmax_grads(Q, K, V, G, scale)
    for g, w in zip(got, want):
        np.testing.assert_allclose(g, w, rtol=0, atol=1e-12)


def test_backward_linear_in_dO_and_batch_driver():
    T, d, C, W = 24, 8, 4, 8
    BH = 3
    rng = np.random.default_rng(5)
    Q, K, V, G = (rng.standard_normal((BH, T, d)) for _ in range(4))
    E = rng.standard_normal((BH, T // C, d))
    bq, bk, bv = oracle.backward_batch(Q, K, V, E, G, C, W)
    for u in range(BH):
        q, k, v = oracle.backward(Q[u], K[u], V[u], E[u], G[u], C, W)
        np.testing.assert_array_equal(bq[u], q)
        np.testing.assert_array_equal(bk[u], k)
        np.testing.assert_array_equal(bv[u], v)
    # L is linear in dO: grads(2 dO1 - dO2) = 2 grads(dO1) - grads(dO2)
    G2 = rng.standard_normal((T, d))
    a = oracle.backward(Q[0], K[0], V[0], E[0], G[0], C, W)
    b = oracle.backward(Q[0], K[0], V[0], E[0], G2, C, W)
    c = oracle.backward(Q[0], K[0], V[0], E[0], 2 * G[0] - G2, C, W)
    for x, y, z in zip(a, b, c):
        np.testing.assert_allclose(z, 2 * x - y, rtol=0, atol=1e-12)


# ---- the variants (NEXT row 3 backward): non-causal partition (R15), summary bias (R16)

def _loss_ext(Q, K, V, E, G, C, W, mode, scale, bias):
    ks, vs = oracle.summarize(K, V, E, C)
    O, _ = oracle.prefill_ext_batch(Q[None], K[None], V[None], ks[None], vs[None], C, W, mode,
                                    scale, bias)
    return float((O[0] * G).sum())


@pytest.mark.parametrize("mode,bias", [(oracle.NONCAUSAL, 0.0), (oracle.NONCAUSAL, 0.9),
                                       (oracle.SLIDING, math.log(2.0)), (oracle.BLOCK, -0.4)])
def test_variant_backward_matches_finite_differences(mode, bias):
    """Every element of dQ, dK, dV against central differences of the forward oracle
    (summarize + oracle_prefill_ext, itself pinned in test_oracle_variants.py)."""
    T, d, C, W, scale = 16, 4, 2, 4, 0.7
    Q, K, V, E, G = _inputs(T, d, C, 31 + mode)
    dQ, dK, dV = oracle.backward(Q, K, V, E, G, C, W, mode, scale, bias=bias)
    h = 1e-6
    for X, dX in ((Q, dQ), (K, dK), (V, dV)):
        num = np.zeros_like(X)
        for idx in np.ndindex(*X.shape):
            x0 = X[idx]
            X[idx] = x0 + h
            lp = _loss_ext(Q, K, V, E, G, C, W, mode, scale, bias)
            X[idx] = x0 - h
            lm = _loss_ext(Q, K, V, E, G, C, W, mode, scale, bias)
            X[idx] = x0
            num[idx] = (lp - lm) / (2 * h)
        np.testing.assert_allclose(dX, num, rtol=0, atol=2e-7)


@pytest.mark.parametrize("C,W,T,mult", [(2, 4, 16, 1.0), (3, 6, 18, 3.0), (2, 6, 12, 1.0)])
def test_noncausal_backward_matches_autograd_of_direct_form(C, W, T, mult):
    """Explicit non-causal sets (own block incl. future, chunks before AND after) with the
    chunk multiplicity as a Z weight; the oracle takes bias = ln(multiplicity)."""
    d, scale = 5, 0.5
    Q, K, V, E, G = _inputs(T, d, C, 200 + C + W + T, scale_kv=0.6)
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (Q, K, V))
    O = _torch_direct(tq, tk, tv, torch.tensor(E), C, W, f"noncausal:{T}", scale,
                      multiplicity=mult)
    (O * torch.tensor(G)).sum().backward()
    got = oracle.backward(Q, K, V, E, G, C, W, oracle.NONCAUSAL, scale, bias=math.log(mult))
    for g, w in zip(got, (tq.grad, tk.grad, tv.grad)):
        np.testing.assert_allclose(g, w.numpy(), rtol=0, atol=1e-11)


@pytest.mark.parametrize("mode", [oracle.SLIDING, oracle.BLOCK])
def test_bias_backward_matches_autograd_with_multiplicity(mode):
    C, W, d, scale = 4, 8, 4, 0.6
    T = 3 * W + 3
    Q, K, V, E, G = _inputs(T, d, C, 300 + mode, scale_kv=0.6)
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (Q, K, V))
    O = _torch_direct(tq, tk, tv, torch.tensor(E), C, W, mode, scale, multiplicity=C)
    (O * torch.tensor(G)).sum().backward()
    got = oracle.backward(Q, K, V, E, G, C, W, mode, scale, bias=math.log(C))
    for g, w in zip(got, (tq.grad, tk.grad, tv.grad)):
        np.testing.assert_allclose(g, w.numpy(), rtol=0, atol=1e-11)


def _full_softmax_grads(Q, K, V, G, scale):
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (Q, K, V))
    (torch.softmax(scale * tq @ tk.T, -1) @ tv * torch.tensor(G)).sum().backward()
    return tq.grad.numpy(), tk.grad.numpy(), tv.grad.numpy()


@pytest.mark.parametrize("C,W,T", [(1, 3, 12), (4, 64, 40), (8, 32, 32)])
def test_noncausal_special_cases_are_full_softmax(C, W, T):
    """Non-causal with C = 1 (every token outside the block is its own summary) or W >= T
    (one block, no summaries) is textbook bidirectional softmax attention (Eq.1)."""
    d, scale = 6, 0.8
    Q, K, V, E, G = _inputs(T, d, C, 9 * C + T)
    got = oracle.backward(Q, K, V, E, G, C, W, oracle.NONCAUSAL, scale)
    for g, w in zip(got, _full_softmax_grads(Q, K, V, G, scale)):
        np.testing.assert_allclose(g, w, rtol=0, atol=1e-12)
