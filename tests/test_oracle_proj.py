"""Pins of oracle.summarize_proj: the learned summary-key projection (NEXT row 4, DESIGN.md
R17: k~_c = P mean(k_c), mu_c = k~_c in Eq.15, beta from Eq.9 with the raw keys).

  * P = I reduces to oracle.summarize exactly (pinned in test_oracle.py);
  * brute force: bruteforce.summary_direct with an explicit double-loop projection and the
    linear-domain xi ratio, on a non-symmetric P (a transposed P fails it);
  * P = 0: k~ = 0 and omega = lambda clip(eps) in closed form;
  * P = a I: k~ = a mean(k).
"""
import numpy as np
import pytest

import oracle
from bruteforce import summary_direct


def _data(T, d, C, seed):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((T, d)) * 0.5
    V = rng.standard_normal((T, d))
    E = rng.standard_normal((T // C, d))
    return K, V, E


def test_identity_projection_is_unprojected():
    K, V, E = _data(40, 8, 4, 1)
    a = oracle.summarize(K, V, E, 4, return_omega=True)
    b = oracle.summarize_proj(K, V, E, np.eye(8), 4, return_omega=True)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("C,d", [(4, 6), (3, 5), (8, 4)])
def test_projection_matches_bruteforce(C, d):
    T = 5 * C + 2
    K, V, E = _data(T, d, C, 10 + C)
    P = np.random.default_rng(C).standard_normal((d, d)) * 0.7   # not symmetric
    ks, vs, om = oracle.summarize_proj(K, V, E, P, C, return_omega=True)
    for c in range(T // C):
        kt, omega, beta = summary_direct(K[c * C:(c + 1) * C], V[c * C:(c + 1) * C], E[c], P=P)
        np.testing.assert_allclose(ks[c], kt, rtol=0, atol=1e-13)
        np.testing.assert_allclose(om[c], omega, rtol=0, atol=1e-13)
        np.testing.assert_allclose(vs[c], beta, rtol=0, atol=1e-12)
    # the transposed projection is a different (wrong) answer here
    kt_T, _ = oracle.summarize_proj(K, V, E, P.T, C)
    assert np.max(np.abs(kt_T - ks)) > 1e-3


def test_zero_projection_closed_form():
    C, d, lam = 4, 6, 0.1
    K, V, E = _data(24, d, C, 3)
    ks, vs, om = oracle.summarize_proj(K, V, E, np.zeros((d, d)), C, return_omega=True)
    np.testing.assert_array_equal(ks, 0.0)
    np.testing.assert_allclose(om, lam * np.clip(E, -1, 1), rtol=0, atol=1e-15)


def test_scaled_identity_scales_the_mean():
    C, d, a = 4, 6, -1.7
    K, V, E = _data(24, d, C, 4)
    ks0, _ = oracle.summarize(K, V, E, C)
    ks, _ = oracle.summarize_proj(K, V, E, a * np.eye(d), C)
    np.testing.assert_allclose(ks, a * ks0, rtol=0, atol=1e-14)


# ---------------------------------------------------------------- backward through the projection
def _loss_proj(Q, K, V, E, P, dO, C, W, mode, scale, lam, clip, om):
    ks, vs = oracle.summarize_proj(K, V, E, P, C, lam=lam, clip=clip, omega_mode=om)
    O, _ = oracle.prefill(Q, K, V, ks, vs, C, W, mode, scale)
    return float(np.sum(O * dO))


import pytest  # noqa: E402


@pytest.mark.parametrize("om", [0, 1])
@pytest.mark.parametrize("mode", [oracle.SLIDING, oracle.BLOCK])
def test_backward_proj_finite_differences(om, mode):
    """dQ, dK, dV and dP of oracle_backward_proj against central differences of the forward
    (summarize_proj + prefill), with a clip that bites (lambda = 1, eps 1.5x) so the Eq.15 gate
    and both omega readings matter, on a non-symmetric P."""
    rng = np.random.default_rng(11 + om + 3 * mode)
    T, d, C, W = 22, 4, 4, 8
    Q, K, V, dO = (rng.standard_normal((T, d)) for _ in range(4))
    E = 1.5 * rng.standard_normal((T // C, d))
    P = rng.standard_normal((d, d)) * 0.7 + np.eye(d)
    lam, clip, scale = 1.0, 1.0, 0.8
    dQ, dK, dV, dP = oracle.backward_proj(Q, K, V, E, P, dO, C, W, mode, scale, lam, clip, om)
    h = 1e-6
    for name, X, G in (("Q", Q, dQ), ("K", K, dK), ("V", V, dV), ("P", P, dP)):
        idx = [tuple(rng.integers(0, s) for s in X.shape) for _ in range(12)]
        for ix in idx:
            Xp, Xm = X.copy(), X.copy()
            Xp[ix] += h
            Xm[ix] -= h
            args = dict(Q=Q, K=K, V=V, P=P)
            args[name] = Xp
            lp = _loss_proj(args["Q"], args["K"], args["V"], E, args["P"], dO, C, W, mode, scale, lam, clip, om)
            args[name] = Xm
            lm = _loss_proj(args["Q"], args["K"], args["V"], E, args["P"], dO, C, W, mode, scale, lam, clip, om)
            fd = (lp - lm) / (2 * h)
            assert abs(fd - G[ix]) <= 1e-6 * max(1.0, abs(fd)), (name, ix, fd, G[ix])


def test_backward_proj_identity_equals_plain_backward():
    """P = I reduces to the pinned oracle_backward (k~ = mean); dP = sum_c g_c mean_c^T."""
    rng = np.random.default_rng(5)
    T, d, C, W = 40, 8, 8, 16
    Q, K, V, dO = (rng.standard_normal((T, d)) for _ in range(4))
    E = rng.standard_normal((T // C, d))
    a = oracle.backward_proj(Q, K, V, E, np.eye(d), dO, C, W, scale=0.5)
    b = oracle.backward(Q, K, V, E, dO, C, W, scale=0.5)
    for x, y in zip(a[:3], b):
        np.testing.assert_allclose(x, y, rtol=0, atol=1e-12)
