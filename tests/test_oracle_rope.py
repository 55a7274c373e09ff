"""Pins of oracle.rope (RoPE fused into the producer, NEXT row 4, R18).

  * position 0 is the identity; d = 2 is the complex rotation e^{i pos};
  * every row keeps its norm (a rotation);
  * the relative-position property: <rope(q, m), rope(k, n)> depends on m - n only;
  * explicit complex-number form (x_2j + i x_2j+1) e^{i pos theta_j} on random rows.
"""
import numpy as np

import oracle


def test_position_zero_is_identity_and_d2_is_complex_rotation():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((1, 8))
    np.testing.assert_array_equal(oracle.rope(X, pos0=0), X)
    Y = oracle.rope(np.array([[1.0, 0.0]] * 5), pos0=3)
    want = np.array([[np.cos(p), np.sin(p)] for p in range(3, 8)])
    np.testing.assert_allclose(Y, want, rtol=0, atol=1e-15)


def test_norm_preserved():
    X = np.random.default_rng(1).standard_normal((50, 16))
    Y = oracle.rope(X, base=500.0, pos0=123)
    np.testing.assert_allclose(np.linalg.norm(Y, axis=1), np.linalg.norm(X, axis=1), rtol=1e-13)


def test_relative_position_property():
    rng = np.random.default_rng(2)
    q, k = rng.standard_normal((1, 32)), rng.standard_normal((1, 32))
    dots = [float((oracle.rope(q, pos0=m) @ oracle.rope(k, pos0=m - 7).T).item()) for m in (7, 50, 1000)]
    np.testing.assert_allclose(dots, dots[0], rtol=0, atol=1e-10)


def test_complex_form():
    rng = np.random.default_rng(3)
    T, d, base, p0 = 6, 12, 10000.0, 40
    X = rng.standard_normal((T, d))
    Y = oracle.rope(X, base=base, pos0=p0)
    theta = base ** (-2.0 * np.arange(d // 2) / d)
    Z = (X[:, 0::2] + 1j * X[:, 1::2]) * np.exp(1j * np.outer(np.arange(p0, p0 + T), theta))
    np.testing.assert_allclose(Y[:, 0::2], Z.real, rtol=0, atol=1e-12)
    np.testing.assert_allclose(Y[:, 1::2], Z.imag, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- rope_ex (R19): partial rotary,
# GPT-NeoX half-split pairs, per-row positions, the inverse
def test_rope_ex_full_interleaved_equals_rope():
    """rotary_dim = d, interleaved, positions pos0 + t: the R18 rotation (pinned above)."""
    X = np.random.default_rng(4).standard_normal((9, 16))
    np.testing.assert_allclose(oracle.rope_ex(X, np.arange(30, 39)), oracle.rope(X, pos0=30), rtol=0, atol=1e-13)


def test_rope_ex_neox_complex_form():
    """Half-split pairs: (x_j + i x_{j+rd/2}) e^{i pos theta_j}, theta_j = base^(-2j/rd)
    (GPT-NeoX rotate_half: y = x cos + rotate_half(x) sin with cos/sin repeated over halves)."""
    rng = np.random.default_rng(5)
    T, d, base = 7, 12, 500.0
    X = rng.standard_normal((T, d))
    pos = rng.integers(0, 5000, T)
    Y = oracle.rope_ex(X, pos, base=base, style=oracle.ROPE_NEOX)
    theta = base ** (-2.0 * np.arange(d // 2) / d)
    Z = (X[:, :d // 2] + 1j * X[:, d // 2:]) * np.exp(1j * np.outer(pos, theta))
    np.testing.assert_allclose(Y[:, :d // 2], Z.real, rtol=0, atol=1e-11)
    np.testing.assert_allclose(Y[:, d // 2:], Z.imag, rtol=0, atol=1e-11)
    # rotate_half written out
    cos = np.cos(np.outer(pos, np.concatenate([theta, theta])))
    sin = np.sin(np.outer(pos, np.concatenate([theta, theta])))
    rot_half = np.concatenate([-X[:, d // 2:], X[:, :d // 2]], axis=1)
    np.testing.assert_allclose(Y, X * cos + rot_half * sin, rtol=0, atol=1e-11)


def test_rope_ex_partial_rotary_dim():
    """Channels >= rotary_dim pass through unchanged; the first rd rotate as a d = rd rope."""
    rng = np.random.default_rng(6)
    X = rng.standard_normal((5, 64))
    pos = np.array([0, 3, 17, 1000, 65535])
    for style in (oracle.ROPE_INTERLEAVED, oracle.ROPE_NEOX):
        Y = oracle.rope_ex(X, pos, rotary_dim=16, style=style)
        np.testing.assert_array_equal(Y[:, 16:], X[:, 16:])
        np.testing.assert_allclose(Y[:, :16], oracle.rope_ex(X[:, :16], pos, style=style), rtol=0, atol=1e-13)
    np.testing.assert_allclose(oracle.rope_ex(X, pos, rotary_dim=16)[:, :16],
                               np.concatenate([oracle.rope(X[t:t + 1, :16], pos0=int(p)) for t, p in enumerate(pos)]),
                               rtol=0, atol=1e-12)


def test_rope_ex_neox_is_interleaved_after_channel_permutation():
    """NeoX on x equals interleaved on the permuted x (channel 2j <- j, 2j+1 <- j + rd/2)."""
    rng = np.random.default_rng(7)
    X = rng.standard_normal((4, 32))
    pos = np.array([1, 9, 400, 77777])
    perm = np.empty(32, dtype=int)
    perm[0::2], perm[1::2] = np.arange(16), np.arange(16, 32)
    A = oracle.rope_ex(X, pos, style=oracle.ROPE_NEOX)
    B = oracle.rope_ex(X[:, perm], pos, style=oracle.ROPE_INTERLEAVED)
    np.testing.assert_allclose(A[:, perm], B, rtol=0, atol=1e-12)


def test_rope_ex_inverse_and_norm_and_relative_position():
    rng = np.random.default_rng(8)
    X = rng.standard_normal((6, 24))
    pos = rng.integers(0, 10 ** 6, 6)
    for style in (0, 1):
        Y = oracle.rope_ex(X, pos, rotary_dim=16, style=style)
        np.testing.assert_allclose(oracle.rope_ex(Y, pos, rotary_dim=16, style=style, inverse=True), X,
                                   rtol=0, atol=1e-9)
        np.testing.assert_allclose(np.linalg.norm(Y, axis=1), np.linalg.norm(X, axis=1), rtol=1e-12)
        q, k = X[:1], X[1:2]
        dots = [float(oracle.rope_ex(q, [m], style=style) @ oracle.rope_ex(k, [m - 11], style=style).T)
                for m in (11, 500, 90000)]
        np.testing.assert_allclose(dots, dots[0], rtol=0, atol=1e-9)
