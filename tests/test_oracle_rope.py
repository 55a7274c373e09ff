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
