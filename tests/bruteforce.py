"""Independent brute-force checker of EVA in its DIRECT form (Eq.9 with Eq.10).

Test helper only.  It shares nothing with oracle/eva_oracle.c: the partition is
enumerated as explicit index SETS from SPEC's 1-indexed text definition
(S:210), the summaries are evaluated in the LINEAR domain as the ratio
sum_m xi(k_m, w) v_m / sum_m xi(k_m, w) (Eq.9 with S = 1), and the
output is the Eq.9/Eq.10 mixture written term by term:

    Z   = sum_{m in E} exp(s q.k_m) + sum_c exp(s q.k~_c)           (Eq.10)
    EVA = sum_{m in E} exp(s q.k_m)/Z v_m + sum_c exp(s q.k~_c)/Z beta_c   (Eq.9)

Linear-domain exp is only safe for small inputs (|x| <~ 1, d <= 8); callers
keep to that.
"""
from __future__ import annotations

import math

import numpy as np


def partition_sets(n: int, C: int, W: int, mode: str):
    """E(n) and the ordered chunk list of query n (0-indexed in/out).

    SPEC S:210: sliding-chunk-aligned E(p) = (a-W, a] cap [1, p] with
    a = C*ceil(p/C); block-local E(p) = p's block of width W.  All earlier
    positions are grouped left to right into chunks of exactly C.
    """
    p = n + 1
    if mode == "sliding":
        a = C * math.ceil(p / C)
        E = [x for x in range(a - W + 1, a + 1) if 1 <= x <= p]
    elif mode == "block":
        b = math.ceil(p / W)
        E = list(range((b - 1) * W + 1, p + 1))
    elif mode.startswith("noncausal:"):
        # non-causal EVA (R15): E(p) = p's whole block of width W (future
        # positions of the block included); every position outside it, before AND after, is
        # grouped left to right into chunks of exactly C (the caller's T is a multiple of C).
        T = int(mode.split(":")[1])
        b = math.ceil(p / W)
        E = list(range((b - 1) * W + 1, min(b * W, T) + 1))
        earlier = list(range(1, min(E)))
        later = list(range(max(E) + 1, T + 1))
        assert len(earlier) % C == 0 and len(later) % C == 0
        chunks = [earlier[i:i + C] for i in range(0, len(earlier), C)] + \
                 [later[i:i + C] for i in range(0, len(later), C)]
        return [x - 1 for x in E], [[x - 1 for x in ch] for ch in chunks]
    else:
        raise ValueError(mode)
    earlier = list(range(1, min(E)))
    assert len(earlier) % C == 0, "partial chunk before the window"
    chunks = [earlier[i:i + C] for i in range(0, len(earlier), C)]
    return [x - 1 for x in E], [[x - 1 for x in ch] for ch in chunks]


def summary_direct(Kc, Vc, eps_c, lam=0.1, clip=1.0, P=None):
    """(k~, omega, beta) of one chunk, linear-domain xi ratio.  P: optional learned projection
    of the summary key, k~ = sum_l P[j, l] mean_l written as an explicit double loop."""
    Kc = np.asarray(Kc, dtype=np.float64)
    Vc = np.asarray(Vc, dtype=np.float64)
    kt = Kc.sum(axis=0) / Kc.shape[0]
    if P is not None:
        m = kt
        kt = np.array([sum(float(P[j][l]) * float(m[l]) for l in range(len(m))) for j in range(len(m))])
    omega = lam * np.clip(kt + np.asarray(eps_c, dtype=np.float64), -clip, clip)
    xi = np.array([math.exp(float(omega @ k) - 0.5 * float(k @ k)) for k in Kc])
    beta = (xi[:, None] * Vc).sum(axis=0) / xi.sum()
    return kt, omega, beta


def eva_direct(Q, K, V, E_eps, C: int, W: int, mode: str, scale: float = 1.0, lam=0.1, clip=1.0,
               multiplicity: float = 1.0):
    """EVA output of one unit, every query by explicit sets.  Returns O [T, d].
    multiplicity: each chunk's Z-term exp(q.k~_c) counts this many times (1 = Eq.10 as
    printed; C = the |P_c| tokens the chunk replaces, R16)."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    T, d = Q.shape
    O = np.zeros((T, V.shape[1]))
    for n in range(T):
        E, chunks = partition_sets(n, C, W, mode)
        num = np.zeros(V.shape[1])
        Z = 0.0
        for m in E:
            w = math.exp(scale * float(Q[n] @ K[m]))
            Z += w
            num += w * V[m]
        for members in chunks:
            c = members[0] // C
            assert members == list(range(c * C, c * C + C))
            kt, _, beta = summary_direct(K[members], V[members], E_eps[c], lam, clip)
            w = multiplicity * math.exp(scale * float(Q[n] @ kt))
            Z += w
            num += w * beta
        O[n] = num / Z
    return O


def exact_causal_softmax(Q, K, V, scale=1.0):
    """Eq.1 with the causal restriction m <= n, two loops."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    T = Q.shape[0]
    O = np.zeros((T, V.shape[1]))
    for n in range(T):
        w = np.array([math.exp(scale * float(Q[n] @ K[m])) for m in range(n + 1)])
        O[n] = (w[:, None] * V[: n + 1]).sum(axis=0) / w.sum()
    return O


def exact_softmax(Q, K, V, scale=1.0):
    """Eq.1 without the causal restriction (every query sees every key), two loops."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    O = np.zeros((Q.shape[0], V.shape[1]))
    for n in range(Q.shape[0]):
        w = np.array([math.exp(scale * float(Q[n] @ K[m])) for m in range(K.shape[0])])
        O[n] = (w[:, None] * V).sum(axis=0) / w.sum()
    return O
