"""fp64 CPU oracle of the FlashEVA hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2511_00576_b200`` never imports it and shares no code with it.

The arithmetic lives in ``oracle/eva_oracle.c`` (plain C, fp64, one
(batch, head) unit at a time, in the paper's order); this module only
marshals numpy arrays.  Citations (P:NN = PAPER.md line, S:NN = SPEC.md line)
are in the C file and in DESIGN.md.

Parity pins: tests/test_oracle*.py.  Every public function here is pinned
(Philox KAT, closed forms, worked examples, exact-softmax special cases,
brute-force Eq.9/10 direct form, streaming == prefill, finite differences and
autograd for the backward, the projection and RoPE identities).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eva_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

SLIDING = 0
BLOCK = 1
NONCAUSAL = 2


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2, fp64, OpenMP over independent units)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC",
                               "-fvisibility=hidden", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        D = ctypes.POINTER(ctypes.c_double)
        I64 = ctypes.POINTER(ctypes.c_int64)
        U32 = ctypes.POINTER(ctypes.c_uint32)
        i, d_ = ctypes.c_int, ctypes.c_double
        lib.oracle_philox4x32_10.argtypes = [U32, U32, U32]
        lib.oracle_eps.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, i, i, D]
        lib.oracle_mask.argtypes = [ctypes.c_int64, i, i, i, I64, I64]
        lib.oracle_summarize.argtypes = [i, i, i, D, D, D, d_, d_, i, D, D, D]
        lib.oracle_summarize_proj.argtypes = [i, i, i, D, D, D, D, d_, d_, i, D, D, D]
        lib.oracle_rope.argtypes = [i, i, d_, ctypes.c_int64, D]
        lib.oracle_rope_ex.argtypes = [i, i, d_, i, i, I64, i, D]
        lib.oracle_backward_proj.argtypes = [i, i, i, i, i, d_, d_, d_, i, D, D, D, D, D, D, D, D, D, D]
        lib.oracle_prefill.argtypes = [i, i, i, i, i, d_, D, D, D, D, D, D, D]
        lib.oracle_summarize_batch.argtypes = [i, i, i, i, D, D, D, d_, d_, i, D, D]
        lib.oracle_prefill_batch.argtypes = [i, i, i, i, i, i, d_, D, D, D, D, D, D, D]
        lib.oracle_prefill_ext_batch.argtypes = [i, i, i, i, i, i, d_, d_, D, D, D, D, D, D, D]
        lib.oracle_prefill_rows.argtypes = [i, i, i, i, i, d_, D, D, D, D, D, i, I64, D, D]
        lib.oracle_backward.argtypes = [i, i, i, i, i, d_, d_, d_, i, D, D, D, D, D, D, D, D]
        lib.oracle_backward_batch.argtypes = [i, i, i, i, i, i, d_, d_, d_, i, D, D, D, D, D, D, D, D]
        lib.oracle_backward_ext.argtypes = [i, i, i, i, i, d_, d_, d_, d_, i, D, D, D, D, D, D, D, D]
        lib.oracle_backward_ext_batch.argtypes = [i, i, i, i, i, i, d_, d_, d_, d_, i, D, D, D, D, D,
                                                  D, D, D]
        lib.oracle_cache_new.argtypes = [i, i, i, i, i, d_, d_, d_, i]
        lib.oracle_cache_new.restype = ctypes.c_void_p
        lib.oracle_cache_free.argtypes = [ctypes.c_void_p]
        lib.oracle_cache_pos.argtypes = [ctypes.c_void_p]
        lib.oracle_cache_pos.restype = ctypes.c_int64
        lib.oracle_cache_sum_k.argtypes = [ctypes.c_void_p]
        lib.oracle_cache_sum_k.restype = D
        lib.oracle_cache_sum_v.argtypes = [ctypes.c_void_p]
        lib.oracle_cache_sum_v.restype = D
        lib.oracle_cache_append.argtypes = [ctypes.c_void_p, D, D, D]
        lib.oracle_cache_append.restype = ctypes.c_int
        lib.oracle_cache_decode.argtypes = [ctypes.c_void_p, D, D]
        lib.oracle_cache_decode.restype = ctypes.c_double
        _lib = lib
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def philox4x32_10(ctr, key):
    """One Philox4x32-10 block: 4 counter words, 2 key words -> 4 words."""
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    _L().oracle_philox4x32_10(c, k, o)
    return [int(x) for x in o]


def eps(seed: int, layer: int, bh: int, nC: int, d: int) -> np.ndarray:
    """eps_c ~ N(0, I_d) for chunks 0..nC-1 of global unit bh (reading R9)."""
    out = np.zeros((nC, d), dtype=np.float64)
    if nC > 0:
        _L().oracle_eps(ctypes.c_uint64(seed), layer, bh, nC, d, _dp(out))
    return out


def eps_units(seed: int, layer: int, bh_begin: int, bh_count: int, nC: int, d: int) -> np.ndarray:
    return np.stack([eps(seed, layer, bh_begin + u, nC, d) for u in range(bh_count)]) \
        if bh_count else np.zeros((0, nC, d))


def mask(n: int, C: int, W: int, mode: int = SLIDING):
    """(lo, nsum) of query n: locals [lo, n], summaries c < nsum (reading R7)."""
    lo = ctypes.c_int64()
    ns = ctypes.c_int64()
    _L().oracle_mask(n, C, W, mode, ctypes.byref(lo), ctypes.byref(ns))
    return lo.value, ns.value


def summarize(K, V, eps_, C: int, lam: float = 0.1, clip: float = 1.0, omega_mode: int = 0,
              return_omega: bool = False):
    """Chunk summaries of one unit: K, V [T, d], eps [nC, d] -> Ksum, Vsum [nC, d]."""
    K, V, E = _f64(K), _f64(V), _f64(eps_)
    T, d = K.shape
    nC = T // C
    ks = np.zeros((nC, d))
    vs = np.zeros((nC, d))
    om = np.zeros((nC, d))
    if nC > 0:
        _L().oracle_summarize(T, d, C, _dp(K), _dp(V), _dp(E), lam, clip, omega_mode,
                              _dp(ks), _dp(vs), _dp(om))
    return (ks, vs, om) if return_omega else (ks, vs)


def rope(X, base: float = 10000.0, pos0: int = 0):
    """Rotary position embedding of rows X [T, d] at positions pos0.. (oracle_rope, R18):
    consecutive channel pairs rotated by pos * base^(-2j/d).  Returns a new array."""
    X = _f64(X).copy()
    T, d = X.shape
    _L().oracle_rope(T, d, base, pos0, _dp(X))
    return X


ROPE_INTERLEAVED = 0
ROPE_NEOX = 1


def rope_ex(X, pos, base: float = 10000.0, rotary_dim=None, style: int = ROPE_INTERLEAVED,
            inverse: bool = False):
    """Generalised RoPE (oracle_rope_ex, R19) of rows X [T, d] at positions pos [T] (int):
    the first rotary_dim (default d) channels rotate, pairs (2j, 2j+1) (style 0) or
    (j, j + rd/2) (style 1, GPT-NeoX), angle pos * base^(-2j/rd); inverse = the transpose."""
    X = _f64(X).copy()
    T, d = X.shape
    rd = d if rotary_dim is None else int(rotary_dim)
    p = np.ascontiguousarray(np.broadcast_to(np.asarray(pos, dtype=np.int64), (T,)))
    _L().oracle_rope_ex(T, d, base, rd, int(style), p.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                        1 if inverse else 0, _dp(X))
    return X


def summarize_proj(K, V, eps_, P, C: int, lam: float = 0.1, clip: float = 1.0, omega_mode: int = 0,
                   return_omega: bool = False):
    """Chunk summaries with the learned summary-key projection (oracle_summarize_proj, R17):
    k~_c = P mean(k), P [d, d]."""
    K, V, E, P = _f64(K), _f64(V), _f64(eps_), _f64(P)
    T, d = K.shape
    assert P.shape == (d, d)
    nC = T // C
    ks, vs, om = np.zeros((nC, d)), np.zeros((nC, d)), np.zeros((nC, d))
    if nC > 0:
        _L().oracle_summarize_proj(T, d, C, _dp(K), _dp(V), _dp(E), _dp(P), lam, clip, omega_mode,
                                   _dp(ks), _dp(vs), _dp(om))
    return (ks, vs, om) if return_omega else (ks, vs)


def prefill(Q, K, V, Ksum, Vsum, C: int, W: int, mode: int = SLIDING, scale: float = 1.0):
    """FlashEVA prefill of one unit: returns O [T, d] and lse [T]."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    T, d = Q.shape
    nC = T // C
    ks = _f64(Ksum).reshape(nC, d) if nC else np.zeros((1, d))
    vs = _f64(Vsum).reshape(nC, d) if nC else np.zeros((1, d))
    O = np.zeros((T, d))
    lse = np.zeros(T)
    _L().oracle_prefill(T, d, C, W, mode, scale, _dp(Q), _dp(K), _dp(V), _dp(ks), _dp(vs),
                        _dp(O), _dp(lse))
    return O, lse


def summarize_batch(K, V, E, C: int, lam: float = 0.1, clip: float = 1.0, omega_mode: int = 0):
    """K, V [BH, T, d], E [BH, nC, d] -> Ksum, Vsum [BH, nC, d] (OpenMP over units)."""
    K, V, E = _f64(K), _f64(V), _f64(E)
    BH, T, d = K.shape
    nC = T // C
    ks = np.zeros((BH, nC, d))
    vs = np.zeros((BH, nC, d))
    if nC > 0 and BH > 0:
        _L().oracle_summarize_batch(BH, T, d, C, _dp(K), _dp(V), _dp(E), lam, clip, omega_mode,
                                    _dp(ks), _dp(vs))
    return ks, vs


def prefill_batch(Q, K, V, Ksum, Vsum, C: int, W: int, mode: int = SLIDING, scale: float = 1.0):
    """[BH, T, d] inputs -> O [BH, T, d], lse [BH, T] (OpenMP over units)."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    BH, T, d = Q.shape
    nC = T // C
    ks = _f64(Ksum) if nC else np.zeros((BH, 1, d))
    vs = _f64(Vsum) if nC else np.zeros((BH, 1, d))
    O = np.zeros((BH, T, d))
    lse = np.zeros((BH, T))
    _L().oracle_prefill_batch(BH, T, d, C, W, mode, scale, _dp(Q), _dp(K), _dp(V), _dp(ks),
                              _dp(vs), _dp(O), _dp(lse))
    return O, lse


def prefill_ext_batch(Q, K, V, Ksum, Vsum, C: int, W: int, mode: int = SLIDING, scale: float = 1.0,
                      bias: float = 0.0):
    """oracle_prefill_ext over [BH, T, d]: mode 0/1 causal, 2 non-causal (R15); bias added to
    every summary logit (R16).  Returns O [BH, T, d], lse [BH, T]."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    BH, T, d = Q.shape
    nC = T // C
    ks = _f64(Ksum) if nC else np.zeros((BH, 1, d))
    vs = _f64(Vsum) if nC else np.zeros((BH, 1, d))
    O = np.zeros((BH, T, d))
    lse = np.zeros((BH, T))
    _L().oracle_prefill_ext_batch(BH, T, d, C, W, mode, scale, bias, _dp(Q), _dp(K), _dp(V), _dp(ks),
                                  _dp(vs), _dp(O), _dp(lse))
    return O, lse


def prefill_rows(Q, K, V, Ksum, Vsum, rows, C: int, W: int, mode: int = SLIDING,
                 scale: float = 1.0):
    """Selected query rows of one unit (sampled parity at full size)."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    T, d = Q.shape
    nC = T // C
    ks = _f64(Ksum) if nC else np.zeros((1, d))
    vs = _f64(Vsum) if nC else np.zeros((1, d))
    rows = np.ascontiguousarray(np.sort(np.asarray(rows, dtype=np.int64)))
    O = np.zeros((len(rows), d))
    lse = np.zeros(len(rows))
    _L().oracle_prefill_rows(T, d, C, W, mode, scale, _dp(Q), _dp(K), _dp(V), _dp(ks), _dp(vs),
                             len(rows), rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                             _dp(O), _dp(lse))
    return rows, O, lse


def backward(Q, K, V, eps_, dO, C: int, W: int, mode: int = SLIDING, scale: float = 1.0,
             lam: float = 0.1, clip: float = 1.0, omega_mode: int = 0, bias: float = 0.0):
    """Gradients (dQ, dK, dV) of L = sum(dO * O) for one unit (oracle_backward_ext; any mode,
    including NONCAUSAL, and the summary-logit bias of R16)."""
    Q, K, V, dO = _f64(Q), _f64(K), _f64(V), _f64(dO)
    T, d = Q.shape
    nC = T // C
    E = _f64(eps_).reshape(nC, d) if nC else np.zeros((1, d))
    dQ, dK, dV = np.zeros((T, d)), np.zeros((T, d)), np.zeros((T, d))
    _L().oracle_backward_ext(T, d, C, W, mode, scale, bias, lam, clip, omega_mode, _dp(Q), _dp(K),
                             _dp(V), _dp(E), _dp(dO), _dp(dQ), _dp(dK), _dp(dV))
    return dQ, dK, dV


def backward_proj(Q, K, V, eps_, P, dO, C: int, W: int, mode: int = SLIDING, scale: float = 1.0,
                  lam: float = 0.1, clip: float = 1.0, omega_mode: int = 0):
    """Gradients (dQ, dK, dV, dP) of L = sum(dO * O) for one unit with the learned summary-key
    projection P [d, d] (oracle_backward_proj, R17); dP is this unit's contribution."""
    Q, K, V, dO, P = _f64(Q), _f64(K), _f64(V), _f64(dO), _f64(P)
    T, d = Q.shape
    nC = T // C
    E = _f64(eps_).reshape(nC, d) if nC else np.zeros((1, d))
    dQ, dK, dV, dP = np.zeros((T, d)), np.zeros((T, d)), np.zeros((T, d)), np.zeros((d, d))
    _L().oracle_backward_proj(T, d, C, W, mode, scale, lam, clip, omega_mode, _dp(Q), _dp(K), _dp(V),
                              _dp(E), _dp(P), _dp(dO), _dp(dQ), _dp(dK), _dp(dV), _dp(dP))
    return dQ, dK, dV, dP


def backward_batch(Q, K, V, E, dO, C: int, W: int, mode: int = SLIDING, scale: float = 1.0,
                   lam: float = 0.1, clip: float = 1.0, omega_mode: int = 0, bias: float = 0.0):
    Q, K, V, dO = _f64(Q), _f64(K), _f64(V), _f64(dO)
    BH, T, d = Q.shape
    nC = T // C
    E = _f64(E) if nC else np.zeros((BH, 1, d))
    dQ, dK, dV = np.zeros_like(Q), np.zeros_like(Q), np.zeros_like(Q)
    _L().oracle_backward_ext_batch(BH, T, d, C, W, mode, scale, bias, lam, clip, omega_mode,
                                   _dp(Q), _dp(K), _dp(V), _dp(E), _dp(dO), _dp(dQ), _dp(dK),
                                   _dp(dV))
    return dQ, dK, dV


class Cache:
    """Streaming decode state of one unit (ring of W tokens + summary list)."""

    def __init__(self, d: int, C: int, W: int, mode: int = SLIDING, cap: int = 1024,
                 scale: float = 1.0, lam: float = 0.1, clip: float = 1.0, omega_mode: int = 0):
        self.d, self.C, self.cap = d, C, cap
        self._p = _L().oracle_cache_new(d, C, W, mode, cap, scale, lam, clip, omega_mode)

    def __del__(self):
        if getattr(self, "_p", None):
            _L().oracle_cache_free(self._p)
            self._p = None

    @property
    def pos(self) -> int:
        return _L().oracle_cache_pos(self._p)

    def append(self, k, v, eps_chunk) -> int:
        k, v, e = _f64(k), _f64(v), _f64(eps_chunk)
        return _L().oracle_cache_append(self._p, _dp(k), _dp(v), _dp(e))

    def decode(self, q):
        q = _f64(q)
        o = np.zeros(self.d)
        lse = _L().oracle_cache_decode(self._p, _dp(q), _dp(o))
        return o, lse

    def summaries(self):
        n = self.pos // self.C
        ks = np.ctypeslib.as_array(_L().oracle_cache_sum_k(self._p), shape=(self.cap * self.d,))
        vs = np.ctypeslib.as_array(_L().oracle_cache_sum_v(self._p), shape=(self.cap * self.d,))
        return ks[: n * self.d].reshape(n, self.d).copy(), vs[: n * self.d].reshape(n, self.d).copy()
