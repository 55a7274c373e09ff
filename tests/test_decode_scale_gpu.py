"""Decode at the benched scale and across split-count changes, against the fp64 oracle.

* configs[3]'s shape (d = 128, C = 64, W = 256) with >= 1024 units and ~700 visible entries
  per query: the two-launch path of eva_decode_step (append kernel, then the split-K decode)
  and eva_decode_step_ragged at per-unit positions, sampled units checked against
  oracle.prefill_rows on the visible set the cache holds (summary rows c < nsum(n) and the
  ring positions [lo(n), n], Eq.12 for one query) and the completed chunk's summary
  against oracle.summarize (Eq.10, Eq.15).
* a long token-by-token generation at 1-2 units where the split count (E / 64 splits,
  E = nsum + |local|) changes between values > 1 at chunk boundaries, every step against the
  oracle's streaming cache: the split-K merge counters must sit at a fixed workspace offset.

The ring and summary rows are seeded N(0, 1) values written straight into the cache (the
decode's work does not depend on how they were produced); the oracle sees the same values.
"""
import numpy as np
import pytest
import torch

import eva_inputs
import oracle

pytestmark = pytest.mark.gpu

TOL = 2e-2  # bf16 path, north_star


@pytest.fixture(scope="module")
def eva(cuda_device):
    import paper_2511_00576_b200 as eva
    return eva


def f64(t):
    return t.detach().float().cpu().double().numpy()


def _fill_cache(cache, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    for t in (cache.ring_k, cache.ring_v, cache.sum_k, cache.sum_v):
        t.copy_(torch.randn(t.shape, generator=g, device="cuda", dtype=torch.float32))


def _oracle_row(cfg, ring_k, ring_v, sum_k, sum_v, extra, q, n, u):
    """Oracle row n of unit u from the cache's content: K/V at positions [lo(n), n] from the
    ring (slot p mod W) or from `extra` {p: (k, v)} (tokens appended by the step), summaries
    c < nsum(n) from sum_k/sum_v (rows the caller has already fixed up)."""
    C, W, d = cfg.chunk, cfg.window, cfg.d_head
    lo, ns = oracle.mask(n, C, W, oracle.SLIDING)
    T = n + 1
    K = np.zeros((T, d))
    V = np.zeros((T, d))
    for p in range(lo, n + 1):
        if p in extra:
            K[p], V[p] = extra[p]
        else:
            K[p], V[p] = ring_k[p % W], ring_v[p % W]
    Q = np.zeros((T, d))
    Q[n] = q
    nC = T // C
    ks = np.zeros((max(nC, 1), d))
    vs = np.zeros((max(nC, 1), d))
    ks[:ns], vs[:ns] = sum_k[:ns], sum_v[:ns]
    _, O, lse = oracle.prefill_rows(Q, K, V, ks[:nC], vs[:nC], [n], C, W, oracle.SLIDING, cfg.scale)
    return O[0], lse[0]


def test_decode_step_1024_units_two_launch_sampled(eva):
    """1024 units (eva_decode_step's two-launch path), context ~30k: ~700 visible entries,
    16 steps crossing a chunk completion; units 0, 517, 1023 against the oracle."""
    BH, d, C, W = 1024, 128, 64, 256
    P0 = 30000 - 1
    steps = 18                     # positions 29999 .. 30016: chunk 468 completes at 30015
    cap = (P0 + steps) // C + 2
    cfg = eva.make_config(1, BH, 0, d, C, W, seed=61)
    cache = eva.DecodeCache(cfg, cap, device="cuda")
    _fill_cache(cache, 62)
    cache.c.pos = P0
    q, k, v = eva_inputs.decode_tokens(0, BH, steps, d, torch.bfloat16, seed=63, device="cuda")
    sample = (0, 517, 1023)
    ring0 = {u: (f64(cache.ring_k[u]), f64(cache.ring_v[u])) for u in sample}
    sums0 = {u: (f64(cache.sum_k[u]), f64(cache.sum_v[u])) for u in sample}
    outs = []
    for t in range(steps):
        o, lse = cache.eva_decode_step(q[t], k[t], v[t])
        outs.append((f64(o), f64(lse)))
    assert cache.pos == P0 + steps
    E_all = {u: oracle.eps(cfg.seed, cfg.layer, u, cap, d) for u in sample}
    for u in sample:
        rk_ring, rv_ring = ring0[u]
        sk, sv = sums0[u][0].copy(), sums0[u][1].copy()
        extra = {}
        for t in range(steps):
            n = P0 + t
            extra[n] = (f64(k[t, u]), f64(v[t, u]))
            if (n + 1) % C == 0:  # the step summarised chunk (n+1)/C - 1 from its C rows
                c = (n + 1) // C - 1
                Kc = np.stack([extra[p][0] if p in extra else rk_ring[p % W] for p in range(c * C, c * C + C)])
                Vc = np.stack([extra[p][1] if p in extra else rv_ring[p % W] for p in range(c * C, c * C + C)])
                rks, rvs = oracle.summarize(Kc, Vc, E_all[u][c:c + 1], C)
                assert np.max(np.abs(f64(cache.sum_k[u, c]) - rks[0])) <= TOL
                assert np.max(np.abs(f64(cache.sum_v[u, c]) - rvs[0])) <= TOL
                sk[c], sv[c] = rks[0], rvs[0]
            ro, rl = _oracle_row(cfg, rk_ring, rv_ring, sk, sv, extra, f64(q[t, u]), n, u)
            lo, ns = oracle.mask(n, C, W, oracle.SLIDING)
            assert ns + (n - lo + 1) >= 650
            assert np.max(np.abs(outs[t][0][u] - ro)) <= TOL, (u, t)
            assert abs(outs[t][1][u] - rl) <= TOL, (u, t)


def test_ragged_decode_1024_units_sampled(eva):
    """eva_decode_step_ragged with 1024 units at per-unit positions 28k..30k (some completing
    a chunk this step): sampled units' outputs, summaries and advanced positions."""
    BH, d, C, W = 1024, 128, 64, 256
    cap = 30000 // C + 4
    cfg = eva.make_config(1, BH, 0, d, C, W, seed=71)
    cache = eva.DecodeCache(cfg, cap, device="cuda")
    _fill_cache(cache, 72)
    g = np.random.default_rng(73)
    pos_h = g.integers(28000, 30000, size=BH).astype(np.int64)
    sample = (0, 1, 400, 777, 1023)
    pos_h[1] = 64 * 460 - 1          # completes chunk 459 this step
    pos_h[777] = 64 * 450 - 1        # completes chunk 449
    pos = torch.tensor(pos_h, device="cuda")
    q, k, v = eva_inputs.decode_tokens(0, BH, 2, d, torch.bfloat16, seed=74, device="cuda")
    ring0 = {u: (f64(cache.ring_k[u]), f64(cache.ring_v[u])) for u in sample}
    sums0 = {u: (f64(cache.sum_k[u]), f64(cache.sum_v[u])) for u in sample}
    outs = []
    for t in range(2):
        o, lse = cache.eva_decode_step_ragged(pos, q[t], k[t], v[t])
        outs.append((f64(o), f64(lse)))
    assert pos.cpu().numpy().tolist() == (pos_h + 2).tolist()
    for u in sample:
        rk_ring, rv_ring = ring0[u]
        sk, sv = sums0[u][0].copy(), sums0[u][1].copy()
        E = oracle.eps(cfg.seed, cfg.layer, u, cap, d)
        extra = {}
        for t in range(2):
            n = int(pos_h[u]) + t
            extra[n] = (f64(k[t, u]), f64(v[t, u]))
            if (n + 1) % C == 0:
                c = (n + 1) // C - 1
                Kc = np.stack([extra[p][0] if p in extra else rk_ring[p % W] for p in range(c * C, c * C + C)])
                Vc = np.stack([extra[p][1] if p in extra else rv_ring[p % W] for p in range(c * C, c * C + C)])
                rks, rvs = oracle.summarize(Kc, Vc, E[c:c + 1], C)
                assert np.max(np.abs(f64(cache.sum_k[u, c]) - rks[0])) <= TOL
                assert np.max(np.abs(f64(cache.sum_v[u, c]) - rvs[0])) <= TOL
                sk[c], sv[c] = rks[0], rvs[0]
            ro, rl = _oracle_row(cfg, rk_ring, rv_ring, sk, sv, extra, f64(q[t, u]), n, u)
            assert np.max(np.abs(outs[t][0][u] - ro)) <= TOL, (u, t)
            assert abs(outs[t][1][u] - rl) <= TOL, (u, t)


@pytest.mark.parametrize("BH,step_fn", [(1, "step"), (2, "append_decode")])
def test_decode_split_count_changes_across_chunks(eva, BH, step_fn):
    """Token-by-token decode from a 4000-token prompt for 300 tokens (W = 256, C = 64): the
    split count E/64 moves between 4 and 5 at every chunk boundary; every step equals the
    oracle's streaming cache (a merge counter overlapping the previous call's partials
    would leave O unwritten)."""
    d, C, W, T0, G = 128, 64, 256, 4000, 300
    cap = (T0 + G) // C + 1
    cfg = eva.make_config(1, BH, T0, d, C, W, seed=81)
    Q, K, V = eva_inputs.qkv(0, BH, T0, d, torch.bfloat16, seed=82, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    cache = eva.DecodeCache(cfg, cap, device="cuda")
    cache.eva_cache_load(K, V, ks, vs)
    q, k, v = eva_inputs.decode_tokens(0, BH, G, d, torch.bfloat16, seed=83, device="cuda")
    orc = [oracle.Cache(d, C, W, oracle.SLIDING, cap=cap, scale=cfg.scale) for _ in range(BH)]
    E = oracle.eps_units(cfg.seed, cfg.layer, 0, BH, cap + 1, d)
    Kh, Vh = f64(K), f64(V)
    for u in range(BH):
        for t in range(T0):
            assert orc[u].append(Kh[u, t], Vh[u, t], E[u, t // C]) == 0
    splits = set()
    worst = 0.0
    for t in range(G):
        cache.c.pos += 1
        nb = cache.workspace_bytes()
        cache.c.pos -= 1
        pad = (BH + 3) // 4 * 4 * 4
        splits.add((nb - pad) // (BH * (d + 2) * 4) if nb else 1)
        if step_fn == "step":
            o, lse = cache.eva_decode_step(q[t], k[t], v[t])
        else:
            cache.eva_cache_append(k[t], v[t])
            o, lse = cache.eva_attn_decode(q[t])
        of, lf = f64(o), f64(lse)
        for u in range(BH):
            assert orc[u].append(f64(k[t, u]), f64(v[t, u]), E[u, (T0 + t) // C]) == 0
            ro, rl = orc[u].decode(f64(q[t, u]))
            err = max(np.max(np.abs(of[u] - ro)), abs(lf[u] - rl))
            assert err <= TOL, (t, u, err)
            worst = max(worst, err)
    multi = sorted(s for s in splits if s > 1)
    assert len(multi) >= 2, splits
