"""Quick probe of the tcgen05 prefill against the SIMT kernel and the oracle (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import eva_inputs, oracle
import paper_2511_00576_b200 as eva

KERNEL = sys.argv[1] if len(sys.argv) > 1 else None
def f64(t): return t.detach().float().cpu().double().numpy()
for (B, H, T, d, C, W, mode) in [(1, 1, 128, 64, 64, 128, "sliding"), (1, 2, 515, 64, 64, 128, "sliding"),
                                 (1, 2, 700, 128, 64, 256, "sliding"), (1, 1, 130, 64, 16, 16, "block"),
                                 (1, 1, 1, 128, 4, 8, "sliding"), (2, 3, 1100, 64, 32, 96, "sliding"),
                                 (1, 3, 300, 128, 16, 32, "block"), (1, 8, 4096, 128, 64, 256, "sliding")]:
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=2, device="cuda")
    O1, l1, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V, simt=True)
    O2, l2, _, _ = eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, kernel=KERNEL)
    torch.cuda.synchronize()
    E = oracle.eps_units(cfg.seed, 0, 0, B * H, T // C, d)
    rk, rv = oracle.summarize_batch(f64(K), f64(V), E, C)
    rO, rl = oracle.prefill_batch(f64(Q), f64(K), f64(V), rk, rv, C, W, 0 if mode == "sliding" else 1, cfg.scale)
    e_simt = np.abs(f64(O1) - rO).max(); e_tc = np.abs(f64(O2) - rO).max()
    el = np.abs(f64(l2) - rl).max()
    bad = np.argwhere(np.abs(f64(O2) - rO).max(-1) > 2e-2)
    print(f"T={T} d={d} C={C} W={W} {mode}: simt {e_simt:.2e}  tc {e_tc:.2e} lse {el:.2e} bad rows {bad[:8].tolist()} n_bad={len(bad)}", flush=True)
