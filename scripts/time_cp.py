"""Context-parallel prefill on one B200: per-rank kernel time of each shard (summarize_range +
prefill_range) vs the single-call prefill, and the exchange volume per rank (dev tool).
    python scripts/time_cp.py [T] [world ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
from paper_2511_00576_b200.context_parallel import seq_shards

T = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
worlds = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
B, H, d, C, W = 1, 32, 128, 64, 256
cfg = eva.make_config(B, H, T, d, C, W)
Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
flush = torch.empty(512 << 18, device="cuda")


def timed(fn, reps=5):
    for _ in range(2): fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


full = timed(lambda: eva.eva_attn_prefill(cfg, Q, K, V))
out = {"T": T, "B": B, "H": H, "d": d, "C": C, "W": W, "single_gpu_ms": full, "worlds": []}
Ks, Vs = eva.eva_summarize(cfg, K, V)
for world in worlds:
    sh = seq_shards(T, world, C, W)
    per = []
    for s in sh:
        sub = eva.make_config(B, H, s.q1 - s.q0, d, C, W)
        Kl, Vl = K[:, s.q0:s.q1].contiguous(), V[:, s.q0:s.q1].contiguous()
        Ql = Q[:, s.q0:s.q1].contiguous()
        Kc, Vc = K[:, s.k0:s.q1].contiguous(), V[:, s.k0:s.q1].contiguous()
        ns = s.q1 // C
        t_sum = timed(lambda: eva.eva_summarize_range(sub, s.q0 // C, Kl, Vl))
        t_pre = timed(lambda: eva.eva_attn_prefill_range(cfg, s.q0, s.k0, Ql, Kc, Vc, Ks[:, :ns].contiguous(),
                                                         Vs[:, :ns].contiguous()))
        exch = B * H * ((T // C) * d * 2 * 2 + (s.q0 - s.k0) * d * 2 * 2)   # summaries in + halo in, bytes
        per.append({"rank": s.rank, "q0": s.q0, "q1": s.q1, "summarize_ms": t_sum, "prefill_ms": t_pre,
                    "exchange_bytes_in": exch})
    mx = max(p["summarize_ms"] + p["prefill_ms"] for p in per)
    out["worlds"].append({"world": world, "max_rank_kernel_ms": mx, "speedup_vs_1gpu": full / mx,
                          "ranks": per})
    print(f"world {world}: max per-rank kernel time {mx:.3f} ms vs single GPU {full:.3f} ms "
          f"(x{full / mx:.2f}); exchange in per rank <= {max(p['exchange_bytes_in'] for p in per) / 1e6:.2f} MB")
print(json.dumps(out))
