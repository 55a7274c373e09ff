"""Prefill (summaries provided) at configs[2] and the configs[4] compute-bound cells, for the
launch-order experiment (EVA_PREFILL_REVERSE) -- dev tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
flush = torch.empty(512 << 18, device="cuda")
for (B, H, T, d, C, W) in [(8, 32, 8192, 128, 64, 256), (1, 32, 65536, 128, 32, 512), (1, 32, 65536, 128, 64, 512),
                           (1, 32, 131072, 128, 32, 512), (1, 32, 131072, 128, 64, 512), (1, 32, 131072, 128, 128, 512)]:
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    O = torch.empty_like(Q)
    f = lambda: eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O, summaries_provided=True)
    for _ in range(2): f()
    ts = []
    for _ in range(7):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"T={T} C={C} W={W}: {ts[3]:.3f} ms", flush=True)
    del Q, K, V, O, ks, vs
