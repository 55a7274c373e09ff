"""summarize -> prefill with and without EVA_PREFILL_OVERLAP, eager and as a CUDA graph (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
for (B, H, T, d, C, W) in [(1, 16, 2048, 64, 64, 128), (8, 32, 8192, 128, 64, 256)]:
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    O = torch.empty_like(Q); lse = torch.empty(B * H, T, device="cuda")
    flush = torch.empty(512 << 18, device="cuda")
    def pair(ov):
        eva.eva_summarize(cfg, K, V, Ksum=ks, Vsum=vs)
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, lse=lse, overlap=ov)
    for ov in (False, True):
        for mode in ("eager", "graph"):
            if mode == "graph":
                g = torch.cuda.CUDAGraph()
                pair(ov); torch.cuda.synchronize()
                with torch.cuda.graph(g):
                    pair(ov)
                run = g.replay
            else:
                run = lambda: pair(ov)
            for _ in range(3): run()
            ts = []
            for _ in range(20):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); run(); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            ts.sort()
            print(f"T={T} d={d} overlap={ov} {mode}: median {ts[10]:.1f} us  min {ts[0]:.1f} us")
