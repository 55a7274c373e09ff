"""Time the prefill step (summaries + attention) at configs[1] and configs[2]'s per-GPU shapes:
fused (EVA_SUMMARIES_FUSED, one launch), separate (eva_summarize + attention, two launches)
and the attention alone with the summaries provided (dev tool).  L2 flushed before each step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
shapes = [(8, 32, 8192, 128, 64, 256), (1, 16, 2048, 64, 64, 128)]
for (B, H, T, d, C, W) in shapes:
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    O = torch.empty_like(Q)
    flush = torch.empty(512 << 18, device="cuda")
    runs = {
        "fused": lambda: eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O, kernel="fused"),
        "separate": lambda: eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O, kernel="separate"),
        "attention_only": lambda: eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O,
                                                       summaries_provided=True),
        "summarize_only": lambda: eva.eva_summarize(cfg, K, V, Ksum=ks, Vsum=vs),
    }
    for name in sys.argv[1:] or list(runs):
        f = runs[name]
        for _ in range(3):
            f()
        ts = []
        for _ in range(20):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        nC = T // C
        gb = B * H * (4 * T * d * 2 + 2 * nC * d * 2 + 4 * T) / 1e9
        if name == "summarize_only":
            gb = B * H * (2 * T * d * 2 + 2 * nC * d * 2) / 1e9
        print(f"T={T} d={d} {name}: median {ts[10]*1e3:.1f} us  min {ts[0]*1e3:.1f} us  -> {gb / (ts[10] / 1e3):.0f} GB/s")
