"""Time RoPE + prefill at configs[1] and configs[2]'s per-GPU shapes: the in-kernel RoPE prefill
(eva_attn_prefill_rope, summaries provided / computed) against the two-pass path (rotated Q, K
written by eva_rope_summarize, then eva_attn_prefill), and the plain prefill (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva

def timeit(f, flush, n=20):
    for _ in range(3):
        f()
    ts = []
    for _ in range(n):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[n // 2] * 1e3

flush = torch.empty(512 << 18, device="cuda")
for (B, H, T, d, C, W) in [(8, 32, 8192, 128, 64, 256), (1, 16, 2048, 64, 64, 128)]:
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
    Qr, Kr, ks, vs = eva.eva_rope_summarize(cfg, Q, K, V)
    O = torch.empty_like(Q)
    runs = {
        "plain prefill (summaries provided)": lambda: eva.eva_attn_prefill(cfg, Qr, Kr, V, Ksum=ks, Vsum=vs, O=O, summaries_provided=True),
        "rope in-kernel (summaries provided)": lambda: eva.eva_attn_prefill_rope(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O),
        "rope in-kernel + rope summaries": lambda: eva.eva_attn_prefill_rope(cfg, Q, K, V, O=O),
        "two-pass: rope_summarize + prefill": lambda: (eva.eva_rope_summarize(cfg, Q, K, V), eva.eva_attn_prefill(cfg, Qr, Kr, V, Ksum=ks, Vsum=vs, O=O, summaries_provided=True)),
    }
    for name, f in runs.items():
        print(f"T={T} d={d} {name}: {timeit(f, flush):.1f} us", flush=True)
