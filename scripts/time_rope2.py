"""RoPE prefill variants at configs[2] (dev tool): full in-kernel, K pre-rotated (Q-only kernel),
two-pass; summaries included."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
flush = torch.empty(512 << 18, device="cuda")
B, H, T, d, C, W = 8, 32, 8192, 128, 64, 256
cfg = eva.make_config(B, H, T, d, C, W)
Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
Qr, Kr, ks, vs = eva.eva_rope_summarize(cfg, Q, K, V)
O = torch.empty_like(Q)
def t(f, n=10):
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[n // 2]
print("plain prefill", t(lambda: eva.eva_attn_prefill(cfg, Qr, Kr, V, Ksum=ks, Vsum=vs, O=O, summaries_provided=True)))
print("Q-only rope prefill (summaries provided)", t(lambda: eva.eva_attn_prefill_rope(cfg, Q, Kr, V, Ksum=ks, Vsum=vs, O=O, summaries_provided=True, k_rotated=True)))
print("full rope prefill (summaries provided)", t(lambda: eva.eva_attn_prefill_rope(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O, summaries_provided=True)))
print("eva_rope K", t(lambda: eva.eva_rope(cfg, K, out=Kr)))
print("step: rope K + summarize + Q-only prefill", t(lambda: (eva.eva_rope(cfg, K, out=Kr), eva.eva_attn_prefill_rope(cfg, Q, Kr, V, Ksum=ks, Vsum=vs, O=O, k_rotated=True))))
print("step: full in-kernel", t(lambda: eva.eva_attn_prefill_rope(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O)))
