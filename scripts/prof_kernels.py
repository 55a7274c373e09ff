"""Launch one hot-path kernel at a BASELINE config a few times (for ncu -k captures).

    python scripts/prof_kernels.py prefill_configs2|prefill_configs1|summarize_configs2|decode_configs3 [reps]

(BASELINE.json configs are 0-indexed: configs[1] = B=1,H=16,T=2048,d=64; configs[2] = B=8,H=32,
T=8192,d=128 per GPU; configs[3] = the decode batch.)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import eva_inputs
import paper_2511_00576_b200 as eva

what = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda:0")
if what in ("prefill_ropeq_configs2", "summarize_rope_configs2"):
    # the Q-only RoPE prefill (EVA_ROPE_K_ROTATED) / the bulk summariser rotating the landed keys
    B, H, T, d, C, W = 8, 32, 8192, 128, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device=dev)
    Kr = eva.eva_rope(cfg, K)
    ks, vs = eva.eva_summarize(cfg, Kr, V)
    O = torch.empty_like(Q)
    for _ in range(reps):
        if what == "prefill_ropeq_configs2":
            eva.eva_attn_prefill_rope(cfg, Q, Kr, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, k_rotated=True)
        else:
            eva.eva_attn_prefill_rope(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O)
elif what == "prefill_rope_configs2":  # RoPE inside the tcgen05 prefill (eva_attn_prefill_rope)
    B, H, T, d, C, W = 8, 32, 8192, 128, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device=dev)
    _, _, ks, vs = eva.eva_rope_summarize(cfg, Q, K, V)
    O = torch.empty_like(Q)
    for _ in range(reps):
        eva.eva_attn_prefill_rope(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O)
elif what in ("prefill_configs2", "summarize_configs2", "prefill_configs1"):
    if what == "prefill_configs1":
        B, H, T, d, C, W = 1, 16, 2048, 64, 64, 128
    else:
        B, H, T, d, C, W = 8, 32, 8192, 128, 64, 256
    cfg = eva.make_config(B, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device=dev)
    ks, vs = eva.eva_summarize(cfg, K, V)
    O = torch.empty_like(Q)
    lse = torch.empty(B * H, T, device=dev)
    for _ in range(reps):
        if what == "summarize_configs2":
            eva.eva_summarize(cfg, K, V, Ksum=ks, Vsum=vs)
        else:
            eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, lse=lse,
                                 kernel=os.environ.get("EVA_PROF_KERNEL") or None)
elif what == "decode_ragged_configs3":
    BH, d, C, W, ctx = 256 * 32, 128, 64, 256, 32768
    cfg = eva.make_config(256, 32, 0, d, C, W)
    cache = eva.DecodeCache(cfg, (ctx + 64) // C + 16, device=dev)
    for t in (cache.ring_k, cache.ring_v, cache.sum_k, cache.sum_v):
        t.normal_()
    cache.c.pos = ctx
    pos = ctx - 64 * (torch.arange(BH, device=dev, dtype=torch.int64) % 64)
    q = torch.randn(BH, d, device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)
    for _ in range(reps):
        cache.eva_decode_step_ragged(pos, q, q, q, O=o, want_lse=False)
elif what == "decode_configs3":
    BH, d, C, W, ctx = 256 * 32, 128, 64, 256, 32768
    cfg = eva.make_config(256, 32, 0, d, C, W)
    cache = eva.DecodeCache(cfg, ctx // C + 16, device=dev)
    for t in (cache.ring_k, cache.ring_v, cache.sum_k, cache.sum_v):
        t.normal_()
    cache.c.pos = ctx
    q = torch.randn(BH, d, device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)
    for _ in range(reps):
        cache.eva_cache_append(q, q)
        cache.eva_attn_decode(q, O=o, want_lse=False)
torch.cuda.synchronize()
print("done", what)
