"""Backward main-pass cost model: time eva_attn_backward's kernels for several windows (local
work items of 128 keys see (128 + W) / 64 query tiles) to separate per-item from per-step cost."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
B, H, T, d, C = 4, 32, 8192, 128, 64
out = []
for W in (64, 128, 256, 512, 1024):
    cfg = eva.make_config(B, H, T, d, C, W, dtype=torch.bfloat16, seed=1)
    Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=1, device="cuda")
    (dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=2, device="cuda")
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    ws = torch.empty(eva.eva_backward_workspace_bytes(cfg), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws)
    b.record(); torch.cuda.synchronize()
    nq = T // 64
    local_items = T // 128
    local_steps = sum(min(nq, (min(T - 1, (((128 * t + 127) // C) + W // C) * C - 1)) // 64 + 1) - 2 * t
                      for t in range(local_items))
    out.append({"W": W, "ms": a.elapsed_time(b) / 5, "local_items_per_unit": local_items,
                "local_steps_per_unit": local_steps})
    print(json.dumps(out[-1]))
