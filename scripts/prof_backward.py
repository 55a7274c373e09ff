"""One eva_attn_backward at configs[2]'s per-GPU shape (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
B, H, T, d, C, W = (int(x) for x in sys.argv[1:7]) if len(sys.argv) > 6 else (8, 32, 8192, 128, 64, 256)
cfg = eva.make_config(B, H, T, d, C, W, dtype=torch.bfloat16, seed=1)
Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=1, device="cuda")
(dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=2, device="cuda")
O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
ws = torch.empty(eva.eva_backward_workspace_bytes(cfg), dtype=torch.uint8, device="cuda")
for _ in range(2):
    eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws)
torch.cuda.synchronize()
