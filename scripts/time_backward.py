"""Time eva_attn_backward (and its three kernels) with CUDA events on the launching stream."""
import json
import sys

import torch

sys.path.insert(0, "/root/repo")
import eva_inputs  # noqa: E402
import paper_2511_00576_b200 as eva  # noqa: E402


def run(B, H, T, d, C, W, reps=5):
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
    for _ in range(reps):
        eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fa.record()
    for _ in range(reps):
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True)
    fb.record()
    torch.cuda.synchronize()
    return {"B": B, "H": H, "T": T, "d": d, "C": C, "W": W, "bwd_ms": ms,
            "fwd_ms": fa.elapsed_time(fb) / reps, "tokens_per_s_bwd": B * T / ms * 1e3}


if __name__ == "__main__":
    out = [run(1, 16, 2048, 64, 64, 128), run(8, 32, 8192, 128, 64, 256, reps=2)]
    for r in out:
        print(json.dumps(r))
