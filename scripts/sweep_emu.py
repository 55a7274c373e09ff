"""configs[4] compute-bound cells with the tile kernel's exp2 split (EVA_SOFTMAX_EMU) on / off (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
import bench
peaks = bench.load_peaks()
for (T, C, W) in [(16384, 64, 512), (65536, 32, 512), (131072, 32, 512), (131072, 64, 512), (8192, 64, 256)]:
    H, d = (32, 128) if T != 8192 else (256, 128)
    cfg = eva.make_config(1, H, T, d, C, W)
    Q, K, V = eva_inputs.qkv(0, H, T, d, torch.bfloat16, seed=0, device="cuda")
    ks, vs = eva.eva_summarize(cfg, K, V)
    O = torch.empty_like(Q)
    f = lambda: eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O)
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    pf = bench.prefill_flops(H, T, d, C, W)
    print(f"EMU={os.environ.get('EVA_SOFTMAX_EMU', '-1')} T={T} C={C} W={W}: {ms:.3f} ms  tensor_frac {pf / (ms / 1e3) / 1e12 / peaks['bf16']:.3f}")
    del Q, K, V, O, ks, vs
    torch.cuda.empty_cache()
