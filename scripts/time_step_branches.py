"""configs[1] step as CUDA graphs (dev tool): the whole step, and each branch after the summaries
alone -- which branch sets the step time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva

B, H, T, d, C, W = 1, 16, 2048, 64, 64, 128
BH, nC = B * H, T // C
cfg = eva.make_config(B, H, T, d, C, W)
Q, K, V = eva_inputs.qkv(0, BH, T, d, torch.bfloat16, seed=0, device="cuda")
Ks = torch.empty(BH, nC, d, dtype=torch.bfloat16, device="cuda"); Vs = torch.empty_like(Ks)
O = torch.empty_like(Q); lse = torch.empty(BH, T, device="cuda")
qn, kn, vn = (x[0] for x in eva_inputs.decode_tokens(0, BH, 1, d, torch.bfloat16, seed=1, device="cuda"))
cache = eva.DecodeCache(cfg, nC + 2, device="cuda")
od = torch.empty(BH, d, dtype=torch.bfloat16, device="cuda")
s = torch.cuda.current_stream(); side = torch.cuda.Stream()
flush = torch.empty(512 << 18, device="cuda")

def summ(): eva.eva_summarize(cfg, K, V, Ksum=Ks, Vsum=Vs)
def pre(): eva.eva_attn_prefill(cfg, Q, K, V, Ksum=Ks, Vsum=Vs, summaries_provided=True, O=O, lse=lse)
def dec():
    cache.c.pos = 0
    cache.eva_cache_load(K, V, Ks, Vs)
    cache.eva_decode_step(qn, kn, vn, O=od, want_lse=False)
def full():
    summ(); side.wait_stream(s)
    with torch.cuda.stream(side):
        dec()
    pre(); s.wait_stream(side)
variants = {"full step": full, "summarize + prefill": lambda: (summ(), pre()),
            "summarize + cache_load + decode_step": lambda: (summ(), dec()),
            "summarize": summ, "prefill": pre, "cache_load + decode_step": dec}
for name, f in variants.items():
    for _ in range(3): f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    for _ in range(5): g.replay()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
    for a, b in ev:
        flush.zero_(); a.record(); g.replay(); b.record()
    torch.cuda.synchronize()
    print(f"{name}: {sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3:.2f} us", flush=True)
