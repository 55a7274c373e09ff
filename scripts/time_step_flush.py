"""configs[1] step graph under different L2 flushes (dev tool): write-flush (the bench's), read-flush,
none; and a one-kernel graph as the floor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
B, H, T, d, C, W = 1, 16, 2048, 64, 64, 128
BH, nC = 16, T // C
cfg = eva.make_config(B, H, T, d, C, W)
Q, K, V = eva_inputs.qkv(0, BH, T, d, torch.bfloat16, seed=0, device="cuda")
Ks = torch.empty(BH, nC, d, dtype=torch.bfloat16, device="cuda"); Vs = torch.empty_like(Ks)
O = torch.empty_like(Q); lse = torch.empty(BH, T, device="cuda")
qn, kn, vn = (x[0] for x in eva_inputs.decode_tokens(0, BH, 1, d, torch.bfloat16, seed=1, device="cuda"))
cache = eva.DecodeCache(cfg, nC + 2, device="cuda")
od = torch.empty(BH, d, dtype=torch.bfloat16, device="cuda")
s = torch.cuda.current_stream(); side = torch.cuda.Stream()
buf = torch.empty(512 << 18, device="cuda")
acc = torch.empty(1, device="cuda")
x = torch.empty(256, device="cuda")
def step():
    cache.c.pos = 0
    eva.eva_summarize(cfg, K, V, Ksum=Ks, Vsum=Vs)
    side.wait_stream(s)
    with torch.cuda.stream(side):
        cache.eva_cache_load(K, V, Ks, Vs)
        cache.eva_decode_step(qn, kn, vn, O=od, want_lse=False)
    eva.eva_attn_prefill(cfg, Q, K, V, Ksum=Ks, Vsum=Vs, summaries_provided=True, O=O, lse=lse)
    s.wait_stream(side)
for name, f in (("step", step), ("tiny", lambda: x.fill_(1.0))):
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    for _ in range(5): g.replay()
    for fl in ("write", "read", "none"):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
        for a, b in ev:
            if fl == "write": buf.zero_()
            elif fl == "read": torch.sum(buf, dim=0, out=acc[0]) if False else acc.copy_(buf.sum().reshape(1))
            a.record(); g.replay(); b.record()
        torch.cuda.synchronize()
        print(f"{name} flush={fl}: {sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3:.2f} us", flush=True)
