"""The bench's e2e step (configs[1], pinned host buffers) broken down (dev tool): device time of
the whole step, of the H2D alone, of the D2H alone, and host-side enqueue time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
B, H, T, d, C, W = 1, 16, 2048, 64, 64, 128
BH = B * H
cfg = eva.make_config(B, H, T, d, C, W)
Q, K, V = eva_inputs.qkv(0, BH, T, d, torch.bfloat16, seed=0, device="cuda")
hQ, hK, hV = (x.cpu().pin_memory() for x in (Q, K, V))
hO = torch.empty(BH, T, d, dtype=torch.bfloat16).pin_memory()
hp = eva.HostPrefill(cfg, max_slices=16)
qn, kn, vn = (x[0] for x in eva_inputs.decode_tokens(0, BH, 1, d, torch.bfloat16, seed=1, device="cuda"))
cache = eva.DecodeCache(cfg, T // C + 2, device="cuda")
hOd = torch.empty(BH, d, dtype=torch.bfloat16).pin_memory()
s = torch.cuda.current_stream()
def step(n_slices=1):
    cache.c.pos = 0
    hp(hQ, hK, hV, hO, n_slices=n_slices)
    cache.eva_cache_load(hp.K, hp.V, hp.Ksum, hp.Vsum)
    od, _ = cache.eva_decode_step(qn, kn, vn, want_lse=False)
    hOd.copy_(od, non_blocking=True)
for ns in (1, 2, 3, 4, 8):
    for _ in range(10): step(ns)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    for _ in range(20): step(ns)
    b.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"n_slices={ns}: device {a.elapsed_time(b) / 20 * 1e3:.0f} us/step, host enqueue {(t1 - t0) / 20 * 1e6:.0f} us/step, wall {(t2 - t0) / 20 * 1e6:.0f} us/step", flush=True)
dQ = torch.empty_like(Q)
for nm, f in (("H2D 12 MB", lambda: (dQ.copy_(hQ, non_blocking=True), hp.K.copy_(hK, non_blocking=True), hp.V.copy_(hV, non_blocking=True))),
              ("D2H 4 MB", lambda: hO.copy_(hp.O, non_blocking=True))):
    for _ in range(5): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    print(f"{nm}: {a.elapsed_time(b) / 20 * 1e3:.0f} us", flush=True)
