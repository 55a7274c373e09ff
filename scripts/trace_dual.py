"""Timeline of CTA 0 of the dual prefill kernel (prefill_dual.cu; dev tool).
    python scripts/trace_dual.py B H T d C W [max_events]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
from paper_2511_00576_b200 import _native as N

B, H, T, d, C, W = (int(x) for x in sys.argv[1:7]) if len(sys.argv) > 6 else (8, 32, 8192, 128, 64, 256)
MAXEV = int(sys.argv[7]) if len(sys.argv) > 7 else 400
PER = 160
cfg = eva.make_config(B, H, T, d, C, W)
Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
ks, vs = eva.eva_summarize(cfg, K, V)
O = torch.empty_like(Q)
lse = torch.empty(B * H, T, device="cuda")
tr = torch.zeros(4 * PER, dtype=torch.int64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
flush = torch.empty(512 << 18, device="cuda")
for _ in range(3):
    flush.zero_()
    N.check(N.lib.eva_debug_trace_prefill(ctypes.byref(cfg), P(Q), P(K), P(V), P(ks), P(vs), P(O), P(lse), P(tr), 3, st))
torch.cuda.synchronize()
names = {1: "TMA Q(i)", 2: "TMA K(j)", 3: "TMA V(j)", 4: "MMA K(j) seen", 5: "MMA S_i(j) issued",
         6: "MMA P_i seen", 7: "MMA PV_i issued", 8: "SM S(j) seen", 9: "SM P(j) done", 10: "EPI O final",
         11: "EPI done", 12: "MMA item", 13: "SM ld done", 14: "SM max done", 15: "SM o_done wait", 16: "SM exps done"}
roles = ["TMA", "MMA", "WG0", "WG1"]
v = [int(x) & 0xFFFFFFFFFFFFFFFF for x in tr.cpu().tolist()]
ev = []
for r in range(4):
    for x in v[r * PER:(r + 1) * PER]:
        if x:
            ev.append((x >> 24, r, (x >> 16) & 0xff, x & 0xffff))
ev.sort()
t0 = ev[0][0]
for (t, r, k, j) in ev[:MAXEV]:
    extra = f"i={j >> 12} j={j & 0xfff}" if k in (1, 5, 6, 7) else f"j={j}"
    print(f"{t - t0:8d}  {roles[r]:4s} {names.get(k, '?'):16s} {extra}")
