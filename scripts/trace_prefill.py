"""Timeline of CTA 0 of the persistent prefill kernel (dev tool).
    python scripts/trace_prefill.py [T] [B] [H] [d]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
from paper_2511_00576_b200 import _native as N

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
H = int(sys.argv[3]) if len(sys.argv) > 3 else 32
d = int(sys.argv[4]) if len(sys.argv) > 4 else 128
cfg = eva.make_config(B, H, T, d, 64, 256)
Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
ks, vs = eva.eva_summarize(cfg, K, V)
O = torch.empty_like(Q)
lse = torch.empty(B * H, T, device="cuda")
cap = 1 << 16
tr = torch.zeros(cap, dtype=torch.int64, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr())
for it in range(3):
    tr.zero_()
    N.check(N.lib.eva_debug_trace_prefill(ctypes.byref(cfg), P(Q), P(K), P(V), P(ks), P(vs), P(O), P(lse), P(tr), cap, st))
torch.cuda.synchronize()
ev = [int(x) & 0xFFFFFFFFFFFFFFFF for x in tr.cpu().tolist() if x != 0]
ev.sort(key=lambda x: x >> 24)
t0 = ev[0] >> 24
names = {1: "TMA issued tile", 2: "MMA S", 3: "MMA PV", 4: "SM got S", 5: "SM P done", 6: "EPI done",
         7: "TMA slot free", 8: "MMA k_full", 9: "MMA p_full", 10: "MMA S begin", 11: "MMA S issued"}
print("events", len(ev))
last = {}
for x in ev[:600]:
    c = x >> 24; code = x & 0xFFFFFF
    kind, t, j = code >> 20, (code >> 16) & 0xF, code & 0xFFFF
    print(f"{c - t0:9d}  {names.get(kind, kind):16s} t={t} j={j}")
# per-kind average intervals
import collections
by = collections.defaultdict(list)
for x in ev:
    c = x >> 24; code = x & 0xFFFFFF
    by[(code >> 20, (code >> 16) & 0xF)].append(c)
for k, v in sorted(by.items()):
    if len(v) > 2:
        d = [b - a for a, b in zip(v, v[1:])]
        print(names.get(k[0]), "t", k[1], "n", len(v), "mean interval", sum(d) / len(d))
print("total cycles CTA0", (ev[-1] >> 24) - t0)
