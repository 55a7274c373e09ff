"""Timeline of 4 CTAs of the one-tile-per-CTA prefill kernel (dev tool).
    python scripts/trace_tile.py B H T d C W [fused]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
from paper_2511_00576_b200 import _native as N

B, H, T, d, C, W = (int(x) for x in sys.argv[1:7]) if len(sys.argv) > 6 else (1, 16, 2048, 64, 64, 128)
FUSED = "fused" in sys.argv[7:]
R = 4  # roles per CTA slot
cfg = eva.make_config(B, H, T, d, C, W)
Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
ks, vs = eva.eva_summarize(cfg, K, V)
O = torch.empty_like(Q)
lse = torch.empty(B * H, T, device="cuda")
NCTA = 4096
tr = torch.zeros(4 * R * 48 + 4 * NCTA, dtype=torch.int64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
flush = torch.empty(512 << 18, device="cuda")
GRAPH = os.environ.get("GRAPH") == "1"   # replay the traced launch(es) from a CUDA graph
if GRAPH:
    N.check(N.lib.eva_debug_trace_prefill(ctypes.byref(cfg), P(Q), P(K), P(V), P(ks), P(vs), P(O), P(lse), P(tr), 2 if FUSED else 1000, st))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        stc = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        N.check(N.lib.eva_debug_trace_prefill(ctypes.byref(cfg), P(Q), P(K), P(V), P(ks), P(vs), P(O), P(lse), P(tr), 2 if FUSED else 1000, stc))
    for _ in range(3):
        flush.zero_()
        tr.zero_()
        g.replay()
    torch.cuda.synchronize()
else:
  for _ in range(3):
    flush.zero_()
    N.check(N.lib.eva_debug_trace_prefill(ctypes.byref(cfg), P(Q), P(K), P(V), P(ks), P(vs), P(O), P(lse), P(tr), 2 if FUSED else 1000, st))
  torch.cuda.synchronize()
names = {1: "start", 2: "MMA: Q arrived", 3: "MMA: K(j) arrived", 4: "MMA: S(j) issued", 5: "MMA: P(j) seen",
         6: "MMA: PV(j) issued", 7: "SM: got S(j)", 8: "SM: P(j) done", 9: "EPI: O final", 10: "EPI: stored",
         11: "TMA: slot free(j)", 12: "TMA: issued(j)", 13: "SUM: tile j landed", 14: "SUM: tile j done",
         15: "SUM: published", 16: "TMA: flag wait", 17: "TMA: flags ready",
         22: "MMA: S(j) elected", 23: "MMA: S(j) mma done", 18: "SUM: k~ sums (c)", 19: "SUM: omega (c)", 20: "SUM: logits (c)", 21: "SUM: beta (c)"}
v = [int(x) & 0xFFFFFFFFFFFFFFFF for x in tr.cpu().tolist()]
for slot in range(4):
    ev = [x for x in v[slot * R * 48:(slot + 1) * R * 48] if x]
    if not ev:
        continue
    ev.sort(key=lambda x: x >> 24)
    t0 = ev[0] >> 24
    print(f"=== CTA slot {slot}: {len(ev)} events, span {(ev[-1] >> 24) - t0} cycles")
    for x in ev:
        print(f"  {(x >> 24) - t0:7d}  {names.get((x >> 16) & 0xff, '?'):20s} j={x & 0xffff}")

# per-CTA entry/exit (globaltimer ns) relative to the earliest entry
ct = v[4 * R * 48:4 * R * 48 + 2 * NCTA]
st = v[4 * R * 48 + 2 * NCTA:]
spans = [(ct[2 * i], ct[2 * i + 1]) for i in range(NCTA) if ct[2 * i]]
if spans:
    sspans = [(st[2 * i], st[2 * i + 1]) for i in range(NCTA) if st[2 * i]]
    g0 = min([a for a, _ in spans] + [a for a, _ in sspans])
    if sspans:
        se = sorted(b - g0 for _, b in sspans)
        ss_ = sorted(a - g0 for a, _ in sspans)
        print(f"=== summarize: {len(sspans)} CTAs start p0/p100 {ss_[0]}/{ss_[-1]}  end p0/p50/p100 {se[0]}/{se[len(se) // 2]}/{se[-1]}")
    ends = sorted(b - g0 for _, b in spans)
    starts = sorted(a - g0 for a, _ in spans)
    dur = sorted(b - a for a, b in spans)
    q = lambda xs, f: xs[min(len(xs) - 1, int(f * len(xs)))]
    print(f"=== {len(spans)} CTAs (ns from first entry): start p0/p50/p100 {starts[0]}/{q(starts, .5)}/{starts[-1]}"
          f"  end p0/p50/p100 {ends[0]}/{q(ends, .5)}/{ends[-1]}  dur p0/p50/p100 {dur[0]}/{q(dur, .5)}/{dur[-1]}")
    for i, (a, b) in enumerate(spans[:8] + spans[-8:]):
        print(f"  cta {i if i < 8 else len(spans) - 16 + i}: {a - g0} -> {b - g0}")
