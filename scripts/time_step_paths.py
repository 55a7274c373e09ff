"""Which branch of the configs[1] step graph is critical: time CUDA graphs of the step's
sub-paths (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva
B, H, T, d, C, W = 1, 16, 2048, 64, 64, 128
cfg = eva.make_config(B, H, T, d, C, W)
Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
ks, vs = eva.eva_summarize(cfg, K, V)
O = torch.empty_like(Q); lse = torch.empty(B * H, T, device="cuda")
qn, kn, vn = (x[0] for x in eva_inputs.decode_tokens(0, B * H, 1, d, torch.bfloat16, seed=1, device="cuda"))
cache = eva.DecodeCache(cfg, T // C + 2, device="cuda")
od = torch.empty(B * H, d, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(512 << 18, device="cuda")
s = torch.cuda.current_stream()
side = torch.cuda.Stream()
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
side_lo = torch.cuda.Stream(priority=0)          # 0 = lowest priority in CUDA
main_hi = torch.cuda.Stream(priority=-1)         # higher priority
def summ(): eva.eva_summarize(cfg, K, V, Ksum=ks, Vsum=vs)
def pre(): eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, lse=lse)
def pre_ov(): eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, lse=lse,
                                   overlap=True)
def full_overlap():
    # the prefill right after the summarize on the same stream, EVA_PREFILL_OVERLAP: its local
    # tiles may start before the summaries are complete; the hand-off forks after the prefill
    summ()
    pre_ov()
    side.wait_stream(s)
    with torch.cuda.stream(side):
        hand()
    s.wait_stream(side)
def full_overlap_fork_first():
    summ()
    ev = torch.cuda.Event()
    ev.record(s)
    pre_ov()
    side.wait_event(ev)
    with torch.cuda.stream(side):
        hand()
    s.wait_stream(side)
def hand():
    cache.c.pos = 0
    cache.eva_cache_load(K, V, ks, vs)
    cache.eva_decode_step(qn, kn, vn, O=od, want_lse=False)
def full():
    summ()
    side.wait_stream(s)
    with torch.cuda.stream(side):
        hand()
    pre()
    s.wait_stream(side)
def full_prefill_first():
    summ()
    side.wait_stream(s)
    pre()
    with torch.cuda.stream(side):
        hand()
    s.wait_stream(side)
def full_prio():
    # main work on a high-priority stream, hand-off + decode on a low-priority one
    s = torch.cuda.current_stream()
    main_hi.wait_stream(s)
    with torch.cuda.stream(main_hi):
        summ()
        side_lo.wait_stream(main_hi)
        with torch.cuda.stream(side_lo):
            hand()
        pre()
        main_hi.wait_stream(side_lo)
    s.wait_stream(main_hi)
paths = {"summarize": summ, "prefill": pre, "summarize+prefill": lambda: (summ(), pre()),
         "handoff+decode": hand, "summarize+handoff+decode": lambda: (summ(), hand()), "full step": full,
         "full, prefill issued first": full_prefill_first, "full, stream priorities": full_prio,
         "summarize+prefill overlap": lambda: (summ(), pre_ov()), "full overlap": full_overlap,
         "full overlap, fork event": full_overlap_fork_first}
for name, fn in paths.items():
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(30):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"{name:28s} median {ts[15]:.1f} us  min {ts[0]:.1f} us")
