"""Prefill variants (NEXT row 3) at configs[2]'s per-GPU shape on one B200: the causal
partitions (sliding, block), the non-causal partition and the ln C summary bias, tcgen05 tile
kernel, L2 flushed between reps.  Prints one JSON line per variant (dev tool)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import eva_inputs
import paper_2511_00576_b200 as eva

B, H, T, d, C, W = 8, 32, 8192, 128, 64, 256
Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda")
flush = torch.empty(512 << 18, device="cuda")
O = torch.empty_like(Q)
lse = torch.empty(B * H, T, device="cuda")
(dO,) = eva_inputs.normal_units(1, 0, B * H, T, d, torch.bfloat16, seed=1, device="cuda")
dQ, dK, dV = torch.empty_like(Q), torch.empty_like(Q), torch.empty_like(Q)


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def keys_per_query(mode):
    n = torch.arange(T, dtype=torch.int64)
    nC = T // C
    if mode == "sliding":
        ns = torch.clamp(n // C - W // C + 1, min=0)
        return (n - ns * C + 1 + ns).double().mean().item()
    lo = (n // W) * W
    if mode == "block":
        return (n - lo + 1 + lo // C).double().mean().item()
    hi = torch.clamp(lo + W, max=T)
    s2 = torch.clamp((lo + W) // C, max=nC)
    return ((hi - lo) + lo // C + (nC - s2)).double().mean().item()


for name, mode, bias in (("sliding", "sliding", 0.0), ("block", "block", 0.0),
                         ("noncausal", "noncausal", 0.0), ("sliding+lnC", "sliding", math.log(C))):
    cfg = eva.make_config(B, H, T, d, C, W, mode=mode, summary_bias=bias)
    ks, vs = eva.eva_summarize(cfg, K, V)
    fwd = lambda: eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True,
                                       O=O, lse=lse)
    fwd(); fwd()
    ms = timed(fwd)
    ws = torch.empty(eva.eva_backward_workspace_bytes(cfg), dtype=torch.uint8, device="cuda")
    bwd = lambda: eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws, dQ=dQ,
                                        dK=dK, dV=dV)
    bwd(); bwd()
    bms = timed(bwd, 5)
    del ws
    kq = keys_per_query(mode)
    gb = B * H * (4 * T * d * 2 + 2 * (T // C) * d * 2 + 4 * T) / 1e9
    tf = B * H * T * kq * 4 * d / 1e12
    print(json.dumps({"variant": name, "ms": ms, "keys_per_query": kq, "hbm_TBps": gb / ms,
                      "alg_TFLOPs": tf / (ms / 1e3), "bwd_ms": bms}))
