"""Ragged decode at configs[3] (dev tool): per-step times of eva_decode_step_ragged with all
units at one position vs spread over 64 positions 64 tokens apart, against eva_decode_step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_00576_b200 as eva

BH, d, C, W, ctx, steps = 256 * 32, 128, 64, 256, 32768, 128
cap = (ctx + steps) // C + 1
cfg = eva.make_config(256, 32, 0, d, C, W)
cache = eva.DecodeCache(cfg, cap, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(5)
for t in (cache.ring_k, cache.ring_v, cache.sum_k, cache.sum_v):
    t.copy_(torch.randn(t.shape, generator=g, device="cuda", dtype=torch.float32))
toks = torch.randn(steps, 3, BH, d, generator=g, device="cuda").to(torch.bfloat16)
o = torch.empty(BH, d, dtype=torch.bfloat16, device="cuda")

def run(fn, label):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record()
    for i in range(steps):
        fn(i)
        ev[i + 1].record()
    torch.cuda.synchronize()
    ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    chunk = [t for i, t in enumerate(ts) if i % 64 == 63]
    other = sorted(t for i, t in enumerate(ts) if i % 64 != 63)
    print(f"{label}: mean {sum(ts) / steps * 1e3:.1f} us/token, median non-completing {other[len(other) // 2] * 1e3:.1f} us, "
          f"completing steps {[round(t * 1e3, 1) for t in chunk]}", flush=True)

cache.c.pos = ctx
cache.eva_attn_decode(toks[0, 0], O=o, want_lse=False)
run(lambda i: cache.eva_decode_step(toks[i, 0], toks[i, 1], toks[i, 2], O=o, want_lse=False), "uniform eva_decode_step")
for label, pos0 in (("ragged, one position", torch.full((BH,), ctx, dtype=torch.int64, device="cuda")),
                    ("ragged, 64 positions 64 apart", ctx - 64 * (torch.arange(BH, device="cuda", dtype=torch.int64) % 64)),
                    ("ragged, 64 positions 1 apart", ctx - (torch.arange(BH, device="cuda", dtype=torch.int64) % 64))):
    pos = pos0.clone()
    cache.eva_decode_step_ragged(pos, toks[0, 0], toks[0, 1], toks[0, 2], O=o, want_lse=False)
    pos.copy_(pos0)
    run(lambda i: cache.eva_decode_step_ragged(pos, toks[i, 0], toks[i, 1], toks[i, 2], O=o, want_lse=False), label)
    pos.copy_(pos0)
    run(lambda i: cache.eva_decode_step_ragged(pos, toks[i, 0], toks[i, 1], toks[i, 2], O=o, want_lse=False,
                                               rope=dict(rope_base=10000.0)), label + " + RoPE folded")
