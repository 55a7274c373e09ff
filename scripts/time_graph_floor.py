"""Event-timed CUDA-graph replay of a trivial kernel after the L2 flush (dev tool): the floor the
step timings sit on."""
import torch
flush = torch.empty(512 << 18, device="cuda")
x = torch.empty(256, device="cuda")
for label, body in (("1 tiny kernel", lambda: x.fill_(1.0)), ("2 tiny kernels", lambda: (x.fill_(1.0), x.add_(1.0)))):
    body(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    for _ in range(5): g.replay()
    for flushed in (True, False):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
        for a, b in ev:
            if flushed: flush.zero_()
            a.record(); g.replay(); b.record()
        torch.cuda.synchronize()
        print(f"{label}, flush={flushed}: {sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3:.2f} us", flush=True)
