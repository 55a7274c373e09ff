"""H2D / D2H copy bandwidth on this box (pinned host memory), alone and concurrent (dev tool)."""
import torch, time
dev = torch.device("cuda")
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(n)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for mb in (1, 4, 12, 64):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory(); d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    h2 = torch.empty(mb << 20, dtype=torch.uint8).pin_memory(); d2 = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    th = t(lambda: d.copy_(h, non_blocking=True)); td = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)
    tb = t(both)
    print(f"{mb:3d} MiB: H2D {mb*1.048576/th:.1f} GB/s ({th*1e3:.0f} us), D2H {mb*1.048576/td:.1f} GB/s, both concurrently {tb*1e3:.0f} us")
