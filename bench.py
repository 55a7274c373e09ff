#!/usr/bin/env python
"""bench.py -- FlashEVA hot path on B200: prefill tokens/s (+ decode tokens/s), % of roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-extras]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)
With --gpus N > 1 and no torchrun environment, bench.py re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (127.0.0.1, a free port) and passes the
rank-0 JSON line through.  --stub runs the launcher and the multi-rank bookkeeping with the
kernels replaced by host sleeps on gloo (the CPU test of the N-rank path).

Workload (BASELINE.json configs[1]): B=1, H=16, T=2048, d=64, C=64, W=128, bf16, sliding
window, Q/K/V ~ N(0,1) synthetic (eva_inputs), eps from the in-kernel Philox.
One STEP = the whole hot path over one batch:
    eva_summarize (a1-a3) -> eva_attn_prefill (a4-a5, summaries provided)
    -> eva_cache_load (a6, prompt hand-off with the prefill's summaries)
    -> eva_decode_step (a6 + a7: append the next token and attend it, one launch)
The step is captured once as a CUDA graph and replayed (it is launch-latency scale).
metric value = prompt tokens (B*T per GPU, all ranks) / device time of the step.
Weak scaling: rank r owns units [r*B*H, (r+1)*B*H) of a global batch of N*B sequences;
no collective on the data path.  L2 (126 MB) is larger than the 17 MB
working set, so a 512 MiB buffer is overwritten before every timed step (outside the
events); config.l2 says so.

Extras (every rank with its own shard; rank 0 prints): configs[2] prefill per GPU (B=8, H=32,
T=8192, d=128, C=64, W=256; weak: 256 units per rank) and configs[2] strong-scaled (its 256
units split over the N ranks, max-over-ranks device time, plus the NCCL gather of O to rank 0
timed separately), configs[3] decode (B=256, H=32, d=128, 32k compressed context, 512
generated tokens), configs[4] long-context cells (T = 4k..128k, H=32, d=128, C, W), the
backward at configs[1]/[2] shapes, each with its roofline; the configs[0] oracle time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(name="configs[1]: B=1,H=16,T=2048,d=64,C=64,W=128 bf16 prefill + cache hand-off + 1 decode",
                B=1, H=16, T=2048, d=64, C=64, W=128)
LARGE = dict(B=8, H=32, T=8192, d=128, C=64, W=256)
DECODE = dict(B=256, H=32, d=128, C=64, W=256, ctx=32768, gen=512)
L2_FLUSH_BYTES = 512 << 20


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return dict(hbm=float(j["hbm_gbs"]), bf16=float(j["bf16_tflops"]),
                    bf16_sus=float(j.get("bf16_tflops_sustained", j["bf16_tflops"])),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ============================================================================ our arm
def prefill_bytes(BH, T, d, C, elem=2, lse=True):
    """Algorithmic HBM bytes of one eva_attn_prefill launch with summaries provided:
    Q, K, V read once + O written once + Ksum, Vsum read once (+ LSE written)."""
    nC = T // C
    return BH * (4 * T * d * elem + 2 * nC * d * elem + (4 * T if lse else 0))


def prefill_flops(BH, T, d, C, W, mode=0):
    """Algorithmic flops: sum_n (|E(n)| + nsum(n)) * 4d."""
    tot = 0
    R = W // C
    for n in range(T):
        if mode == 0:
            ns = max(0, n // C - R + 1)
            lo = ns * C
        else:
            lo = (n // W) * W
            ns = lo // C
        tot += (n - lo + 1) + ns
    return BH * tot * 4 * d


def decode_bytes(BH, d, n, C, W, elem=2):
    """Algorithmic bytes of one fused decode step at query n: K+V of every
    visible entry + q + o + the appended k, v (read once, written to the ring) + when the
    token completes a chunk, the chunk's C key/value rows re-read and its summary written."""
    ns = max(0, n // C - W // C + 1)
    lo = ns * C
    b = (ns + n - lo + 1) * 2 * d * elem + 2 * d * elem + 2 * 2 * d * elem
    if (n + 1) % C == 0:
        b += 2 * C * d * elem + 2 * d * elem
    return BH * b


def run_ours(args, rank, world, local_rank):
    import torch

    import eva_inputs
    import paper_2511_00576_b200 as eva

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    peaks = load_peaks()
    s = torch.cuda.current_stream(dev)

    from paper_2511_00576_b200.parallel import max_over_ranks, shard_for

    wl = WORKLOAD
    B, H, T, d, C, W = (wl[k] for k in ("B", "H", "T", "d", "C", "W"))
    shard = shard_for(rank, world, B * world, H)   # weak scaling: B sequences per GPU
    BH, bh0 = shard.bh_count, shard.bh_begin
    nC = T // C
    cfg = eva.make_config(B * world, H, T, d, C, W, bh_begin=bh0, bh_count=BH, dtype=torch.bfloat16)
    Q, K, V = eva_inputs.qkv(bh0, BH, T, d, torch.bfloat16, seed=0, device=dev)
    Ksum = torch.empty(BH, nC, d, dtype=torch.bfloat16, device=dev)
    Vsum = torch.empty_like(Ksum)
    O = torch.empty_like(Q)
    lse = torch.empty(BH, T, dtype=torch.float32, device=dev)
    qn, kn, vn = eva_inputs.decode_tokens(bh0, BH, 1, d, torch.bfloat16, seed=1, device=dev)
    qn, kn, vn = qn[0], kn[0], vn[0]
    cache = eva.DecodeCache(cfg, nC + 2, device=dev)
    o_dec = torch.empty(BH, d, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    side = torch.cuda.Stream(dev)

    def step_serial():
        """One pass of the whole hot path over the batch."""
        cache.c.pos = 0
        eva.eva_summarize(cfg, K, V, Ksum=Ksum, Vsum=Vsum)                       # a1-a3
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=Ksum, Vsum=Vsum, summaries_provided=True,
                             O=O, lse=lse)                                       # a4-a5
        cache.eva_cache_load(K, V, Ksum, Vsum)                                    # a6 hand-off
        cache.eva_decode_step(qn, kn, vn, O=o_dec, want_lse=False)                # a6 + a7 fused

    def step():
        """The same kernels; the cache hand-off and the first decode token depend only on the
        summaries, so they run on a second stream concurrently with the prefill."""
        cache.c.pos = 0
        eva.eva_summarize(cfg, K, V, Ksum=Ksum, Vsum=Vsum)                       # a1-a3
        side.wait_stream(s)
        with torch.cuda.stream(side):
            cache.eva_cache_load(K, V, Ksum, Vsum)                                # a6 hand-off
            cache.eva_decode_step(qn, kn, vn, O=o_dec, want_lse=False)            # a6 + a7 fused
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=Ksum, Vsum=Vsum, summaries_provided=True,
                             O=O, lse=lse)                                       # a4-a5
        s.wait_stream(side)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    # The step is launch-latency scale (~tens of us), so it is captured once as a CUDA graph
    # and replayed: every replay runs the same libeva kernels on the same buffers.
    n0 = eva.launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    kernels_per_step = eva.launch_count() - n0
    graph_serial = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_serial):
        step_serial()
    for _ in range(args.warmup):
        flush.zero_()
        graph.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if dist: dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(s)
            graph.replay()
            ev[i][1].record(s)
        torch.cuda.synchronize()
        if dist: dist.barrier()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
        n_launch = kernels_per_step * args.steps
        step_ms = [a.elapsed_time(b) for a, b in ev]
        total_ms = max_over_ranks(sum(step_ms), device=dev)

        # ---------------- the same step with the four kernels serialised on one stream
        for _ in range(2):
            flush.zero_()
            graph_serial.replay()
        ser = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            ser[i][0].record(s)
            graph_serial.replay()
            ser[i][1].record(s)
        torch.cuda.synchronize()
        serial_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ser), device=dev) / args.steps

        # ---------------- per-kernel device times (eager launches, same buffers, L2 flushed)
        kev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            # keep the device busy while the host enqueues the four launches and their events, so
            # the event gaps are device time (launch latency and kernel), not host enqueue time
            torch.cuda._sleep(400000)
            e = kev[i]
            cache.c.pos = 0
            e[0].record(s)
            eva.eva_summarize(cfg, K, V, Ksum=Ksum, Vsum=Vsum)
            e[1].record(s)
            eva.eva_attn_prefill(cfg, Q, K, V, Ksum=Ksum, Vsum=Vsum, summaries_provided=True, O=O, lse=lse)
            e[2].record(s)
            cache.eva_cache_load(K, V, Ksum, Vsum)
            e[3].record(s)
            cache.eva_decode_step(qn, kn, vn, O=o_dec, want_lse=False)
            e[4].record(s)
        torch.cuda.synchronize()
        sum_ms = [e[0].elapsed_time(e[1]) for e in kev]
        pre_ms = [e[1].elapsed_time(e[2]) for e in kev]
        app_ms = [e[2].elapsed_time(e[3]) for e in kev]
        dec_ms = [e[3].elapsed_time(e[4]) for e in kev]

        # ---------------- e2e through the public API with pinned host buffers
        hQ, hK, hV = (x.cpu().pin_memory() for x in (Q, K, V))
        hO = torch.empty(BH, T, d, dtype=torch.bfloat16).pin_memory()
        hOd = torch.empty(BH, d, dtype=torch.bfloat16).pin_memory()
        e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]

        hp = eva.HostPrefill(cfg, max_slices=max(16, args.e2e_slices), device=dev)

        def e2e_step(e=None, n_slices=None):
            """Public API from pinned host buffers: eva_attn_prefill_host (H2D of Q/K/V, the
            summarize + prefill kernels and the D2H of O pipelined over unit slices), the
            cache hand-off, one decode step and its D2H."""
            if e: e[0].record(s)
            cache.c.pos = 0
            hp(hQ, hK, hV, hO, n_slices=n_slices or args.e2e_slices)
            cache.eva_cache_load(hp.K, hp.V, hp.Ksum, hp.Vsum)
            od, _ = cache.eva_decode_step(qn, kn, vn, want_lse=False)
            hOd.copy_(od, non_blocking=True)
            if e: e[1].record(s)

        # both variants are warmed up before either is timed: the first timed loop otherwise
        # pays a one-off host-side cost (pinned-page / IOMMU warm-up) that biases the order
        for _ in range(max(args.warmup, 10)):
            e2e_step()
            e2e_step(n_slices=4)
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            e2e_step(e_ev[i])
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in e_ev), device=dev)
        for i in range(args.steps):   # the same with the copies pipelined over 4 unit slices, context
            flush.zero_()
            e2e_step(e_ev[i], n_slices=4)
        torch.cuda.synchronize()
        e2e1_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in e_ev), device=dev)

        extras = {}
        if not args.no_extras:
            extras["prefill_configs2"] = bench_prefill_large(args, eva, torch, dev, s, rank, world, peaks)
            extras["prefill_configs2_strong"] = bench_prefill_strong(args, eva, torch, dev, s, rank, world, peaks, dist)
            extras["sweep_configs4"] = bench_sweep(args, eva, torch, dev, s, rank, world, peaks)
            extras["decode_configs3"] = bench_decode(args, eva, torch, dev, s, rank, world, peaks)
            extras["backward_configs2"] = bench_backward(args, eva, torch, dev, s, rank, world, peaks, LARGE)
            extras["backward_configs1"] = bench_backward(args, eva, torch, dev, s, rank, world, peaks, WORKLOAD)
    clocks = clk.summary()

    tokens = world * B * T * args.steps
    value = tokens / (total_ms / 1e3)
    pre_avg = statistics.mean(pre_ms)
    pbytes = prefill_bytes(BH, T, d, C)
    achieved = pbytes / (pre_avg / 1e3) / 1e9
    result = {
        "metric": "prefill tokens/s (FlashEVA hot path, whole job)",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (Q,K,V ~ N(0,1) seeded per (b,h); eps from in-kernel Philox)",
        "config": {"workload": wl["name"], "B_per_gpu": B, "H": H, "T": T, "d_head": d, "chunk": C,
                   "window": W, "mode": "sliding", "global_batch": B * world,
                   "parallelism": f"(b,h)-sharded x{world}, no data-path collective",
                   "l2": "512 MiB L2 flush before every timed step (outside the events)"},
        "roofline": {"kernel": "eva_attn_prefill (summaries provided)", "bound": "hbm",
                     "achieved": achieved, "peak": peaks["hbm"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm"], "traffic": load_traffic("prefill_configs1"),
                     "alg_bytes_per_launch": pbytes, "avg_launch_ms": pre_avg,
                     "share_of_step": pre_avg / (statistics.mean(sum_ms) + pre_avg + statistics.mean(app_ms)
                                                 + statistics.mean(dec_ms)),
                     "peak_source": peaks["src"]},
        "breakdown_ms": {"summarize": statistics.mean(sum_ms), "prefill": pre_avg,
                         "cache_load": statistics.mean(app_ms), "decode_step": statistics.mean(dec_ms),
                         "note": "eager per-kernel events, launched behind a device-side delay so the host is ahead (device time); the step itself is a CUDA-graph replay",
                     "step_serial_ms": serial_ms,
                     "step_graph": "summarize -> {prefill || cache_load -> decode_step}, PDL launches"},
        "kernels_per_step": kernels_per_step,
        "e2e": {"value": tokens / (e2e_ms / 1e3), "unit": "tokens/s",
                "value_4_slices": tokens / (e2e1_ms / 1e3),
                "h2d_bytes_per_step": 3 * BH * T * d * 2, "d2h_bytes_per_step": BH * T * d * 2 + BH * d * 2,
                "api": "eva_attn_prefill_host (C ABI: H2D / summarize+prefill / D2H pipelined over "
                       f"{min(args.e2e_slices, BH)} unit slices) + eva_cache_load + eva_decode_step, pinned host buffers"},
        "gpu_launches": n_launch,
        "wall_s_timed_region": t_wall,
        "clocks": clocks,
    }
    result.update(extras)
    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, budget_s=args.cpu_budget)
        result["cpu_oracle_configs0"] = cpu_oracle_configs0()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return result


def load_traffic(key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        v = j.get(key)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch")
    return None


def bench_prefill_large(args, eva, torch, dev, s, rank, world, peaks):
    """configs[2] per-GPU shape: B=8, H=32, T=8192, d=128 prefill (inputs > L2)."""
    import eva_inputs
    L = LARGE
    BH = L["B"] * L["H"]
    T, d, C, W = L["T"], L["d"], L["C"], L["W"]
    bh0 = rank * BH
    cfg = eva.make_config(L["B"] * world, L["H"], T, d, C, W, bh_begin=bh0, bh_count=BH)
    Q, K, V = eva_inputs.qkv(bh0, BH, T, d, torch.bfloat16, seed=0, device=dev)
    ks, vs = eva.eva_summarize(cfg, K, V)
    O = torch.empty_like(Q)
    lse = torch.empty(BH, T, dtype=torch.float32, device=dev)
    reps = max(3, min(args.steps, 20))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
    for _ in range(2):
        eva.eva_summarize(cfg, K, V, Ksum=ks, Vsum=vs)
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, lse=lse)
    torch.cuda.synchronize()
    for e in evs:
        e[0].record(s)
        eva.eva_summarize(cfg, K, V, Ksum=ks, Vsum=vs)
        e[1].record(s)
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, lse=lse)
        e[2].record(s)
    torch.cuda.synchronize()
    step = statistics.mean(e[0].elapsed_time(e[2]) for e in evs)
    pre = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    summ = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    pb = prefill_bytes(BH, T, d, C)
    pf = prefill_flops(BH, T, d, C, W)
    out = {"workload": "configs[2] per GPU: B=8,H=32,T=8192,d=128,C=64,W=256 bf16 (summarize + prefill)",
           "tokens_per_s_per_gpu": L["B"] * T / (step / 1e3), "ms_per_step": step,
           "summarize_ms": summ, "prefill_ms": pre,
           "roofline": {"kernel": "eva_attn_prefill", "bound": "hbm",
                        "achieved": pb / (pre / 1e3) / 1e9, "peak": peaks["hbm"], "unit": "GB/s",
                        "frac": pb / (pre / 1e3) / 1e9 / peaks["hbm"],
                        "tensor_tflops_alg": pf / (pre / 1e3) / 1e12,
                        "tensor_frac_of_bf16_peak": pf / (pre / 1e3) / 1e12 / peaks["bf16"],
                        "traffic": load_traffic("prefill_configs2")},
           "summarize_roofline": {"bound": "hbm", "achieved": 2 * BH * T * d * 2 / (summ / 1e3) / 1e9,
                                  "peak": peaks["hbm"], "unit": "GB/s"}}
    # RoPE (NEXT row 4, R18/R19) on the same inputs: rotation inside the tcgen05 prefill
    # (eva_attn_prefill_rope; summaries of the rotated keys by the summaries-only RoPE
    # summariser) against the two-pass form (eva_rope_summarize writes Qr, Kr, then the prefill)
    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(s)
        for _ in range(reps):
            fn()
        ev[1].record(s)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / reps
    Qr, Kr, rks, rvs = eva.eva_rope_summarize(cfg, Q, K, V)
    out["rope"] = {
        "prefill_in_kernel_ms": timed(lambda: eva.eva_attn_prefill_rope(
            cfg, Q, K, V, Ksum=rks, Vsum=rvs, summaries_provided=True, O=O, lse=lse)),
        "step_in_kernel_ms": timed(lambda: eva.eva_attn_prefill_rope(cfg, Q, K, V, Ksum=rks, Vsum=rvs, O=O, lse=lse)),
        "step_two_pass_ms": timed(lambda: (eva.eva_rope_summarize(cfg, Q, K, V),
                                           eva.eva_attn_prefill(cfg, Qr, Kr, V, Ksum=rks, Vsum=rvs,
                                                                summaries_provided=True, O=O, lse=lse))),
        "step_k_prerotated_ms": timed(lambda: (eva.eva_rope(cfg, K, out=Kr),
                                               eva.eva_attn_prefill_rope(cfg, Q, Kr, V, Ksum=rks, Vsum=rvs, O=O,
                                                                         lse=lse, k_rotated=True))),
        "note": "rotary_dim = d, interleaved, base 10000; step = summaries of the rotated keys + prefill; "
                "k_prerotated = eva_rope writes RoPE(K) once, the plain summariser on it, the prefill "
                "rotating Q only (EVA_ROPE_K_ROTATED)"}
    del Q, K, V, O, ks, vs, Qr, Kr, rks, rvs
    torch.cuda.empty_cache()
    return out


def bench_backward(args, eva, torch, dev, s, rank, world, peaks, L):
    """eva_attn_backward (NEXT row 1) at a per-GPU shape (configs[2] or configs[1]): prep +
    tcgen05 main pass + summary chain rule (configs[2]: the fused schedule -- summary tiles,
    coefficients, local tiles applying them, dQ conversion; configs[1]: one main launch +
    finalize, the size rule in backward_simt.cu).  Algorithmic flops: 10d per visible
    (query, key) pair (S recompute, dP, dV, dK, dQ); algorithmic bytes: Q, K, V, O, dO, lse
    read + dQ, dK, dV written once.  L2 is flushed before every rep (configs[1] fits in it)."""
    import eva_inputs
    BH = L["B"] * L["H"]
    T, d, C, W = L["T"], L["d"], L["C"], L["W"]
    bh0 = rank * BH
    cfg = eva.make_config(L["B"] * world, L["H"], T, d, C, W, bh_begin=bh0, bh_count=BH)
    Q, K, V = eva_inputs.qkv(bh0, BH, T, d, torch.bfloat16, seed=0, device=dev)
    (dO,) = eva_inputs.normal_units(1, bh0, BH, T, d, torch.bfloat16, seed=2, device=dev)
    O, lse, ks, vs = eva.eva_attn_prefill(cfg, Q, K, V)
    ws = torch.empty(eva.eva_backward_workspace_bytes(cfg), dtype=torch.uint8, device=dev)
    dQ, dK, dV = (torch.empty_like(Q) for _ in range(3))
    for _ in range(2):
        eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws, dQ=dQ, dK=dK, dV=dV)
    torch.cuda.synchronize()
    reps = max(3, min(args.steps, 10))
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        flush.zero_()
        a.record(s)
        eva.eva_attn_backward(cfg, Q, K, V, ks, vs, O, lse, dO, workspace=ws, dQ=dQ, dK=dK, dV=dV)
        b.record(s)
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    flops = prefill_flops(BH, T, d, C, W) * 10 // 4
    nbytes = BH * T * d * 2 * 8 + BH * T * 4
    out = {"workload": f"B={L['B']},H={L['H']},T={T},d={d},C={C},W={W} bf16 per GPU, eva_attn_backward "
                       + ("(fused: prep, tcgen05 summary tiles, chain-rule coefficients, tcgen05 local tiles, dQ convert)"
                          if BH * T * d >= (1 << 25) else "(prep + tcgen05 main + finalize)"),
           "ms": ms, "tokens_per_s_per_gpu": L["B"] * T / (ms / 1e3),
           "roofline": {"bound": "tensor", "achieved": flops / (ms / 1e3) / 1e12, "peak": peaks["bf16"],
                        "unit": "TFLOP/s", "frac": flops / (ms / 1e3) / 1e12 / peaks["bf16"],
                        "alg_flops": flops, "hbm_alg_bytes": nbytes,
                        "hbm_frac": nbytes / (ms / 1e3) / 1e9 / peaks["hbm"]}}
    del Q, K, V, O, dO, dQ, dK, dV, ws, ks, vs, flush
    torch.cuda.empty_cache()
    return out


def bench_decode(args, eva, torch, dev, s, rank, world, peaks):
    """configs[3]: B=256, H=32, d=128, 32k compressed context (C=64, W=256), 512 tokens.
    The ring and summary list are filled with seeded N(0,1) values at pos = 32768 (their
    values do not change the work); then 512 x (append + decode) are timed."""
    D = DECODE
    BH = D["B"] * D["H"]
    d, C, W, ctx, gen = D["d"], D["C"], D["W"], D["ctx"], D["gen"]
    steps = gen if not args.quick else 64
    cap = (ctx + gen) // C + 1
    cfg = eva.make_config(D["B"] * world, D["H"], 0, d, C, W, bh_begin=rank * BH, bh_count=BH)
    cache = eva.DecodeCache(cfg, cap, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    for t in (cache.ring_k, cache.ring_v, cache.sum_k, cache.sum_v):
        t.copy_(torch.randn(t.shape, generator=g, device=dev, dtype=torch.float32))
    cache.c.pos = ctx
    toks = torch.randn(steps, 3, BH, d, generator=g, device=dev).to(torch.bfloat16)
    o = torch.empty(BH, d, dtype=torch.bfloat16, device=dev)
    cache.eva_attn_decode(toks[0, 0], O=o, want_lse=False)  # warm + workspace
    torch.cuda.synchronize()
    e_app = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    e_dec = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    nbytes = 0
    e_app[0].record(s)
    for i in range(steps):
        e_dec[i].record(s)
        cache.eva_decode_step(toks[i, 0], toks[i, 1], toks[i, 2], O=o, want_lse=False)  # append + decode
        e_app[i + 1].record(s)
        nbytes += decode_bytes(BH, d, cache.pos - 1, C, W)
    torch.cuda.synchronize()
    total = e_app[0].elapsed_time(e_app[-1])
    dec = sum(e_dec[i].elapsed_time(e_app[i + 1]) for i in range(steps))
    # the same tokens through the two-launch path (append kernel + decode kernel), for reference
    cache.c.pos = ctx
    e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e2[0].record(s)
    for i in range(steps):
        cache.eva_cache_append(toks[i, 1], toks[i, 2])
        cache.eva_attn_decode(toks[i, 0], O=o, want_lse=False)
    e2[1].record(s)
    torch.cuda.synchronize()
    two_launch_ms = e2[0].elapsed_time(e2[1]) / steps
    # the same tokens through eva_decode_step_ragged (per-unit positions, NEXT row 4), with
    # the units spread over 64 positions 64 tokens apart below the context
    pos0 = ctx - 64 * (torch.arange(BH, device=dev, dtype=torch.int64) % 64)
    pos = pos0.clone()
    cache.eva_decode_step_ragged(pos, toks[0, 0], toks[0, 1], toks[0, 2], O=o, want_lse=False)  # warm
    pos.copy_(pos0)
    torch.cuda.synchronize()
    er = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    er[0].record(s)
    for i in range(steps):
        cache.eva_decode_step_ragged(pos, toks[i, 0], toks[i, 1], toks[i, 2], O=o, want_lse=False)
    er[1].record(s)
    torch.cuda.synchronize()
    ragged_ms = er[0].elapsed_time(er[1]) / steps
    p_host = pos0.cpu().tolist()
    rbytes = sum(decode_bytes(1, d, p + i, C, W) for i in range(0, steps, max(1, steps // 16))
                 for p in p_host[:64]) * (BH // 64) / len(range(0, steps, max(1, steps // 16)))
    out = {"workload": f"configs[3]: B=256,H=32,d=128,C=64,W=256, context {ctx}, {steps} generated tokens",
           "tokens_per_s_per_gpu": D["B"] * steps / (total / 1e3), "ms_per_token": total / steps,
           "decode_ms_per_token": dec / steps,
           "two_launch_ms_per_token": two_launch_ms,
           "ragged_ms_per_token": ragged_ms,
           "ragged_hbm_frac": rbytes / (ragged_ms / 1e3) / 1e9 / peaks["hbm"],
           "ragged_note": "eva_decode_step_ragged (ragged_append + decode, 2 launches/token), units at "
                          "64 positions 64 tokens apart; bytes sampled over 16 steps",
           "roofline": {"kernel": "eva_attn_decode", "bound": "hbm",
                        "achieved": nbytes / (dec / 1e3) / 1e9, "peak": peaks["hbm"], "unit": "GB/s",
                        "frac": nbytes / (dec / 1e3) / 1e9 / peaks["hbm"],
                        "alg_bytes_per_launch": nbytes / steps, "traffic": load_traffic("decode_configs3")}}
    del cache, toks
    torch.cuda.empty_cache()
    return out



def bench_prefill_strong(args, eva, torch, dev, s, rank, world, peaks, dist):
    """configs[2] strong-scaled: its 256 (b,h) units split contiguously over the N ranks
    (paper_2511_00576_b200.parallel.shard_units), summarize + prefill per rank on the rank's own
    synthetic inputs (RNG keyed by the global unit), device time max over ranks.  The path has
    no exchange step; the NCCL all-gather of O into rank 0's [256, T, d] buffer (the
    "scatter/gather of the shards") is timed separately and is not part of the value."""
    import eva_inputs
    from paper_2511_00576_b200.parallel import max_over_ranks, shard_units
    L = LARGE
    units = L["B"] * L["H"]
    T, d, C, W = L["T"], L["d"], L["C"], L["W"]
    sh = shard_units(units, world)[rank]
    BH, bh0 = sh.bh_count, sh.bh_begin
    cfg = eva.make_config(L["B"], L["H"], T, d, C, W, bh_begin=bh0, bh_count=BH)
    Q, K, V = eva_inputs.qkv(bh0, BH, T, d, torch.bfloat16, seed=0, device=dev)
    ks, vs = eva.eva_summarize(cfg, K, V)
    O = torch.empty_like(Q)
    lse = torch.empty(BH, T, dtype=torch.float32, device=dev)
    reps = max(3, min(args.steps, 20))
    for _ in range(2):
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O, lse=lse)
    torch.cuda.synchronize()
    if dist: dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, O=O, lse=lse)
    b.record(s)
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b) / reps, device=dev)
    gather_ms = None
    nccl = None
    if dist and world > 1:
      try:
        # O of every rank into one [units, T, d] buffer (equal shards when world | 256)
        per = (units + world - 1) // world
        buf = torch.zeros(per, T, d, dtype=torch.bfloat16, device=dev)
        buf[:BH].copy_(O)
        out = torch.empty(per * world, T, d, dtype=torch.bfloat16, device=dev)
        dist.all_gather_into_tensor(out, buf)
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(s)
        dist.all_gather_into_tensor(out, buf)
        g1.record(s)
        torch.cuda.synchronize()
        gather_ms = max_over_ranks(g0.elapsed_time(g1), device=dev)
        nccl = {"nranks": world, "backend": dist.get_backend(), "collective": "all_gather_into_tensor(O)",
                "bytes_per_rank": per * T * d * 2}
        del buf, out
      except Exception as exc:  # the gather is context, not the measured value: never fail the line on it
        nccl = {"nranks": world, "error": f"{type(exc).__name__}: {exc}"[:200]}
    pb = prefill_bytes(BH, T, d, C)
    pf = prefill_flops(BH, T, d, C, W)
    # per-rank ideal at the HBM roofline (the rank's algorithmic bytes / peak)
    out = {"workload": f"configs[2] strong-scaled: {units} units of T={T},d={d},C={C},W={W} split over "
                       f"{world} rank(s) ({BH} on rank {rank}); eva_attn_prefill, summaries provided",
           "units_total": units, "units_per_rank": BH, "ms": ms,
           "tokens_per_s_total": units // L["H"] * T / (ms / 1e3),
           "per_rank_alg_bytes": pb, "per_rank_ms_at_hbm_peak": pb / (peaks["hbm"] * 1e9) * 1e3,
           "roofline": {"bound": "hbm", "achieved": pb / (ms / 1e3) / 1e9, "peak": peaks["hbm"],
                        "unit": "GB/s", "frac": pb / (ms / 1e3) / 1e9 / peaks["hbm"],
                        "tensor_frac_of_bf16_peak": pf / (ms / 1e3) / 1e12 / peaks["bf16"]},
           "gather_o_ms": gather_ms, "nccl": nccl}
    del Q, K, V, O, ks, vs, lse
    torch.cuda.empty_cache()
    return out


SWEEP = [(4096, 128, 128), (16384, 64, 512), (65536, 32, 512), (65536, 64, 512),
         (131072, 32, 512), (131072, 64, 512), (131072, 128, 512)]


def bench_sweep(args, eva, torch, dev, s, rank, world, peaks):
    """configs[4] long-context cells (H=32 units of one sequence, d=128, sliding): T, C, W as in
    SWEEP.  Per cell: eva_attn_prefill with the summaries provided (the tensor-core kernel) and
    eva_summarize, device time (CUDA events), algorithmic flops / bytes as in the headline
    roofline, tensor fraction against the measured bf16 burst peak.  Each rank runs the whole
    cell on its own (weak)."""
    import eva_inputs
    H, d = 32, 128
    cells = []
    for (T, C, W) in (SWEEP if not args.quick else SWEEP[:2]):
        cfg = eva.make_config(1, H, T, d, C, W)
        Q, K, V = eva_inputs.qkv(0, H, T, d, torch.bfloat16, seed=0, device=dev)
        ks, vs = eva.eva_summarize(cfg, K, V)
        O = torch.empty_like(Q)
        lse = torch.empty(H, T, dtype=torch.float32, device=dev)
        eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, lse=lse)
        torch.cuda.synchronize()
        reps = 5
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(s)
        for _ in range(reps):
            eva.eva_summarize(cfg, K, V, Ksum=ks, Vsum=vs)
        e[1].record(s)
        for _ in range(reps):
            eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O, lse=lse)
        e[2].record(s)
        torch.cuda.synchronize()
        sm = e[0].elapsed_time(e[1]) / reps
        pm = e[1].elapsed_time(e[2]) / reps
        pf = prefill_flops(H, T, d, C, W)
        pb = prefill_bytes(H, T, d, C)
        cells.append({"T": T, "C": C, "W": W, "prefill_ms": pm, "summarize_ms": sm,
                      "tokens_per_s": T / ((pm + sm) / 1e3),
                      "tensor_tflops_alg": pf / (pm / 1e3) / 1e12,
                      "tensor_frac": pf / (pm / 1e3) / 1e12 / peaks["bf16"],
                      "hbm_frac": pb / (pm / 1e3) / 1e9 / peaks["hbm"]})
        del Q, K, V, O, ks, vs, lse
        torch.cuda.empty_cache()
    return {"workload": "configs[4]: B=1, H=32, d=128, sliding, bf16; cells (T, C, W)",
            "peak_bf16_tflops": peaks["bf16"], "peak_hbm_gbs": peaks["hbm"], "peak_source": peaks["src"],
            "cells": cells}

# ============================================================================ oracle (CPU) arm
def cpu_baseline(args, budget_s=12.0):
    """The fp64 oracle as it stands, on this host's cores, over whole workload passes
    (summaries + prefill of all B*H units + 1 decode row) until ~budget_s of CPU time."""
    import numpy as np
    import torch

    import eva_inputs
    import oracle

    wl = WORKLOAD
    B, H, T, d, C, W = (wl[k] for k in ("B", "H", "T", "d", "C", "W"))
    BH = B * H
    Q, K, V = (x.float().double().numpy() for x in eva_inputs.qkv(0, BH, T, d, torch.bfloat16, seed=0))
    E = oracle.eps_units(1234, 0, 0, BH, T // C, d)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    t0 = time.perf_counter()
    passes = 0
    while True:
        ks, vs = oracle.summarize_batch(K, V, E, C)
        oracle.prefill_batch(Q, K, V, ks, vs, C, W, 0, 1 / math.sqrt(d))
        passes += 1
        el = time.perf_counter() - t0
        if el >= budget_s or passes >= 50:
            break
    return {"value": passes * B * T / el, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{passes} full pass(es) of the configs[1] workload (summaries + prefill of all "
                      f"{BH} units, fp64 C oracle, OpenMP over units) in {el:.1f} s"}


def cpu_oracle_configs0():
    """BASELINE configs[0] (B=1, H=1, T=256, d=16, C=16, W=32, fp32): the fp64 oracle's time
    for the whole pass (summaries + prefill) on this host -- "CPU oracle in seconds"."""
    import torch

    import eva_inputs
    import oracle
    B, H, T, d, C, W = 1, 1, 256, 16, 16, 32
    Q, K, V = (x.double().numpy() for x in eva_inputs.qkv(0, B * H, T, d, torch.float32, seed=0))
    E = oracle.eps_units(1234, 0, 0, B * H, T // C, d)
    t0 = time.perf_counter()
    reps = 0
    while True:
        ks, vs = oracle.summarize_batch(K, V, E, C)
        oracle.prefill_batch(Q, K, V, ks, vs, C, W, 0, 1 / math.sqrt(d))
        reps += 1
        if time.perf_counter() - t0 > 1.0 or reps >= 1000:
            break
    sec = (time.perf_counter() - t0) / reps
    return {"workload": "configs[0]: B=1,H=1,T=256,d=16,C=16,W=32 (summaries + prefill)", "seconds": sec,
            "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), "kind": "oracle",
            "reps": reps}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    per_step = []
    import numpy as np  # noqa: F401
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(args, budget_s=0.0)  # one full pass per step
        if i >= args.warmup:
            per_step.append(r)
    wl = WORKLOAD
    tok = wl["B"] * wl["T"]
    secs = [tok / r["value"] for r in per_step]
    value = tok * len(secs) / sum(secs)
    return {"metric": "prefill tokens/s (FlashEVA hot path, whole job)", "impl": "reference",
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (same seeded inputs as our arm)",
            "config": {"workload": wl["name"], "B_per_gpu": wl["B"], "H": wl["H"], "T": wl["T"],
                       "d_head": wl["d"], "chunk": wl["C"], "window": wl["W"], "mode": "sliding",
                       "global_batch": wl["B"] * world,
                       "parallelism": "rank 0 only (host cores); the other ranks exit without work"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "kind": "oracle",
                             "cores": per_step[0]["cores"],
                             "sample": "each step = one full pass of the configs[1] workload on the fp64 oracle"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_stub(args, rank, world):
    """--stub: the N-rank plumbing of run_ours with every kernel replaced by a host sleep (gloo,
    CPU): shard bounds of the weak (configs[1]) and strong (configs[2]) legs, barrier-bracketed
    timing, max over ranks, the rank-0 line.  Used by tests/test_bench_launcher.py."""
    import torch  # noqa: F401
    from paper_2511_00576_b200.parallel import max_over_ranks, shard_for, shard_units
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    wl = WORKLOAD
    weak = shard_for(rank, world, wl["B"] * world, wl["H"])
    strong = shard_units(LARGE["B"] * LARGE["H"], world)[rank]
    if dist: dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(0.001 * (1 + rank))  # the slowest rank sets the time
    el = time.perf_counter() - t0
    if dist: dist.barrier()
    total_s = max_over_ranks(el)
    shards = [None] * world
    if dist:
        dist.all_gather_object(shards, (strong.bh_begin, strong.bh_count))
    else:
        shards = [(strong.bh_begin, strong.bh_count)]
    res = {"metric": "prefill tokens/s (FlashEVA hot path, whole job)", "stub": True,
           "value": world * wl["B"] * wl["T"] * args.steps / total_s, "unit": "tokens/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_s * 1e3 / args.steps,
           "higher_is_better": True, "scaling": "weak",
           "config": {"workload": wl["name"], "global_batch": wl["B"] * world,
                      "weak_shard_rank0": [weak.bh_begin, weak.bh_count] if rank == 0 else None,
                      "strong_shards": shards}}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return res


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="shorter decode extra (profiling)")
    ap.add_argument("--stub", action="store_true", help="launcher / multi-rank bookkeeping only (CPU, gloo)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--e2e-slices", type=int, default=1, help="unit slices of the host-copy pipeline (1: no overlap; see DESIGN.md §8)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # self-launch: one process per GPU under torch.distributed.run; rank 0's line passes through
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
        cmd += sys.argv[1:]
        sys.exit(subprocess.run(cmd).returncode)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"--gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.stub:
        res = run_stub(args, rank, world)
    elif args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
