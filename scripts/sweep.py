"""BASELINE configs[4] long-context sweep on one GPU: T = 4k..128k, H = 32, d = 128,
C in {32, 64, 128}, W in {128, 512}, B = 131072 / T (constant 128k tokens per head, P:355's
constant-token protocol).  Times eva_summarize and eva_attn_prefill (tile kernel) with CUDA
events (L2 flushed between reps) and reports tokens/s and roofline fractions.

    python scripts/sweep.py [--out profiles/r01_sweep.json]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import eva_inputs
import paper_2511_00576_b200 as eva


def alg(BH, T, d, C, W):
    nC = T // C
    R = W // C
    keys = 0
    # sum over n of |E(n)| + nsum(n), closed form by chunk blocks
    for n in range(T):
        ns = max(0, n // C - R + 1)
        keys += (n - ns * C + 1) + ns
    return BH * (4 * T * d * 2 + 2 * nC * d * 2 + 4 * T), BH * keys * 4 * d


def main():
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    pp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    # measured peaks when the driver wrote them, else the fallback of B200_PROFILING.md
    peaks = json.load(open(pp)) if os.path.exists(pp) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
                                                            "source": "fallback"}
    H, d, tokens = 32, 128, 131072
    flush = torch.empty(512 << 18, device="cuda")
    rows = []
    for T in (4096, 8192, 16384, 32768, 65536, 131072):
        B = tokens // T
        Q, K, V = eva_inputs.qkv(0, B * H, T, d, torch.bfloat16, seed=0, device="cuda") if T >= 0 else None
        for C in (32, 64, 128):
            for W in (128, 512):
                if W < C:
                    continue
                cfg = eva.make_config(B, H, T, d, C, W)
                ks, vs = eva.eva_summarize(cfg, K, V)
                O = torch.empty_like(Q)
                for _ in range(2):
                    eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O)
                ts, tp = [], []
                for _ in range(5):
                    flush.zero_()
                    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                    e[0].record()
                    eva.eva_summarize(cfg, K, V, Ksum=ks, Vsum=vs)
                    e[1].record()
                    eva.eva_attn_prefill(cfg, Q, K, V, Ksum=ks, Vsum=vs, summaries_provided=True, O=O)
                    e[2].record()
                    torch.cuda.synchronize()
                    ts.append(e[0].elapsed_time(e[1]))
                    tp.append(e[1].elapsed_time(e[2]))
                s_ms, p_ms = statistics.median(ts), statistics.median(tp)
                pb, pf = alg(B * H, T, d, C, W)
                r = {"T": T, "B": B, "C": C, "W": W, "summarize_ms": s_ms, "prefill_ms": p_ms,
                     "tokens_per_s": B * T / ((s_ms + p_ms) / 1e3),
                     "prefill_hbm_frac": pb / (p_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                     "prefill_tensor_frac_alg": pf / (p_ms / 1e3) / 1e12 / peaks["bf16_tflops"],
                     "keys_per_query": pf / (B * H * T * 4 * d)}
                rows.append(r)
                print(json.dumps(r), flush=True)
                del ks, vs, O
        del Q, K, V
        torch.cuda.empty_cache()
    if out:
        with open(out, "w") as f:
            json.dump({"config": "BASELINE configs[4] on 1 GPU, tile prefill kernel, bf16, sliding",
                       "peaks": {"hbm_gbs": peaks["hbm_gbs"], "bf16_tflops": peaks["bf16_tflops"]},
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
