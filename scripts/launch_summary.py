"""Summarise an ncu launch list (gpu__time_duration.sum) by kernel: count, avg, share.

    python scripts/launch_summary.py gpurun_out/launches_r01.csv [--ours]
"""
import collections
import csv
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    out = []
    for r in rows[1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            out.append((r[ki], float(r[vi].replace(",", ""))))
    return out


def short(name):
    n = name.replace("void ", "")
    if "eva::" in n or "prefill_sm100" in n:
        n = n.split("(")[0]
        return n.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return "torch/other: " + n.split("<")[0].split("(")[0][:60]


def main():
    path = sys.argv[1]
    ours = "--ours" in sys.argv
    agg = collections.OrderedDict()
    for name, t in load(path):
        s = short(name)
        if ours and s.startswith("torch/other"):
            continue
        a = agg.setdefault(s, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'avg_us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:70]:70s} {n:8d} {t / n / 1e3:9.2f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main()
