"""Stall breakdown of an ncu --set full report from its SASS page: totals per stall reason and
the top instructions by samples (dev tool).   python scripts/sass_stalls.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

NAMES = ['stall_barrier', 'stall_branch_resolving', 'stall_dispatch', 'stall_drain', 'stall_lg', 'stall_long_sb',
         'stall_math', 'stall_membar', 'stall_mio', 'stall_misc', 'stall_no_inst', 'stall_not_selected',
         'stall_selected', 'stall_short_sb', 'stall_sleep', 'stall_tex', 'stall_wait']


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    idx = {n: hdr.index(n) for n in NAMES if n in hdr}
    data = rows[2:]
    tot = {n: sum(int(r[i] or 0) for r in data) for n, i in idx.items()}
    allv = sum(tot.values()) or 1
    print(rows[0][0][:120] if rows[0] else "")
    print("instructions:", len(data), " executed:", sum(int(r[iex] or 0) for r in data))
    for n, v in sorted(tot.items(), key=lambda x: -x[1]):
        if v:
            print(f"  {n:24s} {v:9d}  {100.0 * v / allv:5.1f} %")
    print("top instructions (samples, executed, sass):")
    base = int(data[0][ia], 16)
    for r in sorted(data, key=lambda r: -int(r[iss] or 0))[:top]:
        print(f"  {int(r[iss] or 0):7d} {int(r[iex] or 0):11d}  +{int(r[ia], 16) - base:06x}  {r[isrc][:80]}")


if __name__ == "__main__":
    main()
