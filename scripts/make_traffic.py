"""Write profiles/ncu_traffic.json (dram__bytes_read.sum + dram__bytes_write.sum per launch)
from the `ncu --set full` captures of a round.   python scripts/make_traffic.py r01g"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, r = rows[0], rows[1], rows[2]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        tot += float(r[i].replace(",", "")) * UNIT[units[i]]
    ti = hdr.index("gpu__time_duration.sum")
    t_us = float(r[ti].replace(",", "")) * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                                           "nsecond": 1e-3, "second": 1e6}.get(units[ti], 1.0)
    return tot, t_us, r[hdr.index("Kernel Name")].split("(")[0]


def main():
    tag = sys.argv[1]
    res = {"note": f"one `ncu --set full --clock-control none` capture per kernel, round tag {tag}; "
                   "bytes are per launch (cold L2 under ncu replay)"}
    for key in ("prefill_configs1", "prefill_configs2", "decode_configs3", "summarize_configs2", "bwd_main"):
        rep = f"gpurun_out/prof_{key}_{tag}.ncu-rep"
        if os.path.exists(rep):
            b, t, name = dram_bytes(rep)
            res[key] = {"kernel": name, "dram_bytes_per_launch": b, "ncu_time_us": t}
    with open("profiles/ncu_traffic.json", "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
