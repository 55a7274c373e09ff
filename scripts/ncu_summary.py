"""Key metrics of an ncu --set full report (one row per captured launch).

    python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep [--stalls]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "occ_smem"),
    ("launch__occupancy_limit_registers", "occ_regs"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum", "l1_ld_bytes"),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        print(name[:110])
        for k, short in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {short:16s} {r[i]:>16s} {units[i]}")
    if "--stalls" in sys.argv:
        for r in rows[2:]:
            st = []
            for i, k in enumerate(hdr):
                if k.startswith("smsp__average_warp_latency_issue_stalled_") or \
                   k.startswith("smsp__pcsamp_warps_issue_stalled_"):
                    try:
                        v = float(r[i].replace(",", ""))
                    except ValueError:
                        continue
                    st.append((v, k))
            st.sort(reverse=True)
            for v, k in st[:14]:
                print(f"   {k:90s} {v:12.1f}")


if __name__ == "__main__":
    main()
