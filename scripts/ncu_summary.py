"""Summarise an ncu --set full report: one block per profiled launch with the
metrics the roofline argument uses (time, DRAM bytes / throughput, SM and
pipe utilisation, occupancy, registers) and the top warp-stall reasons.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/…txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active", "fmaheavy_pipe_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(path):
    hdr, units, rows = raw(path)
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
    if not stall:
        stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    for r in rows:
        name = r[idx["Kernel Name"]]
        print(f"== {name[:90]}")
        for m, short in METRICS:
            if m in idx:
                print(f"   {short:20s} {r[idx[m]]:>14s} {units[idx[m]]}")
        vals = []
        for h in stall:
            try:
                vals.append((float(r[idx[h]].replace(",", "")), h))
            except ValueError:
                pass
        vals.sort(reverse=True)
        if vals:
            tot = sum(v for v, _ in vals) or 1.0
            top = ", ".join(f"{h.split('stalled_')[1].split('.')[0]} {100 * v / tot:.0f}%" for v, h in vals[:5])
            print(f"   top stalls           {top}")


if __name__ == "__main__":
    main(sys.argv[1])
