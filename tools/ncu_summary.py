"""Summarise an `ncu --set full` report (.ncu-rep) into the numbers we judge by:
duration, DRAM traffic, pipe utilisation, issue, occupancy, stall reasons and
the top stalled SASS lines. Usage: python tools/ncu_summary.py rep.ncu-rep > out.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep):
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("kernel:", name[:150])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {row[i]:>16s} {units[i]}")
    det = list(csv.reader(io.StringIO(ncu([rep, "--page", "details", "--csv"]))))
    print("details:")
    for row in det[1:]:
        if len(row) > 14 and row[12] in ("Issued Ipc Active", "No Eligible", "Eligible Warps Per Scheduler",
                                          "Warp Cycles Per Issued Instruction", "Achieved Occupancy",
                                          "Theoretical Occupancy"):
            print(f"  {row[12]:45s} {row[14]:>10s} {row[13]}")
    src = ncu([rep, "--page", "source", "--csv", "--print-source", "sass"])
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) > 2:
        h = rows[1]
        ia, isrc = h.index("Address"), h.index("Source")
        iall = h.index("Warp Stall Sampling (All Samples)")
        data = rows[2:]
        tot = sum(float(r[iall] or 0) for r in data) or 1
        print("top warp-stall SASS lines (share of all samples):")
        for r in sorted(data, key=lambda r: -float(r[iall] or 0))[:16]:
            print(f"  {100 * float(r[iall] or 0) / tot:5.1f}%  {r[isrc].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
