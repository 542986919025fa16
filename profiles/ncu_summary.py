"""Summarise an ncu report: key metrics + stall reasons (used for profiles/*.md).

    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "SM Frequency", "Memory Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler",
        "No Eligible", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "gpu__time_duration.sum"]


def run(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                          text=True).stdout


def main(rep):
    rows = list(csv.DictReader(io.StringIO(run(rep, "details"))))
    kname = rows[0]["Kernel Name"] if rows else "?"
    print(f"kernel: {kname[:110]}")
    seen = set()
    for r in rows:
        n = r.get("Metric Name", "")
        if n in KEYS and n not in seen:
            seen.add(n)
            print(f"  {n:40s} {r['Metric Value']:>16s} {r['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run(rep, "raw"))))
    h, v = raw[0], raw[2]
    print("  -- raw")
    stalls = {}
    for i, n in enumerate(h):
        if n in RAW:
            print(f"  {n:70s} {v[i]}")
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    print("  -- warp-state samples (share)")
    for k, x in sorted(stalls.items(), key=lambda t: -t[1])[:10]:
        print(f"  {k:30s} {x / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
