"""Summarise an ncu report: SOL / occupancy / stall mix / instruction mix per
warp-iteration. Usage: python tools/ncu_summary.py REPORT.ncu-rep [warp_iters]"""
import collections
import csv
import io
import re
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    witers = float(sys.argv[2]) if len(sys.argv) > 2 else None
    det = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = det[0]
    keep = ["Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput",
            "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput",
            "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
            "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler",
            "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Executed Instructions", "Dynamic Shared Memory Per Block"]
    for row in det[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in keep:
            print(f"{d['Metric Name']:<40} {d['Metric Value']:>16} {d.get('Metric Unit', '')}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    rh, ru, rv = raw[0], raw[1], raw[2]
    for name in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                 "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                 "smsp__inst_executed.sum"]:
        if name in rh:
            i = rh.index(name)
            print(f"{name:<60} {rv[i]:>16} {ru[i]}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source",
                                            "sass"]))))
    h, data = src[1], src[2:]
    cats = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    iE = h.index("Instructions Executed")
    tot = {c: sum(int(r[h.index(c)] or 0) for r in data) for c in cats}
    T = sum(tot.values()) or 1
    print("stall mix:", ", ".join(f"{c[6:]} {100 * v / T:.1f}%" for c, v in
                                  sorted(tot.items(), key=lambda x: -x[1])[:8]))
    ops = collections.Counter()
    for r in data:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1])
        ops[m.group(2) if m else "?"] += int(r[iE] or 0)
    total = sum(ops.values())
    if witers:
        print(f"instructions per warp-iteration: {total / witers:.1f}")
        print("  " + ", ".join(f"{k} {v / witers:.1f}" for k, v in ops.most_common(16)))


if __name__ == "__main__":
    main()
