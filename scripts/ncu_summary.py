"""Summarise an ncu report (``--set full``) into the text committed under profiles/.

usage: python scripts/ncu_summary.py REPORT.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Registers Per Thread", "Block Size", "Grid Size", "Theoretical Occupancy", "Achieved Occupancy",
        "Achieved Active Warps Per SM", "Dynamic Shared Memory Per Block", "Branch Efficiency"]


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
    hdr = rows[0]
    print(f"# ncu --set full summary of {rep}")
    kernel = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if kernel != d.get("Kernel Name"):
            kernel = d.get("Kernel Name")
            print(f"\n## kernel: {kernel}")
        if d.get("Metric Name") in KEYS:
            print(f"  {d['Metric Name']:40s} {d['Metric Value']:>18s} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
    if len(raw) > 2:
        names, units, vals = raw[0], raw[1], raw[2]
        print("\n## raw counters")
        for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
            if want in names:
                i = names.index(want)
                print(f"  {want:55s} {vals[i]:>18s} {units[i]}")
    # hottest source lines (CUDA view) by warp-stall samples and executed instructions
    src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    out, cur, hdr = [], None, None
    for r in src:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0] and len(r) > 8:
            try:
                out.append((cur, int(r[0]), int(r[4]), int(r[7]), r[1].strip()[:100]))
            except ValueError:
                pass
    if out:
        ts = sum(o[2] for o in out) or 1
        ti = sum(o[3] for o in out) or 1
        print("\n## top source lines by warp-stall samples (share of samples / of executed instructions)")
        for o in sorted(out, key=lambda o: -o[2])[:30]:
            print(f"  {o[0]:18s}:{o[1]:<5d} {100 * o[2] / ts:5.1f}% {100 * o[3] / ti:5.1f}%  {o[4]}")


if __name__ == "__main__":
    main()
