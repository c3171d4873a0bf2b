"""Top CUDA source lines of an ncu report by warp-stall samples (and executed instructions).

usage: python scripts/ncu_lines.py REPORT.ncu-rep [TOP]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    samples, insts = defaultdict(int), defaultdict(int)
    src = {}
    path = "?"
    cur = None
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur = (path, int(r[0]))
            src[cur] = r[1].strip()[:90]
            continue
        if cur is None or r[2] in ("...", "-"):
            continue
        try:
            samples[cur] += int(r[4])
            insts[cur] += int(r[7])
        except ValueError:
            pass
    tot_s = sum(samples.values()) or 1
    tot_i = sum(insts.values()) or 1
    print(f"total samples {tot_s}  total warp instructions {tot_i}")
    for k, v in sorted(samples.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / tot_s:6.2f}% smp {100 * insts[k] / tot_i:6.2f}% inst  {k[0]}:{k[1]:<5d} {src.get(k, '')}")


if __name__ == "__main__":
    main()
