"""Sum per-launch ncu metrics of our kernels over one step and record them for bench.py.
usage: python scripts/ncu_step_counts.py REPORT.ncu-rep INSTANCE NODES [OUT.json]
NODES: the reference's node count of the step's answer (the bench value's node basis)."""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "": 1, "nsecond": 1, "usecond": 1e3,
         "msecond": 1e6}


def main():
    rep, inst, nodes = sys.argv[1], sys.argv[2], int(sys.argv[3])
    out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                              "r02_ncu_traffic.json")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    keys = {"dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
            "smsp__inst_executed.sum": "inst_executed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
            "gpu__time_duration.sum": "duration_ns_under_ncu"}
    tot = {v: 0.0 for v in keys.values()}
    n = 0
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")
        if "search_kernel" not in name and "propagate_kernel" not in name:
            continue
        n += 1
        for k, v in keys.items():
            if k in d and d[k] not in ("", "n/a"):
                u = units[hdr.index(k)]
                tot[v] += float(d[k].replace(",", "")) * SCALE.get(u, 1)
    rec = {"kernel": f"{n} search launches (one step, summed)", **tot, "nodes": nodes, "report": os.path.basename(rep),
           "per": "step"}
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[inst] = rec
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
