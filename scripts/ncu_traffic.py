"""Record the DRAM traffic of the search kernel from one `ncu --set full` capture.

usage: python scripts/ncu_traffic.py REPORT.ncu-rep INSTANCE [OUT.json]
Writes {INSTANCE: {"dram_read_bytes", "dram_write_bytes", "kernel", "report"}} into
profiles/r02_ncu_traffic.json (bench.py reads it for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    rep, inst = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                              "r02_ncu_traffic.json")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    rec = None
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if "search_kernel" not in d.get("Kernel Name", ""):
            continue
        u = dict(zip(hdr, units))
        val = lambda k: float(d[k].replace(",", "")) * SCALE[u[k]]
        rec = {"kernel": d["Kernel Name"], "dram_read_bytes": val("dram__bytes_read.sum"),
               "dram_write_bytes": val("dram__bytes_write.sum"),
               "duration_ns_under_ncu": float(d["gpu__time_duration.sum"].replace(",", "")) *
               {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}[u["gpu__time_duration.sum"]],
               "report": os.path.basename(rep)}
    if rec is None:
        sys.exit("no search_kernel in " + rep)
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[inst] = rec
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
