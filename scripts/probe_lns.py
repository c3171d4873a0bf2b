"""LNS throughput: batched neighbourhoods on the B200 vs the reference's OpenMP LNS on the host.

Runs the unmodified fdsolve CLI twice (oracle/_ref/fdsolve = CPU reference with --threads nproc,
adapter/_build/fdsolve_b200 = B200) on the same golomb instances and LNS settings, checks the
outputs agree (time_ms masked) and prints both wall times."""
import json
import os
import re
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_09213_b200 import models  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "fdsolve")
B200 = os.path.join(ROOT, "adapter", "_build", "fdsolve_b200")


def run(binary, args, threads):
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    t = time.perf_counter()
    p = subprocess.run([binary] + args, capture_output=True, text=True, env=env, timeout=1800)
    dt = time.perf_counter() - t
    ms = [float(x) for x in re.findall(r'"time_ms":\s*([0-9.]+)', p.stdout)]
    return p.returncode, re.sub(r'"time_ms":\s*[0-9.]+', '"time_ms":0', p.stdout), dt, (ms[-1] if ms else None)


def main():
    nproc = os.cpu_count() or 1
    cases = [("assign20", 10, 148, 0.4, 0), ("assign30", 5, 592, 0.35, 1000), ("assign40", 5, 1184, 0.3, 2000)]
    if len(sys.argv) > 1:
        cases = cases[: int(sys.argv[1])]
    with tempfile.TemporaryDirectory() as d:
        for name, iters, nbs, rate, limit in cases:
            path = os.path.join(d, name + ".fd")
            with open(path, "w") as f:
                f.write(models.named_instance(name))
            args = ["solve", path, "--lns", "--iters", str(iters), "--neighborhoods", str(nbs), "--destroy", str(rate),
                    "--node-limit", str(limit), "--seed", "1", "--json", "--stats", "--threads", str(nproc)]
            rc_g, out_g, t_g, ms_g = run(B200, args, 1)
            rc_r, out_r, t_r, ms_r = run(REF, args, nproc)
            print(json.dumps({"case": name, "iters": iters, "neighborhoods": nbs, "node_limit": limit,
                              "b200_wall_s": round(t_g, 3), "ref_wall_s": round(t_r, 3), "ref_threads": nproc,
                              "b200_solve_ms": ms_g, "ref_solve_ms": ms_r,
                              "speedup_solve": round(ms_r / ms_g, 2) if ms_g and ms_r else None, "identical": out_g == out_r and rc_g == rc_r == 0,
                              "b200_tail": out_g.strip().splitlines()[-1][:200] if out_g.strip() else ""}),
                  flush=True)


if __name__ == "__main__":
    main()
