"""Golden sha256 of complete solution streams, produced by the UNMODIFIED reference solver.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/make_stream_hashes.py [--long]

For each case the reference (oracle/_ref/fdref_driver --solutions-bin) writes every solution it
hands to the callback, in callback order (search.cpp:134-156, DFS order), as little-endian int64
rows. The committed fixture keeps only the row count and the sha256 of those bytes
(tests/golden/stream_hashes.json); the GPU tests hash the int64 array cubics_enumerate returns
and compare (tests/test_gpu_headline.py). nq14 all takes ~200 s on one core (--long).
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "fdref_driver")
MODELS = os.path.join(HERE, "models")
OUT = os.path.join(HERE, "stream_hashes.json")

# (case key, instance, flags, long?)
CASES = [
    ("nq8|--all", "nq8", ["--all"], False),
    ("nq10|--all", "nq10", ["--all"], False),
    ("nq12|--all", "nq12", ["--all"], False),
    ("magic3|--all", "magic3", ["--all"], False),
    ("magic4|--all", "magic4", ["--all"], True),
    ("nq14|--all", "nq14", ["--all"], True),
]


def one(case):
    key, inst, flags, _ = case
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "sols.bin")
        r = subprocess.run([DRIVER, "solve", os.path.join(MODELS, inst + ".fd")] + flags + ["--solutions-bin", path],
                           capture_output=True, text=True, check=True,
                           preexec_fn=lambda: __import__("resource").setrlimit(
                               __import__("resource").RLIMIT_STACK, (-1, -1)))
        res = json.loads(r.stdout)
        h = hashlib.sha256()
        size = 0
        with open(path, "rb") as f:
            for chunk in iter(lambda: f.read(1 << 20), b""):
                h.update(chunk)
                size += len(chunk)
    n_vars = len(res["first"]) if "first" in res else 0
    rec = {"sha256": h.hexdigest(), "rows": res["solutions"], "n_vars": n_vars, "bytes": size,
           "stats": [res["nodes"], res["failures"], res["rounds"], res["solutions"]],
           "first": res.get("first"), "reference_ms": res["time_ms"]}
    assert size == 8 * n_vars * res["solutions"], (key, size)
    return key, rec


def main():
    long_runs = "--long" in sys.argv
    todo = [c for c in CASES if long_runs or not c[3]]
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    with ThreadPoolExecutor(max_workers=len(todo)) as ex:
        for key, rec in ex.map(one, todo):
            out[key] = rec
            print(key, rec["rows"], rec["sha256"][:16], f"{rec['reference_ms']:.0f} ms", flush=True)
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
