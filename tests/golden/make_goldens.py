"""Generate the golden fixtures by running the UNMODIFIED reference solver.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/make_goldens.py [--long]

Outputs (committed, small):
  tests/golden/models/*.fd          pinned model texts (sha256-checked against SURVEY.md)
  tests/golden/goldens.json         stats + first/optimal solution per (instance, mode)
  tests/golden/corpus.json          per-seed results on the reference test corpora:
                                    all solutions, fixpoints (GAC and FC), first solution,
                                    input-order stats, branch-and-bound optima
The reference binary is oracle/_ref/fdref_driver (see oracle/Makefile and oracle/ref_driver.cpp).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_1909_09213_b200 import models  # noqa: E402

DRIVER = os.path.join(ROOT, "oracle", "_ref", "fdref_driver")
MODELS = os.path.join(HERE, "models")

NAMED = ["nq4", "nq6", "nq8", "nq10", "nq12", "nq14", "nq24", "nq40",
         "golomb5", "golomb6", "golomb7", "golomb8", "golomb9", "golomb10",
         "magic3", "magic4", "magic5", "rcsp_1000", "rcsp_10000", "rcsp_100000"]

# (instance, flags, long?)  -- flags are fdref_driver solve flags
CASES = [
    ("nq4", ["--all"], False), ("nq6", ["--all"], False), ("nq8", ["--all"], False),
    ("nq8", ["--max", "1"], False), ("nq10", ["--all"], False), ("nq12", ["--all"], False),
    ("nq14", ["--max", "1"], False), ("nq24", ["--max", "1"], False), ("nq40", ["--max", "1"], False),
    ("nq8", ["--all", "--fc"], False), ("nq8", ["--all", "--input"], False),
    ("nq10", ["--all", "--node-limit", "1000"], False),
    ("golomb5", [], False), ("golomb6", [], False), ("golomb7", [], False), ("golomb8", [], False),
    ("golomb9", [], False), ("golomb7", ["--max", "1"], False),
    ("magic3", ["--all"], False), ("magic4", ["--max", "1"], False), ("magic5", ["--max", "1"], False),
    ("magic5", ["--max", "1", "--node-limit", "500"], False),
    ("magic4", ["--all", "--node-limit", "20000"], False),
    ("rcsp_10000", ["--max", "1", "--node-limit", "200"], False),
    ("rcsp_100000", ["--max", "1", "--node-limit", "200"], False),
    ("nq14", ["--all", "--node-limit", "200000"], False),
    # long runs (minutes each on one core)
    ("nq14", ["--all"], True), ("golomb10", [], True), ("magic4", ["--all"], True),
    ("rcsp_1000", ["--max", "1"], True),
]


def run(args, timeout=3600):
    r = subprocess.run([DRIVER] + args, capture_output=True, text=True, timeout=timeout,
                       preexec_fn=lambda: __import__("resource").setrlimit(
                           __import__("resource").RLIMIT_STACK, (-1, -1)))
    if r.returncode != 0:
        raise RuntimeError(f"{args}: {r.stderr}")
    return json.loads(r.stdout)


def case_key(inst, flags):
    return inst + ("|" + " ".join(flags) if flags else "")


def write_models():
    os.makedirs(MODELS, exist_ok=True)
    for name in NAMED:
        with open(os.path.join(MODELS, name + ".fd"), "w") as f:
            f.write(models.named_instance(name))


def solve_text(text, flags):
    with tempfile.NamedTemporaryFile("w", suffix=".fd", delete=False) as f:
        f.write(text)
        path = f.name
    try:
        return run(["solve", path] + flags)
    finally:
        os.unlink(path)


def fixpoint_text(text, flags):
    with tempfile.NamedTemporaryFile("w", suffix=".fd", delete=False) as f:
        f.write(text)
        path = f.name
    try:
        return run(["fixpoint", path] + flags)
    finally:
        os.unlink(path)


def corpus_record(seed):
    text = models.corpus_instance(seed)
    rec = {
        "all": solve_text(text, ["--all", "--solutions"]),
        "all_fc": solve_text(text, ["--all", "--fc"]),
        "all_input": solve_text(text, ["--all", "--input"]),
        "first": solve_text(text, ["--max", "1"]),
        "fix_gac": fixpoint_text(text, []),
        "fix_fc": fixpoint_text(text, ["--fc"]),
    }
    return rec


def opt_record(seed):
    text, goal = models.optimization_instance(seed)
    return solve_text(models.with_goal(text, goal), [])


def random_record(seed):
    text, _ = models.random_instance(seed)
    return solve_text(text, ["--all", "--solutions"])


def main():
    long_runs = "--long" in sys.argv
    write_models()
    gpath = os.path.join(HERE, "goldens.json")
    goldens = json.load(open(gpath)) if os.path.exists(gpath) else {}
    todo = [(i, f) for (i, f, lng) in CASES if (long_runs or not lng)]
    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        futs = {ex.submit(run, ["solve", os.path.join(MODELS, i + ".fd")] + f): (i, f) for i, f in todo}
        for fut, (i, f) in futs.items():
            res = fut.result()
            goldens[case_key(i, f)] = res
            print(case_key(i, f), {k: res.get(k) for k in ("nodes", "failures", "rounds", "solutions", "time_ms")},
                  flush=True)
    with open(gpath, "w") as f:
        json.dump(goldens, f, indent=1, sort_keys=True)

    corpus = {"corpus": {}, "optimization": {}, "random": {}}
    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        cs = list(ex.map(corpus_record, range(200)))
        os_ = list(ex.map(opt_record, range(50)))
        rs = list(ex.map(random_record, range(100, 140)))
    for s, r in enumerate(cs):
        corpus["corpus"][str(s)] = r
    for s, r in enumerate(os_):
        corpus["optimization"][str(s)] = r
    for s, r in zip(range(100, 140), rs):
        corpus["random"][str(s)] = r
    for grp in corpus.values():
        for r in grp.values():
            for sub in (r.values() if "nodes" not in r else [r]):
                if isinstance(sub, dict):
                    sub.pop("time_ms", None)
    with open(os.path.join(HERE, "corpus.json"), "w") as f:
        json.dump(corpus, f, sort_keys=True, separators=(",", ":"))
    print("wrote", gpath)


if __name__ == "__main__":
    main()
