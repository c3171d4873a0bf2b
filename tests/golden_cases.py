"""Shared helpers: load the golden fixtures (made by the unmodified reference) and map their
fdref_driver flags to a SearchConfig."""
from __future__ import annotations

import json
import os

from paper_1909_09213_b200 import solver as S

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def goldens():
    with open(os.path.join(GOLDEN, "goldens.json")) as f:
        return json.load(f)


def corpus():
    with open(os.path.join(GOLDEN, "corpus.json")) as f:
        return json.load(f)


def model_text(inst: str) -> str:
    with open(os.path.join(GOLDEN, "models", inst + ".fd")) as f:
        return f.read()


def cfg_from_flags(flags) -> S.SearchConfig:
    c = S.SearchConfig()
    i = 0
    while i < len(flags):
        f = flags[i]
        if f == "--max":
            c.max_solutions = int(flags[i + 1])
            i += 1
        elif f == "--fc":
            c.alldiff = 0
        elif f == "--input":
            c.var_heuristic = 0
        elif f == "--node-limit":
            c.node_limit = int(flags[i + 1])
            i += 1
        i += 1
    return c


def split_key(key: str):
    inst, _, fl = key.partition("|")
    return inst, fl.split()


def expected_tuple(g):
    return (g["nodes"], g["failures"], g["rounds"], g["solutions"])


# golden cases the CPU oracle port finishes in a few seconds
FAST_CASES = [
    "nq4|--all", "nq6|--all", "nq8|--all", "nq8|--max 1", "nq8|--all --fc", "nq8|--all --input",
    "nq10|--all --node-limit 1000", "nq14|--max 1", "nq24|--max 1", "nq40|--max 1",
    "golomb5", "golomb6", "golomb7", "golomb7|--max 1", "golomb8", "magic3|--all", "magic4|--max 1",
    "magic5|--max 1", "magic5|--max 1 --node-limit 500", "rcsp_10000|--max 1 --node-limit 200",
]
