"""Pin the instance generators to the reference's own output (run in the build container, where
oracle/_ref/fdref_driver - the unmodified reference generators - is built).

    python tests/golden/make_generator_fixtures.py   -> tests/golden/generators.json

Stores the sha256 of every generated model text: fd::gen_nqueens (generators.cpp:13-33),
fd::gen_random (generators.cpp:35-112) over a parameter grid, and the acceptance corpus
(acceptance.cpp:47-54, via `fdref_driver corpus`); null where the reference rejects the
parameters (it aborts). tests/test_models.py checks
paper_1909_09213_b200/models.py against them byte for byte.
"""
import hashlib
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "..", "oracle", "_ref", "fdref_driver")

NQ = list(range(1, 41))
RANDOM = [(v, w, c, s) for v in (1, 2, 5, 12, 40) for w in (1, 2, 7, 33, 64) for c in (0, 1, 6, 30) for s in (0, 1, 99)]
CORPUS = list(range(200))


def run(*args):
    r = subprocess.run([DRIVER, *map(str, args)], capture_output=True, text=True)
    return r.stdout if r.returncode == 0 else None  # the reference rejects the parameters


def h(text):
    return None if text is None else hashlib.sha256(text.encode()).hexdigest()


def main():
    out = {
        "nqueens": {str(n): h(run("gen-nqueens", n)) for n in NQ},
        "random": {",".join(map(str, p)): h(run("gen-random", *p)) for p in RANDOM},
        "corpus": {str(s): h(run("corpus", s)) for s in CORPUS},
    }
    with open(os.path.join(HERE, "generators.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print({k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
