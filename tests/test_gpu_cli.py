"""The reference's own CLI (tools/fdsolve.cpp, unmodified; CLI11 replaced by adapter/shim) built
twice: over the reference library (oracle/_ref/fdsolve, CPU) and over the drop-in adapter
(adapter/_build/fdsolve_b200, B200). Outputs must be identical byte for byte except time_ms."""
import os
import re
import resource
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "fdsolve")
B200 = os.path.join(ROOT, "adapter", "_build", "fdsolve_b200")
M = os.path.join(ROOT, "tests", "golden", "models")

CASES = [
    ["solve", f"{M}/nq8.fd"],
    ["solve", f"{M}/nq8.fd", "--all", "--stats"],
    ["solve", f"{M}/nq8.fd", "--all", "--json"],
    ["solve", f"{M}/nq8.fd", "--first", "5", "--stats"],
    ["solve", f"{M}/nq8.fd", "--all", "--heuristic", "input", "--stats"],
    ["solve", f"{M}/nq10.fd", "--all", "--stats"],
    ["solve", f"{M}/golomb7.fd", "--all", "--stats"],
    ["solve", f"{M}/golomb7.fd", "--stats"],
    ["solve", f"{M}/golomb6.fd", "--lns", "--iters", "3", "--neighborhoods", "2", "--seed", "3", "--stats"],
    ["solve", f"{M}/golomb6.fd", "--lns", "--iters", "2", "--destroy", "0.5", "--node-limit", "40", "--json"],
    ["solve", f"{M}/golomb7.fd", "--lns", "--iters", "4", "--neighborhoods", "16", "--seed", "11", "--stats"],
    ["solve", f"{M}/golomb7.fd", "--lns", "--iters", "3", "--neighborhoods", "9", "--destroy", "0.6",
     "--node-limit", "150", "--json"],
    ["solve", f"{M}/assign20.fd", "--lns", "--iters", "5", "--neighborhoods", "32", "--destroy", "0.4", "--stats"],
    ["solve", f"{M}/assign30.fd", "--lns", "--iters", "3", "--neighborhoods", "64", "--destroy", "0.35",
     "--node-limit", "1000", "--seed", "4", "--json", "--stats"],
    ["solve", f"{M}/magic3.fd", "--all", "--json"],
    ["solve", f"{M}/magic4.fd", "--stats"],
    ["gen-nqueens", "6"],
    ["gen-random", "--vars", "5", "--width", "6", "--constraints", "7", "--seed", "9"],
    ["solve", f"{M}/does_not_exist.fd"],
    ["solve", f"{M}/nq8.fd", "--heuristic", "bad"],
]


def _run(binary, args):
    def lim():
        resource.setrlimit(resource.RLIMIT_STACK, (resource.RLIM_INFINITY, resource.RLIM_INFINITY))

    r = subprocess.run([binary] + args, capture_output=True, text=True, timeout=300, preexec_fn=lim)
    norm = lambda s: re.sub(r'time_ms[=":]+\d+', "time_ms=T", s)  # noqa: E731
    return r.returncode, norm(r.stdout), norm(r.stderr)


@pytest.mark.parametrize("args", CASES, ids=[" ".join(a[:1] + [os.path.basename(x) for x in a[1:]]) for a in CASES])
def test_fdsolve_on_b200_matches_reference_cli(args):
    assert os.path.exists(B200) and os.path.exists(REF), "build with __graft_entry__.build() in the build container"
    assert _run(B200, args) == _run(REF, args)
