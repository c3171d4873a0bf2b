"""Instance generators in the reference's model-text format.

These produce the *inputs* of the hot path; they are not accelerated.

* ``gen_nqueens`` restates ``fd::gen_nqueens`` (reference ``proj/src/generators.cpp:13-33``).
* ``gen_random`` restates ``fd::gen_random`` (``proj/src/generators.cpp:35-112``) on top of
  ``Rng``, a restatement of the reference's splitmix64 (``proj/include/fd/rng.hpp:12-43``).
  Both are pinned byte-for-byte against the reference's own generator output by
  ``tests/test_models.py`` (fixtures written by ``tests/golden/make_goldens.py``).
* ``corpus_instance`` / ``random_instance`` / ``optimization_instance`` restate the seeded
  corpora of the reference's tests (``tests/acceptance.cpp:47-54``,
  ``tests/test_search.cpp:41-55``, ``tests/acceptance.cpp:408-419``).
* ``golomb``, ``magic`` and ``rcsp`` are the pinned SURVEY.md Appendix-B scripts (the
  reference ships no model text for them).
"""
from __future__ import annotations

import random

MASK64 = (1 << 64) - 1


class Rng:
    """splitmix64, as ``fd::Rng`` (rng.hpp:12-43)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    @staticmethod
    def _mix(z: int) -> int:
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    @classmethod
    def derive(cls, seed: int, a: int, b: int) -> "Rng":
        r = cls(seed)
        r.state ^= cls._mix((a + 0x9E3779B97F4A7C15) & MASK64)
        r.state ^= cls._mix((b + 0xBF58476D1CE4E5B9) & MASK64)
        return r

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        return self._mix(self.state)

    def below(self, n: int) -> int:
        return self.next() % n

    def range(self, lo: int, hi: int) -> int:
        return lo + self.below((hi - lo + 1) & MASK64)


def gen_nqueens(n: int) -> str:
    if n < 1:
        raise ValueError("n-queens requires n >= 1")
    out = [f"var q{i} in 1..{n};" for i in range(1, n + 1)]
    if n >= 2:
        out.append("constraint alldifferent(" + ", ".join(f"q{i}" for i in range(1, n + 1)) + ");")
        for i in range(1, n + 1):
            for j in range(i + 1, n + 1):
                d = j - i
                out.append(f"constraint q{i} != q{j} + {d};")
                out.append(f"constraint q{i} != q{j} - {d};")
    out.append("solve satisfy;")
    return "\n".join(out) + "\n"


def gen_random(nvars: int, width: int, ncons: int, seed: int) -> str:
    if nvars < 1 or width < 1 or ncons < 1:
        raise ValueError("gen_random requires vars, width and constraints >= 1")
    rng = Rng.derive(seed, 0xABCDEF, 0x123456)
    out = []
    ranges = []
    for i in range(nvars):
        lo = rng.range(-5, 5)
        w = rng.range(1, width)
        hi = lo + w - 1
        ranges.append((lo, hi))
        out.append(f"var v{i} in {lo}..{hi};")
    rel_ops = ["<", "<=", ">", ">=", "=", "!="]
    for _ in range(ncons):
        kind = rng.below(3 if nvars >= 2 else 2)
        if kind == 0:
            x = rng.below(nvars)
            op = rel_ops[rng.below(6)]
            if nvars >= 2 and rng.below(2) == 0:
                y = rng.below(nvars)
                line = f"constraint v{x} {op} v{y}"
                if rng.below(2) == 0:
                    off = rng.range(1, 3)
                    line += (" + " if rng.below(2) == 0 else " - ") + str(off)
                out.append(line + ";")
            else:
                lit = rng.range(ranges[x][0] - 1, ranges[x][1] + 1)
                out.append(f"constraint v{x} {op} {lit};")
        elif kind == 1:
            nterms = rng.below(min(nvars, 3)) + 1
            line = "constraint "
            max_sum = 0
            for t in range(nterms):
                coeff = rng.range(1, 3)
                if rng.below(4) == 0:
                    coeff = -coeff
                v = rng.below(nvars)
                if t == 0:
                    if coeff != 1:
                        line += f"{coeff}*"
                else:
                    line += " - " if coeff < 0 else " + "
                    if coeff not in (1, -1):
                        line += f"{abs(coeff)}*"
                line += f"v{v}"
                c1, c2 = coeff * ranges[v][0], coeff * ranges[v][1]
                max_sum += max(c1, c2)
            eq = rng.below(4) == 0
            bound = rng.range(-2, max(max_sum, -1))
            line += (" = " if eq else " <= ") + str(bound)
            out.append(line + ";")
        else:
            count = rng.below(nvars - 1) + 2
            ids = list(range(nvars))
            members = []
            for i in range(count):
                j = i + rng.below(nvars - i)
                ids[i], ids[j] = ids[j], ids[i]
                members.append(f"v{ids[i]}")
            out.append("constraint alldifferent(" + ", ".join(members) + ");")
    out.append("solve satisfy;")
    return "\n".join(out) + "\n"


def corpus_instance(seed: int) -> str:
    """acceptance.cpp:47-54: <= 6 vars, <= 10 values per domain, <= 8 constraints."""
    rng = Rng((seed * 7919 + 13) & MASK64)
    nvars = rng.below(5) + 2
    width = rng.below(9) + 2
    ncons = rng.below(8) + 1
    return gen_random(nvars, width, ncons, seed)


def random_instance(seed: int, optimization: bool = False) -> tuple[str, tuple | None]:
    """test_search.cpp:41-55. Returns (text, goal) where goal is ('min'|'max', var) or None."""
    rng = Rng(seed)
    nvars = rng.below(5) + 2
    width = rng.below(8) + 2
    ncons = rng.below(6) + 1
    text = gen_random(nvars, width, ncons, seed)
    goal = None
    if optimization:
        obj = rng.below(nvars)
        goal = ("min", obj) if rng.below(2) == 0 else ("max", obj)
    return text, goal


def optimization_instance(seed: int) -> tuple[str, tuple]:
    """acceptance.cpp:408-419."""
    rng = Rng((seed * 31 + 5) & MASK64)
    nvars = rng.below(4) + 2
    text = gen_random(nvars, rng.below(7) + 2, rng.below(5) + 1, seed)
    obj = rng.below(nvars)
    goal = ("min", obj) if rng.below(2) == 0 else ("max", obj)
    return text, goal


def with_goal(text: str, goal: tuple | None) -> str:
    """Replace the trailing ``solve satisfy;`` with a minimize/maximize item on var index."""
    if goal is None:
        return text
    kind, var = goal
    assert text.endswith("solve satisfy;\n")
    word = "minimize" if kind == "min" else "maximize"
    return text[: -len("solve satisfy;\n")] + f"solve {word} v{var};\n"


# --- SURVEY.md Appendix B (pinned by sha256 prefix in tests) ---------------------------------

def golomb(m: int, L: int) -> str:
    out = ["var x1 in 0..0;"] + [f"var x{i} in 1..{L};" for i in range(2, m + 1)]
    ds = []
    for i in range(1, m + 1):
        for j in range(i + 1, m + 1):
            out.append(f"var d{i}_{j} in 1..{L};")
            ds.append(f"d{i}_{j}")
    for i in range(1, m):
        out.append(f"constraint x{i} < x{i + 1};")
    for i in range(1, m + 1):
        for j in range(i + 1, m + 1):
            out.append(f"constraint x{j} - x{i} - d{i}_{j} = 0;")
    out.append("constraint alldifferent(" + ", ".join(ds) + ");")
    out.append(f"constraint d1_2 < d{m - 1}_{m};")
    out.append(f"solve minimize x{m};")
    return "\n".join(out) + "\n"


def magic(n: int) -> str:
    N = n * n
    S = n * (N + 1) // 2

    def v(r, c):
        return f"m{r}_{c}"

    out = [f"var {v(r, c)} in 1..{N};" for r in range(n) for c in range(n)]
    out.append("constraint alldifferent(" + ", ".join(v(r, c) for r in range(n) for c in range(n)) + ");")
    for r in range(n):
        out.append("constraint " + " + ".join(v(r, c) for c in range(n)) + f" = {S};")
    for c in range(n):
        out.append("constraint " + " + ".join(v(r, c) for r in range(n)) + f" = {S};")
    out.append("constraint " + " + ".join(v(i, i) for i in range(n)) + f" = {S};")
    out.append("constraint " + " + ".join(v(i, n - 1 - i) for i in range(n)) + f" = {S};")
    out.append("solve satisfy;")
    return "\n".join(out) + "\n"


def rcsp(n: int, k: int, ratio: float, seed: int) -> str:
    rnd = random.Random(seed)
    lines = [f"var v{i} in 1..{k};" for i in range(n)]
    m = int(ratio * n)
    seen = set()
    while len(seen) < m:
        a, b = rnd.randrange(n), rnd.randrange(n)
        if a == b or (min(a, b), max(a, b)) in seen:
            continue
        seen.add((min(a, b), max(a, b)))
        lines.append(f"constraint v{a} != v{b};")
    lines.append("solve satisfy;")
    return "\n".join(lines) + "\n"


# sha256 prefixes recorded by the survey
PINNED_SHA256 = {
    "nq8": "20154c5452817a9c",
    "nq14": "866c44e6c2c6e821",
    "golomb10": "6f6464c4fe8afab5",
    "magic5": "5266ef4693f5f5a9",
    "magic4": "7d7cc87603b1f0db",
    "rcsp_1000": "8c741c17cae3253d",
    "rcsp_10000": "521ce1345289ed19",
    "rcsp_100000": "9f513aacc32e0b2f",
}


def random_binary_csp(n: int, d: int, m: int, tightness: float, seed: int, connect: bool = False) -> str:
    """Random binary CSP, model B (BASELINE config 5; extension beyond the reference grammar):
    n variables over 1..d, m distinct random pairs, each a positive table that allows
    round((1 - tightness) * d^2) tuples drawn without replacement. The phase transition sits
    near tightness* = 1 - d^(-n/m) (expected number of solutions = 1)."""
    rnd = random.Random(seed)
    lines = [f"var v{i} in 1..{d};" for i in range(n)]
    allowed = max(1, round((1.0 - tightness) * d * d))
    tuples = [(a, b) for a in range(1, d + 1) for b in range(1, d + 1)]
    seen = set()
    order = list(range(n))
    if connect:
        rnd.shuffle(order)
    while len(seen) < m:
        if connect and len(seen) < n - 1:  # a random spanning path first, so the graph is connected
            a, b = order[len(seen)], order[len(seen) + 1]
        else:
            a, b = rnd.randrange(n), rnd.randrange(n)
        if a == b or (min(a, b), max(a, b)) in seen:
            continue
        seen.add((min(a, b), max(a, b)))
        tab = sorted(rnd.sample(tuples, allowed))
        lines.append(f"constraint table(v{a}, v{b} : " + ", ".join(f"{x} {y}" for x, y in tab) + ");")
    lines.append("solve satisfy;")
    return "\n".join(lines) + "\n"


def phase_transition_tightness(n: int, d: int, m: int) -> float:
    return 1.0 - d ** (-n / m)


def assignment(n: int, seed: int, forbid: int | None = None) -> str:
    """Weighted assignment: a permutation x of 1..n minimising sum c_i * x_i under random
    forbidden offsets x_i != x_j + k. An optimisation model whose LNS neighbourhoods (free
    variables re-permuted under the incumbent's bound) are real searches, unlike golomb's."""
    rnd = random.Random(seed)
    c = [rnd.randint(1, 9) for _ in range(n)]
    lo = sum(a * b for a, b in zip(sorted(c), range(n, 0, -1)))
    hi = sum(a * b for a, b in zip(sorted(c), range(1, n + 1)))
    hi = min(hi, lo + 1023)
    out = [f"var x{i} in 1..{n};" for i in range(1, n + 1)]
    out.append(f"var cost in {lo}..{hi};")
    out.append("constraint alldifferent(" + ", ".join(f"x{i}" for i in range(1, n + 1)) + ");")
    for _ in range(forbid if forbid is not None else 2 * n):
        i, j = rnd.sample(range(1, n + 1), 2)
        k = rnd.randint(1, 3)
        out.append(f"constraint x{i} != x{j} + {k};")
    out.append("constraint " + " + ".join(f"{c[i - 1]}*x{i}" for i in range(1, n + 1)) + " - cost = 0;")
    out.append("solve minimize cost;")
    return "\n".join(out) + "\n"


def named_instance(name: str) -> str:
    """The model text of a named benchmark instance (nqN, golombM, magicN, rcsp_N)."""
    if name.startswith("nq"):
        return gen_nqueens(int(name[2:]))
    if name.startswith("assign"):  # assign<n> or assign<n>_<seed>
        a, _, b = name[len("assign"):].partition("_")
        return assignment(int(a), int(b or 1))
    if name.startswith("golomb"):
        m = int(name[len("golomb"):])
        return golomb(m, m * m)
    if name.startswith("magic"):
        return magic(int(name[len("magic"):]))
    if name.startswith("rbcsp_"):  # rbcsp_<n>: config-5 random binary CSP, d=10, m=2n, near the transition
        n = int(name[len("rbcsp_"):])
        m = 2 * n
        t = phase_transition_tightness(n, 10, m) - 0.06
        return random_binary_csp(n, 10, m, t, 5)
    if name.startswith("rcsp_"):
        n = int(name[len("rcsp_"):])
        ratio = 1.0 if n >= 100000 else 2.0
        return rcsp(n, 3, ratio, 1)
    raise KeyError(name)
