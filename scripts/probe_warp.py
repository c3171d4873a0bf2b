"""A/B probe: warp-context kernel vs the block kernel on the small golden instances.

    python scripts/probe_warp.py [reps]

Runs each case with the default engine choice (warp contexts when eligible) and with
CUBICS_NO_WARP=1 semantics emulated by a subprocess, checks the stats against the reference
goldens and prints device times. Run on the GPU box."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CASES = [("nq8|--all", "parallel"), ("nq10|--all", "parallel"), ("nq12|--all", "parallel"),
         ("nq14|--all", "parallel"), ("magic4|--all", "parallel"), ("magic3|--all", "parallel"),
         ("nq14|--max 1", "parallel"), ("magic5|--max 1", "parallel"), ("magic5|--max 1", "parity"),
         ("nq12|--all", "parity"), ("magic4|--max 1", "parity"), ("nq40|--max 1", "parity")]


def child(reps):
    import golden_cases as G
    from paper_1909_09213_b200 import _abi as A
    from paper_1909_09213_b200 import solver as S

    S.lib().cubics_warmup(0)
    out = []
    for key, eng in CASES:
        inst, flags = G.split_key(key)
        m = S.parse_model(G.model_text(inst))
        cfg = G.cfg_from_flags(flags)
        cfg.engine = {"parallel": A.ENGINE_PARALLEL, "parity": A.ENGINE_PARITY}[eng]
        cfg.device = 0
        cfg.count_only = True
        if cfg.max_solutions == 1:
            cfg.count_only = False
        ts = []
        st = None
        for _ in range(reps):
            r = S.solve_satisfy(m, cfg, (lambda s: True) if not cfg.count_only else None)
            ts.append(r.device_ms)
            st = r.stats.as_tuple()
        g = G.goldens().get(key)
        ok = g is not None and st == G.expected_tuple(g)
        out.append({"case": key, "engine": eng, "ok": ok, "stats": st, "ms_min": min(ts),
                    "ms_mean": sum(ts) / len(ts), "ctx": r.contexts})
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "child":
        child(int(sys.argv[1]))
        sys.exit(0)
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    res = {}
    variants = [("warp", {}), ("block", {"CUBICS_NO_WARP": "1"})]
    # PROBE_VARIANTS="label:K=V,K=V;label2:..." replaces the default pair (first one is the baseline)
    if os.environ.get("PROBE_VARIANTS"):
        variants = []
        for item in os.environ["PROBE_VARIANTS"].split(";"):
            label, _, kvs = item.partition(":")
            variants.append((label, dict(kv.split("=", 1) for kv in kvs.split(",") if kv)))
    only = os.environ.get("PROBE_CASES")
    if only:
        keep = only.split(";")
        CASES[:] = [c for c in CASES if c[0] in keep]
    for label, env in variants:
        e = dict(os.environ, **env)
        if "CUBICS_LIB" in e and not os.path.isabs(e["CUBICS_LIB"]):
            e["CUBICS_LIB"] = os.path.join(ROOT, e["CUBICS_LIB"])
        p = subprocess.run([sys.executable, __file__, str(reps), "child"], env=e, capture_output=True, text=True)
        if p.returncode:
            print(label, "FAILED", p.stderr[-3000:])
            continue
        res[label] = json.loads(p.stdout.strip().splitlines()[-1])
    labels = [v[0] for v in variants if v[0] in res]
    for i, case in enumerate(res[labels[0]] if labels else []):
        line = f"{case['case']:<18} {case['engine']:<8}"
        for lb in labels:
            c = res[lb][i]
            line += f" | {lb} {'ok' if c['ok'] else 'BAD'} {c['ms_min']:8.3f} ms ctx {c['ctx']}"
        print(line)
    if not labels:
        print(json.dumps(res))
