"""Benchmark: search nodes/s and time-to-all-solutions, N-Queens n=14 all solutions (BASELINE.json
configs[1]), on B200 through the C ABI, beside the reference CPU solver.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--instance nq14]

One step = one complete all-solutions search of the instance (4,864,749 nodes for nq14).
value   = nodes / device time of the search kernel (CUDA events on the launching stream),
          max over ranks for N > 1, whole-job aggregate.
e2e     = the same metric through cubics_solve_satisfy with host buffers: model upload, search,
          and the download of every solution (365,596 x 14 values) inside the timed region.
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "search nodes/sec and time-to-all-solutions at 1/2/4/8 B200 vs CPU ref"
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "fdref_driver")
MODELS = os.path.join(ROOT, "tests", "golden", "models")


# instance -> (mode, config.workload string, reference CLI flags, golden key). The headline is
# nq14 (BASELINE configs[1]); golomb10 and rcsp_1000 are the N>1 branch-and-bound and
# first-solution workloads of BASELINE configs[2] / configs[4].
WORKLOADS = {
    "nq14": ("all", "nq14 all solutions (N-Queens n=14, BASELINE configs[1])", ["--all"], "nq14|--all"),
    "golomb10": ("optimize", "Golomb ruler m=10, branch and bound to the optimum 55 (BASELINE configs[2])", [],
                 "golomb10"),
    "rcsp_1000": ("first", "random binary CSP n=1000, exact first solution (BASELINE configs[4], 1k point)",
                  ["--max", "1"], "rcsp_1000|--max 1"),
}


def workload(instance):
    return WORKLOADS.get(instance, ("all", f"{instance} all solutions", ["--all"], f"{instance}|--all"))


def workload_name(instance):
    """The config.workload string, identical on both arms (this one and --impl reference)."""
    return workload(instance)[1]


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": model}


def l2_probe(device):
    """Measured L2 read bandwidth: a 48 MiB buffer (resident in the 126 MB L2) summed 50 times,
    CUDA events (the roofline denominator for L2-resident traffic; MEASURED_PEAKS has HBM only)."""
    import torch

    x = torch.ones(12 << 20, dtype=torch.float32, device=f"cuda:{device}")
    for _ in range(5):
        x.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(device)
    e0.record()
    for _ in range(50):
        x.sum()
    e1.record()
    torch.cuda.synchronize(device)
    return x.numel() * 4 * 50 / (e0.elapsed_time(e1) / 1e3) / 1e9


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def ncu_traffic(instance):
    """roofline.traffic: dram__bytes_read.sum + dram__bytes_write.sum of the search kernel from one
    committed ncu capture of this workload (scripts/ncu_traffic.py: per launch; for the multi-launch
    B&B / first-solution steps scripts/ncu_step_counts.py: summed over one step)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as f:
            rec = json.load(f)[instance]
        return rec["dram_read_bytes"] + rec["dram_write_bytes"], rec["report"]
    except Exception:  # noqa: BLE001
        return None, None


def ncu_counts(instance):
    """Per-launch instruction / shared-memory counts of the committed ncu capture (with its nodes)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as f:
            return json.load(f)[instance]
    except Exception:  # noqa: BLE001
        return None


def algorithmic_bytes(model, stats):
    """A = rounds*(4*S + 8*V) + nodes*(4*V), W_v = ceil(width_v/32) u32 words."""
    wv = [(w + 31) // 32 for w in model.widths]
    V = sum(wv)
    S_ = 0
    for c in range(model.n_cons):
        scope = set(model.term_var[model.con_start[c]:model.con_start[c + 1]])
        S_ += sum(wv[v] for v in scope)
    return stats.rounds * (4 * S_ + 8 * V) + stats.nodes * (4 * V), S_, V


class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu):
        self.gpu, self.samples, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(int(float(s[0])) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(int(float(s[1])) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def run_reference(path, flags, threads=1, timeout=3600):
    import resource

    def lim():
        resource.setrlimit(resource.RLIMIT_STACK, (resource.RLIM_INFINITY, resource.RLIM_INFINITY))

    r = subprocess.run([REF_DRIVER, "solve", path, "--threads", str(threads)] + flags, capture_output=True,
                       text=True, timeout=timeout, preexec_fn=lim)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return json.loads(r.stdout)


def cpu_sample(instance, node_limit, threads):
    flags = workload(instance)[2] + (["--node-limit", str(node_limit)] if node_limit else [])
    out = run_reference(os.path.join(MODELS, instance + ".fd"), flags, threads)
    return out["nodes"] / (out["time_ms"] / 1e3), out


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def impl_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    if not os.path.exists(REF_DRIVER):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/fdref_driver not built"}))
        return 0
    nproc = os.cpu_count() or 1
    # bounded sample of the same workload: the first N nodes of the reference's DFS for it
    # (branch and bound / first solution: a few seconds of the reference's much slower nodes)
    limit = args.ref_node_limit if workload(args.instance)[0] == "all" else min(args.ref_node_limit, 10000)
    # the reference's only parallel knob (OpenMP propagation) slows this workload down
    # (SURVEY.md 2.3); pick whichever of 1 / nproc threads is faster on a short probe
    probe = {t: cpu_sample(args.instance, 20000 if limit > 20000 else 2000, t)[0] for t in sorted({1, nproc})}
    threads = max(probe, key=probe.get)
    vals = []
    for i in range(args.warmup + args.steps):
        v, out = cpu_sample(args.instance, limit, threads)
        if i >= args.warmup:
            vals.append(v)
    value = sum(vals) / len(vals)
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "nodes/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": limit / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": {"workload": workload_name(args.instance)},
        "run": {"sample": f"first {limit} DFS nodes"},
        "cpu_baseline": {"value": value, "unit": "nodes/s", "cores": threads, "kind": "reference",
                         "sample": f"first {limit} nodes of the reference's DFS for: {workload_name(args.instance)}, "
                                   f"threads={threads}",
                         "probe_nodes_per_s": probe, "host": host_info()},
        "e2e": {"value": value, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


GOLDEN = os.path.join(ROOT, "tests", "golden", "goldens.json")


def ref_same_run(key, g, budget_ms=4000):
    """The unmodified reference (oracle/_ref/fdref_driver, 1 thread) on THIS host for one config:
    the full search when the golden run took <= 2 x budget on the build box, else the first N nodes
    of the same DFS (N sized for ~budget) and the full time extrapolated from the golden node count."""
    inst, _, fl = key.partition("|")
    path = os.path.join(MODELS, inst + ".fd")
    if not g or not g.get("time_ms") or not os.path.exists(REF_DRIVER) or not os.path.exists(path):
        return None
    full = g["time_ms"] <= 2 * budget_ms
    lim = None if full else max(1000, int(g["nodes"] * budget_ms / g["time_ms"]))
    out = run_reference(path, fl.split() + (["--node-limit", str(lim)] if lim else []), 1)
    rate = out["nodes"] / (out["time_ms"] / 1e3)
    rec = {"ms": out["time_ms"] if full else None, "nodes_per_s": rate, "threads": 1, "same_host": True,
           "sample": "full search" if full else f"first {lim} nodes of the same DFS"}
    if not full:
        rec["est_full_ms"] = g["nodes"] / rate * 1e3
    return rec


def run_extras(S, A, device, cpu=True):
    """The other BASELINE.json configs, one run each (device time; stats vs the reference goldens),
    each beside the unmodified reference run on this same host (ref_same_run)."""
    gold = json.load(open(GOLDEN))
    out = {}
    cases = [
        ("golomb10", "golomb10", A.ENGINE_AUTO, {},
         "B&B, exact parallel engine (AUTO: the reference's node order, stats and incumbents)"),
        ("golomb10_shared_bound", "golomb10", A.ENGINE_PARALLEL, {},
         "B&B to optimum, parallel engine with a shared bound (node count schedule-dependent)"),
        ("golomb10_parity", "golomb10", A.ENGINE_PARITY, {}, "B&B, parity engine (reference node order)"),
        ("magic5_first", "magic5|--max 1", A.ENGINE_AUTO, {"max_solutions": 1},
         "exact first solution (AUTO: parallel engine, reference stats)"),
        ("magic4_all", "magic4|--all", A.ENGINE_PARALLEL, {}, "all solutions, parallel engine"),
        ("rcsp_1000_first", "rcsp_1000|--max 1", A.ENGINE_AUTO, {"max_solutions": 1},
         "exact first solution (AUTO: parallel engine, reference stats)"),
        ("rcsp_100000_limit200", "rcsp_100000|--max 1 --node-limit 200", A.ENGINE_AUTO,
         {"max_solutions": 1, "node_limit": 200}, "node-limited, reference node order (grid-wide context)"),
        # BASELINE config 5 as stated: random binary CSP with extensional tables near the phase
        # transition (d=10, m=2n, tightness = transition - 0.06). No reference counterpart: stats
        # are checked against the oracle port in tests/test_gpu_parity.py.
        ("config5_rbcsp_1000_limit2000", "rbcsp_1000", A.ENGINE_AUTO, {"max_solutions": 1, "node_limit": 2000},
         "tables, 1k vars / 2k tables, node-limited"),
        ("config5_rbcsp_10000_limit200", "rbcsp_10000", A.ENGINE_AUTO, {"max_solutions": 1, "node_limit": 200},
         "tables, 10k vars / 20k tables, node-limited (grid-wide context)"),
        ("config5_rbcsp_100000_limit200", "rbcsp_100000", A.ENGINE_AUTO, {"max_solutions": 1, "node_limit": 200},
         "tables, 100k vars / 200k tables, node-limited (grid-wide context)"),
    ]
    for name, key, engine, kw, what in cases:
        inst = key.split("|")[0]
        g = gold.get(key)
        path = os.path.join(MODELS, inst + ".fd")
        from paper_1909_09213_b200 import models as MD
        m = S.parse_model(open(path).read() if os.path.exists(path) else MD.named_instance(inst))
        cfg = S.SearchConfig(engine=engine, device=device, count_only=True, **kw)
        try:
            for attempt in range(2):  # a second, warm run when the first is short (kernel loading)
                if m.goal != 0:
                    r = S.solve_optimize(m, cfg)
                    extra = {"objective": r.best.objective if r.best else None}
                else:
                    r = S.solve_satisfy(m, cfg)
                    extra = {}
                if r.device_ms > 2000:
                    break
            st = r.stats.as_tuple()
            exp = (g["nodes"], g["failures"], g["rounds"], g["solutions"]) if g else None
            rec = {"what": what, "device_ms": round(r.device_ms, 3), "nodes": st[0], "stats": list(st),
                   "engine": {1: "parity", 2: "parallel", 3: "grid"}.get(r.engine, r.engine),
                   "nodes_per_s": st[0] / (r.device_ms / 1e3) if r.device_ms else None,
                   "stats_equal_reference": (st == exp) if exp else None,
                   "reference_cpu": ref_same_run(key, g) if cpu else None,
                   "reference_cpu_ms_build_box": g.get("time_ms") if g else None, **extra}
            if name.startswith("config5_"):  # extensional constraints: no reference counterpart
                rec["parity_note"] = ("unpinned: the reference has no table constraint; the table propagators are "
                                      "checked against the oracle's table extension and brute force in tests/")
            ref = rec["reference_cpu"]
            if ref and r.device_ms:
                rec["speedup_vs_reference_cpu"] = (ref["ms"] or ref["est_full_ms"]) / r.device_ms
            if m.goal != 0 and g:
                rec["objective_equal_reference"] = extra["objective"] == g.get("objective")
            out[name] = rec
        except Exception as e:  # noqa: BLE001 - reported, never hidden
            out[name] = {"what": what, "error": repr(e)}
    # LNS with every neighbourhood of an iteration in ONE batched launch
    # (cubics_solve_optimize_batch); reference-identical trajectory (tests/test_gpu_lns.py)
    try:
        from paper_1909_09213_b200 import models as MD
        m = S.parse_model(MD.named_instance("assign30"))
        lc = S.LnsConfig(destroy_rate=0.35, iterations=5, neighborhoods=592, seed=1, per_iteration_node_limit=1000)
        r = S.lns_optimize(m, lc)
        out["lns_assign30"] = {"what": "LNS 5 iterations x 592 neighbourhoods, node limit 1000, one launch per iteration",
                               "device_ms": round(r.device_ms, 3), "nodes": r.stats.nodes,
                               "nodes_per_s": r.stats.nodes / (r.device_ms / 1e3) if r.device_ms else None,
                               "objective": r.best.objective if r.best else None, "trajectory": r.trajectory}
    except Exception as e:  # noqa: BLE001
        out["lns_assign30"] = {"error": repr(e)}
    return out


def impl_ours(args):
    from paper_1909_09213_b200 import _abi as A
    from paper_1909_09213_b200 import solver as S

    rank, world, local = dist_env()
    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        # one process per GPU over NCCL; CUBICS_BENCH_BACKEND=gloo with fewer GPUs than ranks is
        # a functional check of this code path only (ranks then share a device)
        backend = os.environ.get("CUBICS_BENCH_BACKEND", "nccl")
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        dist.init_process_group(backend)
    device = local if world > 1 else 0
    coll_dev = f"cuda:{local}" if (dist is None or dist.get_backend() == "nccl") else "cpu"

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(device)

    def max_over_ranks(vals):
        if dist is None:
            return list(vals)
        t = torch.tensor(list(vals), dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()
    text = open(os.path.join(MODELS, args.instance + ".fd")).read()
    model = S.parse_model(text)
    mode, _, _, gkey = workload(args.instance)
    gold = json.load(open(GOLDEN)).get(gkey)
    cfg = S.SearchConfig(engine=A.ENGINE_PARALLEL, device=device, count_only=True, contexts=args.contexts,
                         block_threads=args.block, max_solutions=1 if mode == "first" else A.UINT64_MAX)

    # N > 1: frontier subtrees are claimed dynamically through one counter in rank 0's HBM that
    # every rank maps over NVLink (CUDA IPC); CUBICS_BENCH_STATIC=1 selects the static t % N split
    queue = None
    if world > 1 and os.environ.get("CUBICS_BENCH_STATIC", "0") != "1":
        from paper_1909_09213_b200 import distributed as D

        try:  # collective; every rank gets the same outcome
            queue = D.shared_task_queue(rank, world, device)
        except S.EngineUnavailable as e:
            if rank == 0:
                print(f"shared task queue unavailable, static split: {e}", file=sys.stderr)

    def one_step(count_only=True):
        c = S.SearchConfig(**{**cfg.__dict__, "count_only": count_only})
        if world > 1:
            if queue is not None:
                if rank == 0:
                    queue.reset()
                dist.barrier()
            if mode == "optimize":  # shared incumbent through the queue state
                return S.solve_optimize_shard(model, c, rank, world, queue=queue)
            if mode == "first":  # DFS-order claims, shared best-key prefix
                part = S.solve_first_shard(model, c, rank, world, queue=queue)
                part.close()
                return part.result
            return S.solve_shard(model, c, rank, world, queue=queue)
        if mode == "optimize":  # AUTO: the exact parallel B&B (reference stats)
            return S.solve_optimize(model, S.SearchConfig(**{**c.__dict__, "engine": A.ENGINE_AUTO}))
        return S.solve_satisfy(model, c, (lambda s: True) if not count_only else None)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")  # > 126 MB L2

    def flush_l2():
        flush.zero_()
        torch.cuda.synchronize(device)

    for _ in range(args.warmup):
        one_step()
    stats0 = None
    dev_ms = []
    with ClockSampler(device) as clk:
        for _ in range(args.steps):
            flush_l2()
            barrier()  # every rank starts the step together; device time is CUDA events
            r = one_step()
            dev_ms.append(r.device_ms)
            stats0 = r.stats
    barrier()
    dev_ms = max_over_ranks(dev_ms)  # per step, the slowest rank
    tot = S.SearchStats(*stats0.as_tuple())
    if dist is not None:  # whole-job stats: one all-reduce (sum) of the shards' partial stats
        t = torch.tensor(list(stats0.as_tuple()), dtype=torch.int64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        tot = S.SearchStats(*[int(x) for x in t.tolist()])
    e2e_ms, h2d, d2h, e2e_launches = [], 0, 0, 0
    exact = None  # the reference's stats / objective reproduced by the public API call
    if world == 1:
        # e2e: through the public C ABI with host buffers: model upload, search, results back
        full = S.SearchConfig(**{**cfg.__dict__, "count_only": False})
        for i in range(args.warmup + args.steps):  # the same W warm-up calls on this path first
            if i == args.warmup:
                e2e_ms = []
            flush_l2()
            t0 = time.perf_counter()
            if mode == "all":  # every solution, DFS-ordered on the device, into a host int64 array
                arr, r2 = S.enumerate_array(model, full)
                assert arr.shape[0] == r2.stats.solutions
                exact = r2.stats.as_tuple()
            elif mode == "optimize":  # the optimum's values (exact parallel B&B)
                r2 = S.solve_optimize(model, S.SearchConfig(**{**full.__dict__, "engine": A.ENGINE_AUTO}))
                exact = (r2.stats.as_tuple(), r2.best.objective if r2.best else None)
            else:  # the DFS-first solution through the solution callback
                got = []
                r2 = S.solve_satisfy(model, full, lambda s: got.append(s.values) or True)
                exact = r2.stats.as_tuple()
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
            h2d, d2h, e2e_launches = r2.h2d_bytes, r2.d2h_bytes, r2.kernel_launches
        e2e_api = {"all": "cubics_enumerate (all solutions in DFS order into a host int64 array)",
                   "optimize": "cubics_solve_optimize (branch and bound; optimum values to the host)",
                   "first": "cubics_solve_satisfy with a callback, max_solutions 1 (exact first solution)"}[mode]
    else:
        # e2e at N GPUs: the public multi-GPU API (distributed.solve_distributed -> cubics_solve_shard
        # + one all-reduce of the stats), wall time per rank, max over ranks
        from paper_1909_09213_b200 import distributed as D

        for _ in range(args.steps):
            flush_l2()
            barrier()
            t0 = time.perf_counter()
            st, res, _ = D.solve_distributed(model, cfg, rank, world, collect=False, device=coll_dev, queue=queue)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
            if mode == "all":
                assert tuple(st) == tot.as_tuple()
                exact = tuple(st)
            elif mode == "optimize":
                exact = res.objective if res else None
            else:
                exact = tuple(st)
        e2e_ms = max_over_ranks(e2e_ms)
        h2d, d2h = r.h2d_bytes, r.d2h_bytes
        e2e_launches = r.kernel_launches
        e2e_api = ("distributed.solve_distributed (%s per rank + all-reduce of the stats)"
                   % {"all": "cubics_solve_shard" + ("_shared" if queue is not None else ""),
                      "optimize": "cubics_solve_optimize_shard, shared incumbent",
                      "first": "cubics_solve_first_shard + min-key all-gather"}[mode])
    extras = run_extras(S, A, device, cpu=not args.no_cpu) if (rank == 0 and not args.no_extras) else None
    l2_gbs = l2_probe(device) if rank == 0 else None
    if rank != 0:
        dist.destroy_process_group()
        return 0
    mean_ms = sum(dev_ms) / len(dev_ms)
    # all solutions: every node is visited exactly once, nodes = the reference's. Branch and bound
    # and first solution: the GPUs search a different (speculative / schedule-dependent) node set,
    # so value = the reference's node count for the same answer / time to the answer
    # ("reference-equivalent nodes/s", a time-to-answer ratio against the CPU arm's nodes/s)
    nodes = tot.nodes if mode == "all" or not gold else gold["nodes"]
    value = nodes / (mean_ms / 1e3)
    if mode == "all":
        parity_ok = gold is not None and exact == (gold["nodes"], gold["failures"], gold["rounds"], gold["solutions"])
    elif mode == "optimize":  # N=1: stats and optimum; N>1 (shared bound): the optimum
        want = ((gold["nodes"], gold["failures"], gold["rounds"], gold["solutions"]), gold.get("objective")) if gold else None
        parity_ok = gold is not None and (exact == want if world == 1 else exact == gold.get("objective"))
    else:
        parity_ok = gold is not None and exact == (gold["nodes"], gold["failures"], gold["rounds"], gold["solutions"])
    parity = {gkey: parity_ok}
    for name, rec in (extras or {}).items():
        if rec.get("stats_equal_reference") is False and rec.get("objective_equal_reference") is not None:
            parity[name + "_objective"] = rec["objective_equal_reference"]  # schedule-dependent node count
        elif rec.get("stats_equal_reference") is not None:
            parity[name] = rec["stats_equal_reference"]
    A_bytes, S_, V = algorithmic_bytes(model, tot)
    peak, peak_kind = load_peaks()
    achieved = A_bytes / (mean_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(args.instance)
    clocks = clk.summary()
    sm_hz = (clocks.get("sm_mhz") or 1965) * 1e6
    # the rooflines that bind this latency-bound search (counts per node from the committed ncu
    # capture of this workload, scaled by this run's nodes and time)
    issue = smem = None
    cap = ncu_counts(args.instance)
    if cap and cap.get("inst_executed") and cap.get("nodes"):
        # per node of the value's basis (the reference's nodes for B&B / first solution, where the
        # capture sums every launch of one step: speculative work included)
        per_node = cap["inst_executed"] / cap["nodes"]
        ach = per_node * nodes / (mean_ms / 1e3)
        peak_i = 148 * 4 * sm_hz  # 4 schedulers x 1 warp-instruction / cycle per SM
        issue = {"achieved": ach / 1e9, "peak": peak_i / 1e9, "unit": "G warp-inst/s", "frac": ach / peak_i,
                 "warp_inst_per_node": per_node, "source": cap["report"]}
        if cap.get("smem_wavefronts"):
            wn = cap["smem_wavefronts"] / cap["nodes"]
            ach_s = wn * nodes / (mean_ms / 1e3)
            peak_s = 148 * sm_hz  # one shared-memory wavefront per cycle per SM
            smem = {"achieved": ach_s / 1e9, "peak": peak_s / 1e9, "unit": "G wavefronts/s", "frac": ach_s / peak_s,
                    "wavefronts_per_node": wn}
    # CPU baseline: the unmodified reference on this host, bounded sample
    cpu = None
    if os.path.exists(REF_DRIVER) and not args.no_cpu and world == 1:
        lim = args.cpu_node_limit if mode == "all" else min(args.cpu_node_limit, 10000)
        v, out = cpu_sample(args.instance, lim, 1)
        cpu = {"value": v, "unit": "nodes/s", "cores": 1, "kind": "reference",
               "sample": f"first {lim} nodes of the reference's DFS for: {workload_name(args.instance)} "
                         f"(oracle/_ref/fdref_driver, thread_count=1, {out['time_ms']:.0f} ms)",
               "host": host_info()}
        if args.cpu_full:  # the whole search, measured (not extrapolated): minutes for nq14
            full = run_reference(os.path.join(MODELS, args.instance + ".fd"), workload(args.instance)[2], 1)
            cpu["full_search_ms"] = full["time_ms"]
            cpu["full_search_nodes"] = full["nodes"]
    e2e_mean = sum(e2e_ms) / len(e2e_ms)  # same statistic as value (mean over the timed steps)
    line = {
        "metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": workload_name(args.instance)},
        "run": {"engine": "parallel", "contexts": r.contexts, "l2": "flushed (256 MiB write) before every timed step",
                   "devices_visible": torch.cuda.device_count(),
                   "ranks_share_devices": world > torch.cuda.device_count(),
                   "balancing": ("in-GPU work-sharing ring" if world == 1 else
                                 "shared subtree queue (claim counter in rank 0 HBM, CUDA IPC over NVLink) + "
                                 "in-GPU work-sharing ring" if queue is not None else
                                 "static t % N frontier split + in-GPU work-sharing ring"),
                   "stats": {"nodes": tot.nodes, "failures": tot.failures, "rounds": tot.rounds,
                             "solutions": tot.solutions},
                   "value_nodes": "nodes visited (exact)" if mode == "all" else
                                  f"the reference's {nodes} nodes for this answer / device time to the answer "
                                  f"(searched: {tot.nodes})"},
        "time_to_all_solutions_ms" if mode == "all" else
        ("time_to_optimum_ms" if mode == "optimize" else "time_to_first_solution_ms"): mean_ms,
        # rounds x constraints / device time (every constraint counted every round,
        # as the reference evaluates them; the engine itself skips untriggered ones)
        "propagator_evals_per_s": tot.rounds * model.n_cons / (mean_ms / 1e3),
        "e2e": {"value": nodes / (e2e_mean / 1e3), "unit": "nodes/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_mean, "steps": len(e2e_ms), "api": e2e_api,
                "gpu_launches": e2e_launches},
        "gpu_launches": r.kernel_launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind,
                     "algorithmic_bytes": A_bytes, "S_words": S_, "V_words": V,
                     "l2": {"achieved": achieved, "peak": l2_gbs, "unit": "GB/s",
                            "frac": achieved / l2_gbs if l2_gbs else None,
                            "peak_kind": "measured in this run (l2_probe: 48 MiB L2-resident read)"},
                     "issue": issue, "smem": smem,
                     "note": "the algorithmic bytes never reach DRAM (traffic = ncu dram bytes per launch); "
                             "the binding limit is instruction issue (roofline.issue)"},
        "parity": parity,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "other_configs": extras,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instance", default="nq14")
    ap.add_argument("--contexts", type=int, default=0)
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--cpu-node-limit", type=int, default=400000)
    ap.add_argument("--ref-node-limit", type=int, default=200000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--cpu-full", action="store_true", help="also time the reference's complete search")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_spawn(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return impl_reference(args)
    return impl_ours(args)


def self_spawn(args):
    """`python bench.py --gpus N` without a launcher: re-run this script as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1). With fewer visible GPUs
    than ranks the ranks share devices over gloo (a functional check of the N-rank path; the
    line then says so in config.devices_visible)."""
    import socket

    import torch

    ngpu = torch.cuda.device_count()
    env = dict(os.environ)
    if ngpu < args.gpus:
        env.setdefault("CUBICS_BENCH_BACKEND", "gloo")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


if __name__ == "__main__":
    sys.exit(main())
