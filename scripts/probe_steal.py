"""Two processes on one GPU sharing a task queue (CUDA IPC): cross-GPU stealing diagnostics.
usage: python scripts/probe_steal.py [ctx0] [ctx1] [instance]   (WORLD=k: k processes, contexts cycle)"""
import os
import socket
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))


def worker(rank, world, port, ctxs, inst):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import time

    import torch.distributed as dist

    import golden_cases as G
    from paper_1909_09213_b200 import distributed as D
    from paper_1909_09213_b200 import solver as S

    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = S.parse_model(G.model_text(inst))
    q = D.shared_task_queue(rank, world, device=0)
    bad = 0
    import torch
    iters = int(os.environ.get("ITERS", "3"))
    for it in range(iters):
        if rank == 0:
            q.reset()
        dist.barrier()
        t0 = time.perf_counter()
        r = S.solve_shard(m, S.SearchConfig(device=0, contexts=ctxs[rank], count_only=True), rank, world, queue=q)
        dist.barrier()  # nobody resets the queue while another rank still searches
        t = torch.tensor(list(r.stats.as_tuple()) + [r.remote_in, r.remote_out], dtype=torch.int64)
        dist.all_reduce(t)
        ok = tuple(t.tolist()[:4]) == (4864749, 2066779, 11003828, 365596) if inst == "nq14" else True
        bad += 0 if ok else 1
        if rank == 0 and (not ok or it < 3):
            print(f"it {it}: {t.tolist()} ok={ok} dev {r.device_ms:.1f} ms", flush=True)
    if rank == 0:
        print(f"bad {bad} of {iters}", flush=True)
    dist.barrier()
    q.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    ctxs = [int(sys.argv[1]) if len(sys.argv) > 1 else 32, int(sys.argv[2]) if len(sys.argv) > 2 else 256]
    inst = sys.argv[3] if len(sys.argv) > 3 else "nq14"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = int(os.environ.get("WORLD", "2"))
    ctxs = [ctxs[i % 2] for i in range(world)]
    mp.spawn(worker, args=(world, port, ctxs, inst), nprocs=world)
