"""Config 4: 64 independent Witsenhausen instances (k in [0.05, 1], sigma in
{3, 5, 7}) at the default grid, solved to convergence; "replicas only"
across GPUs (torchrun: instance k on rank k % world).  Prints one JSON line.

    python tools/bench_sweep.py [--instances 64] [--concurrency 16] [--cpu-instances 2]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1908_04489_b200 as P  # noqa: E402


def params(n):
    return [(0.05 + 0.95 * i / (n - 1), (3.0, 5.0, 7.0)[i % 3]) for i in range(n)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", type=int, default=64)
    ap.add_argument("--concurrency", type=int, default=16)
    ap.add_argument("--cpu-instances", type=int, default=2, help="instances timed with the CPU oracle (0: skip)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    sh = P.from_process_group() if world > 1 else P.LOCAL
    par = params(args.instances)
    warm = P.Witsenhausen()
    P.solve(warm, P.SolverConfig(max_rounds=1))  # context + first launches
    # first launches of the batched kernels (lazy module loading)
    P.solve_many([P.Witsenhausen(k=k, sigma=s) for k, s in params(4)], P.SolverConfig(max_rounds=2))
    probs = [P.Witsenhausen(k=k, sigma=s) for k, s in par]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    res = P.solve_many(probs, P.SolverConfig(), concurrency=args.concurrency, sharding=sh)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    mine = [r for r in res if r is not None]
    tt = torch.tensor([wall], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    wall = float(tt.item())
    seq = None
    if rank == 0 and world == 1:
        t0 = time.perf_counter()
        for p in probs[:8]:
            P.solve(p, P.SolverConfig())
        torch.cuda.synchronize()
        seq = (time.perf_counter() - t0) / 8
    cpu = None
    if rank == 0 and args.cpu_instances > 0:
        from oracle import oracle as orc

        ts = []
        for k, s in par[: args.cpu_instances]:
            p = orc.OracleWitsenhausen(k=k, sigma=s)
            t = time.perf_counter()
            orc.solve(p)
            ts.append(time.perf_counter() - t)
        cpu = {"s_per_instance": float(np.mean(ts)), "instances_timed": len(ts), "cores": orc.num_threads(),
               "kind": "port", "total_s_extrapolated": float(np.mean(ts)) * args.instances}
    if rank == 0:
        print(json.dumps({
            "metric": "instance solves/s (config 4: 64 Witsenhausen instances, d=2000, to convergence)",
            "value": args.instances / wall, "unit": "solves/s", "n_gpus": world, "wall_s": wall,
            "engine": "batch (one kernel over (instance, point) per step)" if P.solver.BATCH_ENGINE else
            f"threads+streams (concurrency {args.concurrency})", "sequential_gpu_s_per_instance": seq,
            "rounds": [r.total_rounds for r in mine][:8], "J_first": [r.final_objective for r in mine][:4],
            "cpu_baseline": cpu, "scaling": "weak-free (replicas only)"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
