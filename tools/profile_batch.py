"""Kernel-time breakdown (CUPTI via torch.profiler) of the batched config-4 solve.

    python tools/profile_batch.py [--instances 64] [--d 2000]
"""
import argparse
import json
import sys
import time
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_1908_04489_b200 as P  # noqa: E402
from paper_1908_04489_b200 import _lib  # noqa: E402
from paper_1908_04489_b200.batch import solve_batch  # noqa: E402
from bench_sweep import params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--instances", type=int, default=64)
ap.add_argument("--d", type=int, default=2000)
args = ap.parse_args()
torch.cuda.set_device(0)
mk = lambda: [P.Witsenhausen(k=k, sigma=s, grids=[(-25.0, 25.0, args.d)] * 2) for k, s in params(args.instances)]
solve_batch(mk()[:4], P.SolverConfig(max_rounds=2))
torch.cuda.synchronize()
walls = []
for rep in range(3):
    probs = mk()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    l0 = _lib.launch_count()
    res = solve_batch(probs, P.SolverConfig())
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
    from paper_1908_04489_b200.batch import LAST_STATS
    print(json.dumps({"rep": rep, "wall": walls[-1], **LAST_STATS}), flush=True)
    launches = _lib.launch_count() - l0
wall = min(walls)
probs = mk()
for p in probs:
    p.device_context()
torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    solve_batch(probs, P.SolverConfig())
    torch.cuda.synchronize()
for e in prof.events():
    if e.device_type.name == "CUDA":
        name = e.name.split("(")[0].replace("void ", "").split("<")[0]
        name = name.split("::")[-1] or e.name[:60]
        agg[name][0] += 1
        agg[name][1] += e.device_time_total / 1e3
busy = sum(v[1] for v in agg.values())
top = sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]
print(json.dumps({"instances": args.instances, "d": args.d, "wall_s": wall, "walls": walls, "abi_launches": launches,
                  "rounds_max": max(r.total_rounds for r in res), "rounds_sum": sum(r.total_rounds for r in res),
                  "kernel_busy_ms_sum": busy,
                  "top": {k: {"n": v[0], "ms": round(v[1], 2), "us_per": round(1e3 * v[1] / v[0], 1)} for k, v in top}},
                 indent=1))
