"""Where config 4's time goes: per-instance kernel time (CUPTI), launches and
wall for sequential solves, then solve_many at several concurrencies.

    python tools/profile_c4.py [--instances 64] [--profile 8]
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
from bench_sweep import params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--instances", type=int, default=64)
ap.add_argument("--profile", type=int, default=8)
ap.add_argument("--conc", default="1,8,16,32,64")
args = ap.parse_args()
torch.cuda.set_device(0)
par = params(args.instances)
P.solve(P.Witsenhausen(), P.SolverConfig(max_rounds=1))
torch.cuda.synchronize()

# kernel time of a few sequential instances
probs = [P.Witsenhausen(k=k, sigma=s) for k, s in par[: args.profile]]
for p in probs:
    P.solve(p, P.SolverConfig(max_rounds=1))
torch.cuda.synchronize()
per_kernel = defaultdict(lambda: [0, 0.0])
l0 = _lib.launch_count()
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rounds = []
    for p in probs:
        rounds.append(P.solve(p, P.SolverConfig()).total_rounds)
    torch.cuda.synchronize()
wall = time.perf_counter() - t0
launches = _lib.launch_count() - l0
for e in prof.events():
    if e.device_type.name == "CUDA":
        per_kernel[e.name.split("(")[0]][0] += 1
        per_kernel[e.name.split("(")[0]][1] += e.device_time_total / 1e3
busy = sum(v[1] for v in per_kernel.values())
top = sorted(per_kernel.items(), key=lambda kv: -kv[1][1])[:12]
print(json.dumps({"sequential_instances": len(probs), "rounds": rounds, "wall_s_under_profiler": wall,
                  "kernel_busy_ms": busy, "abi_launches": launches,
                  "top": {k: {"n": v[0], "ms": round(v[1], 3), "us_per": round(1e3 * v[1] / v[0], 2)} for k, v in top}}),
      flush=True)

for c in [int(x) for x in args.conc.split(",")]:
    ps = [P.Witsenhausen(k=k, sigma=s) for k, s in par]
    for p in ps:
        p.device_context()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    t0 = time.perf_counter()
    P.solve_many(ps, P.SolverConfig(), concurrency=c)
    torch.cuda.synchronize()
    print(json.dumps({"concurrency": c, "wall_s": time.perf_counter() - t0, "launches": _lib.launch_count() - l0}),
          flush=True)
