"""One bench step at 2^20 for profiling (ncu launch lists / --set full captures).

Warm start comes from the committed d=2000 reference solution
(tests/golden/wc_solve_d2000.npz) so no C1 solve runs under the profiler.

    python tools/profile_step.py [--log2d 20] [--steps 1] [--phases local0,local1,exh0,exh1,obj]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1908_04489_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2d", type=int, default=20)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=0)
ap.add_argument("--phases", default="local0,local1,exh0,exh1,obj")
args = ap.parse_args()

sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
d = 1 << args.log2d
u0, u1 = bench.resample(sol["u0"], d), bench.resample(sol["u1"], d)
prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
dev = prob.device
cfg = P.SolverConfig(search_radius=19.5 * prob.grids[0].spacing)
U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
phases = args.phases.split(",")


def step(U):
    out = {}
    for name in phases:
        t = time.perf_counter()
        if name == "obj":
            prob.device_objective(U)
        else:
            kind, m = ("local", int(name[-1])) if name.startswith("local") else ("exhaustion", int(name[-1]))
            sweep = prob.device_local_update if kind == "local" else prob.device_exhaustion
            sweep(m, U, cfg)
        torch.cuda.synchronize()
        out[name] = (time.perf_counter() - t) * 1e3
    return out


for _ in range(args.warmup):
    step(U)
for _ in range(args.steps):
    print({k: round(v, 2) for k, v in step(U).items()}, flush=True)
prob.flush_errors()
