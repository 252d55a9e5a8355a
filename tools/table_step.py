"""One bench step (four phases + objective) in the opt-in table arithmetic on
the bench snapshot, event-timed per phase (for ncu launch lists of the
expansion kernels).

    python tools/table_step.py [--log2d 20] [--reps 2]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1908_04489_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2d", type=int, default=20)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
d = 1 << args.log2d
sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
u0, u1 = bench.resample(sol["u0"], d), bench.resample(sol["u1"], d)
prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2, arithmetic="table")
cfg = P.SolverConfig(search_radius=19.5 * prob.grids[0].spacing)
U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
ms = {}
for rep in range(args.reps + 1):
    for name, kind, m in list(bench.PHASES) + [("objective", "objective", 0)]:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if kind == "objective":
            prob.device_objective(U)
        else:
            (prob.device_local_update if kind == "local" else prob.device_exhaustion)(m, U, cfg)
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ms[name] = ms.get(name, 0.0) + e0.elapsed_time(e1) / args.reps
print(json.dumps({"log2d": args.log2d, "arithmetic": "table", "ms": ms, "step_ms": sum(ms.values())}))
