"""Per-kernel device times (CUPTI via torch.profiler) for one block of each
kind at a given grid size, on the converged default-grid snapshot.

    python tools/kernel_times.py [--d 2000] [--iters 10]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1908_04489_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=2000)
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
prob = P.Witsenhausen(grids=[(-25.0, 25.0, args.d)] * 2)
u0, u1 = (sol["u0"], sol["u1"]) if args.d == 2000 else (bench.resample(sol["u0"], args.d),
                                                        bench.resample(sol["u1"], args.d))
U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
cfg = P.SolverConfig()
for kind in ("local", "exhaustion"):
    P.run_block(prob, U, cfg, 2, kind)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.run_block(prob, U, cfg, args.iters, kind)
        torch.cuda.synchronize()
    print(f"== {kind} block, {args.iters} iterations, d={args.d}")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
prob.flush_errors()
