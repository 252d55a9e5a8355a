"""Time-to-converge of the full adaptive solve on the GPU (BASELINE metric's
second half) at sizes beyond the default grid.

    python tools/converge.py --d 14000                 # the paper's grid size, identity start
    python tools/converge.py --d 1048576 --warm --radius-nodes 39 --max-rounds 4

--warm starts from the converged d=2000 solution (tests/golden) linearly
interpolated onto the grid (bench.py's snapshot); --radius-nodes sets
search_radius = (n/2) h.  Prints one JSON line with the per-round record.
"""
import argparse
import json
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
ap.add_argument("--d", type=int, default=14000)
ap.add_argument("--warm", action="store_true")
ap.add_argument("--radius-nodes", type=float, default=None)
ap.add_argument("--max-rounds", type=int, default=10000)
ap.add_argument("--arithmetic", default="reference", choices=["reference", "fma", "table"],
                help="Witsenhausen arithmetic (the non-reference ones are opt-in, tolerance-stated)")
args = ap.parse_args()

prob = P.Witsenhausen(grids=[(-25.0, 25.0, args.d)] * 2, arithmetic=args.arithmetic)
h = prob.grids[0].spacing
cfg = P.SolverConfig(max_rounds=args.max_rounds,
                     search_radius=None if args.radius_nodes is None else (args.radius_nodes / 2.0) * h)
initial = None
if args.warm:
    sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
    initial = P.ControllerSet(tuple(P.SampledController(g, bench.resample(sol[f"u{m}"], args.d))
                                    for m, g in enumerate(prob.grids)))
P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2).objective(
    P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2).identity_controllers())  # context warm-up
torch.cuda.synchronize()
t = time.perf_counter()
t_last = [t]


def progress(r):
    now = time.perf_counter()
    print(json.dumps({"round": r.round_index, "J": r.objective, "local_iters": r.local_iters,
                      "elapsed_s": now - t, "round_s": now - t_last[0]}), flush=True)
    t_last[0] = now


res = P.solve(prob, cfg, initial=initial, on_round=progress)
torch.cuda.synchronize()
wall = time.perf_counter() - t
print(json.dumps({"d": args.d, "warm": args.warm, "arithmetic": args.arithmetic, "search_radius": cfg.radius_for(prob.grids[0]),
                  "wall_s": wall, "rounds": res.total_rounds, "termination": res.termination,
                  "final_J": res.final_objective,
                  "per_round": [[r.round_index, r.objective, r.local_iters, r.exhaustion_iters, round(r.wall_ms, 1)]
                                for r in res.rounds],
                  "gpu": torch.cuda.get_device_name()}), flush=True)
