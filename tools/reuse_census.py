"""Potential of result reuse in stage-0 exhaustion: within an exhaustion
block, iteration t's stage-0 result at point i equals iteration t-1's when
u1 is unchanged since then and no u0 value in i's window changed (the
candidate costs are a function of exactly those).  Counts the stage-0
candidates such reuse would skip.

    python tools/reuse_census.py [--d 2000]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1908_04489_b200 as P  # noqa: E402
from paper_1908_04489_b200.grids import node_window_bounds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=2000)
args = ap.parse_args()
prob = P.Witsenhausen(grids=[(-25.0, 25.0, args.d)] * 2)
cfg = P.SolverConfig()
g0 = prob.grids[0]
lo, hi = node_window_bounds(g0, cfg.radius_for(g0))
U = prob.identity_controllers()
n = cfg.iters_per_round
n_local = n // 2
current = prob.device_objective(U)
tot = skip = 0
for rnd in range(1, cfg.max_rounds + 1):
    Js = []
    for kind, iters in (("local", n_local), ("exhaustion", n - n_local)):
        sweep = prob.device_local_update if kind == "local" else prob.device_exhaustion
        prev = None
        for _ in range(iters):
            u0 = U.values(0).copy()
            u1 = U.values(1).copy()
            if kind == "exhaustion":
                # distinct candidates per point (adjacent dedup), as the kernel evaluates
                same = np.r_[False, u0[1:] == u0[:-1]]
                cs = np.cumsum(~same)
                ncand = cs[hi] - cs[lo] + 1
                tot += ncand.sum()
                if prev is not None and np.array_equal(prev[1].view(np.int64), u1.view(np.int64)):
                    changed = (prev[0].view(np.int64) != u0.view(np.int64)).astype(np.int64)
                    cc = np.r_[0, np.cumsum(changed)]
                    win_changed = cc[hi + 1] - cc[lo]
                    skip += ncand[win_changed == 0].sum()
                prev = (u0, u1)
            for m in (0, 1):
                U = U.replace(m, P.SampledController(prob.grids[m], sweep(m, U, cfg).clone(), _trusted_device=True))
        Js.append(prob.device_objective(U))
    gl, ge = abs(current - Js[0]), abs(Js[0] - Js[1])
    current = Js[1]
    if gl + ge <= cfg.precision:
        break
    n_local, _ = P.adaptive_allocation(gl, ge, n)
print(json.dumps({"d": args.d, "rounds": rnd, "J": current, "stage0_exh_candidates": int(tot),
                  "reusable": int(skip), "fraction": skip / max(tot, 1)}))
