"""How many block iterations of a full solve leave both controllers unchanged
(a fixed point: every later iteration of that block would repeat it bit for
bit)?  Runs the solve loop with per-iteration device sweeps and compares.

    python tools/fixed_point_census.py [--d 2000]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1908_04489_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=2000)
args = ap.parse_args()
prob = P.Witsenhausen(grids=[(-25.0, 25.0, args.d)] * 2)
cfg = P.SolverConfig()
U = prob.identity_controllers()
n = cfg.iters_per_round
n_local = n // 2
current = prob.device_objective(U)
stats = {"local": [0, 0], "exhaustion": [0, 0]}  # [iterations, fixed-point repeats]
for rnd in range(1, cfg.max_rounds + 1):
    Js = []
    for kind, iters in (("local", n_local), ("exhaustion", n - n_local)):
        sweep = prob.device_local_update if kind == "local" else prob.device_exhaustion
        stable = False
        for _ in range(iters):
            stats[kind][0] += 1
            if stable:
                stats[kind][1] += 1
            old = [U.device_values(m, prob.device).clone() for m in (0, 1)]
            for m in (0, 1):
                U = U.replace(m, P.SampledController(prob.grids[m], sweep(m, U, cfg).clone(), _trusted_device=True))
            stable = all(torch.equal(old[m].view(torch.int64), U.device_values(m, prob.device).view(torch.int64))
                         for m in (0, 1))
        Js.append(prob.device_objective(U))
    gl, ge = abs(current - Js[0]), abs(Js[0] - Js[1])
    current = Js[1]
    if gl + ge <= cfg.precision:
        break
    n_local, _ = P.adaptive_allocation(gl, ge, n)
print(json.dumps({"d": args.d, "rounds": rnd, "J": current, "iterations": stats}))
