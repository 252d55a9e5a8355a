"""Randomised soak: device solve vs the CPU oracle (bitwise) on random
Witsenhausen grids / parameters / radii, a couple of rounds each.

    python tools/soak_solve.py [--trials 20]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1908_04489_b200 as P  # noqa: E402
from oracle import oracle as orc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--trials", type=int, default=20)
args = ap.parse_args()
orc.build()
rng = np.random.default_rng(7)
bad = 0
for t in range(args.trials):
    d0, d1 = int(rng.integers(3, 500)), int(rng.integers(3, 500))
    a, b = float(rng.uniform(-30, -8)), float(rng.uniform(8, 30))
    g0, g1 = (a, b, d0), (a - float(rng.uniform(0, 3)), b + float(rng.uniform(0, 3)), d1)
    k, s = float(rng.uniform(0.05, 1.0)), float(rng.choice([2.0, 3.0, 5.0, 7.0]))
    r = float(rng.choice([0.1, 0.5, 2.0]))
    mr = int(rng.integers(1, 3))
    prob = P.Witsenhausen(k=k, sigma=s, grids=[g0, g1])
    res = P.solve(prob, P.SolverConfig(max_rounds=mr, search_radius=r))
    p = orc.OracleWitsenhausen(k=k, sigma=s, grid0=g0, grid1=g1, f0=prob._f0, fw0=prob._fw0)
    u0, u1, J, rounds, term = orc.solve(p, orc.OracleConfig(max_rounds=mr, search_radius=r))
    ok = (res.final_objective == J and
          np.array_equal(np.asarray(res.controllers.values(0)).view(np.uint64), np.asarray(u0).view(np.uint64)) and
          np.array_equal(np.asarray(res.controllers.values(1)).view(np.uint64), np.asarray(u1).view(np.uint64)))
    if not ok:
        bad += 1
        print("MISMATCH", t, g0, g1, k, s, r, mr, res.final_objective, J, flush=True)
print("soak done, trials:", args.trials, "mismatches:", bad)
