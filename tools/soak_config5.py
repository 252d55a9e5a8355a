"""Randomised soak for the config-5 problems: device solve vs the oracle's
solve_generic (bitwise) on random ZeroDelay / Inventory grids and parameters.

    python tools/soak_config5.py [--trials 40]
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
ap.add_argument("--trials", type=int, default=40)
args = ap.parse_args()
orc.build()
rng = np.random.default_rng(11)
bad = 0
for t in range(args.trials):
    mr = int(rng.integers(1, 3))
    if t % 2 == 0:
        g0 = (float(rng.uniform(-6, -3)), float(rng.uniform(3, 6)), int(rng.integers(5, 400)))
        g1 = (float(rng.uniform(-7, -4)), float(rng.uniform(4, 7)), int(rng.integers(5, 400)))
        pw = float(rng.uniform(0.3, 3.0))
        prob = P.ZeroDelay(power_weight=pw, grids=[g0, g1])
        p = orc.OracleZeroDelay(power_weight=pw, grid0=g0, grid1=g1, f0=prob._f0, fw0=prob._fw0)
    else:
        M = int(rng.integers(1, 5))
        quad = bool(rng.integers(0, 2))
        oc = float(rng.uniform(0.0, 0.5))
        grids = [(float(rng.uniform(-3.5, -2.5)), float(rng.uniform(2.5, 3.5)), int(rng.integers(5, 300))) for _ in range(M)]
        st = "quadratic" if quad else "piecewise_linear"
        prob = P.Inventory(stages=M, order_cost=oc, stage_cost=st, grids=grids)
        p = orc.OracleInventory(stages=M, order_cost=oc, stage_cost=st, grids=grids)
    res = P.solve(prob, P.SolverConfig(max_rounds=mr))
    Us, J, rounds, term = orc.solve_generic(p, orc.OracleConfig(max_rounds=mr))
    ok = res.final_objective == J and all(
        np.array_equal(np.asarray(res.controllers.values(m)).view(np.uint64), np.asarray(Us[m]).view(np.uint64))
        for m in range(prob.M))
    if not ok:
        bad += 1
        print("MISMATCH", t, prob.name, res.final_objective, J, flush=True)
print("soak done, trials:", args.trials, "mismatches:", bad)
