"""Randomised soak of the throughput-mode kernels (the headline path): random
Witsenhausen grids of 6k-40k points, parameters and controllers, windows wide
enough that the stage-0 walks run k_*<0> with the no-op tail exit and the
stage-1 moments run the persistent k_moments; every phase over the whole grid
on the device, checked bitwise against the oracle on sampled points (grid ends
included).

    python tools/soak_throughput.py [--trials 30]
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
ap.add_argument("--trials", type=int, default=30)
ap.add_argument("--points", type=int, default=48)
args = ap.parse_args()
orc.build()
rng = np.random.default_rng(11)
bad = 0
for t in range(args.trials):
    d0, d1 = int(rng.integers(6000, 40000)), int(rng.integers(6000, 40000))
    a, b = float(rng.uniform(-30, -10)), float(rng.uniform(10, 30))
    g0, g1 = (a, b, d0), (a - float(rng.uniform(0, 3)), b + float(rng.uniform(0, 3)), d1)
    k, s = float(rng.uniform(0.05, 1.0)), float(rng.choice([2.0, 3.0, 5.0, 7.0]))
    prob = P.Witsenhausen(k=k, sigma=s, grids=[g0, g1])
    y0, y1 = prob.grids[0].points, prob.grids[1].points
    kind = rng.integers(0, 3)
    if kind == 0:    # smooth
        u0 = -0.8 * y0 + rng.normal(0, 0.05, d0)
        u1 = 0.9 * y1 + 0.3 * np.sin(y1)
    elif kind == 1:  # step-like (converged-looking) with repeats
        u0 = np.round(s * np.sign(y0) - y0, 2)
        u1 = np.round(s * np.tanh(y1), 3)
    else:            # rough
        u0 = rng.normal(0, s, d0)
        u1 = rng.normal(0, 3, d1) + y1
    h = prob.grids[0].spacing
    r = float(rng.choice([9.5, 19.5, 40.5])) * h
    cfg, ocfg = P.SolverConfig(search_radius=r), orc.OracleConfig(search_radius=r)
    U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
    p = orc.OracleWitsenhausen(k=k, sigma=s, grid0=g0, grid1=g1, f0=prob._f0, fw0=prob._fw0)
    for m, d in ((0, d0), (1, d1)):
        pts = np.unique(np.concatenate([[0, d - 1], rng.choice(d, args.points, replace=False)])).astype(np.int64)
        for kind_, dev, ref in (("local", P.local_update_phase, orc.local_update_phase),
                                ("exhaustion", P.partial_exhaustion_phase, orc.partial_exhaustion_phase)):
            got = dev(prob, m, U, cfg)[pts]
            want = ref(p, m, u0, u1, ocfg, points=pts)
            if got.view(np.uint64).tolist() != np.asarray(want).view(np.uint64).tolist():
                bad += 1
                print(f"MISMATCH trial {t} {kind_}{m} d0={d0} d1={d1} k={k} s={s} r={r / h}h", flush=True)
    pts = np.unique(np.concatenate([[0, d0 - 1], rng.choice(d0, args.points, replace=False)])).astype(np.int64)
    terms = prob.device_objective_terms(U).cpu().numpy()
    if terms[pts].view(np.uint64).tolist() != p.cost_batch(0, u0[pts], pts, u0, u1).view(np.uint64).tolist():
        bad += 1
        print(f"MISMATCH trial {t} objective", flush=True)
print(f"{args.trials} trials, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
