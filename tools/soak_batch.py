"""Randomised soak: batched engine vs single solves (bitwise) on random grids,
parameters, radii and instance counts.  python tools/soak_batch.py [trials]"""
import sys, numpy as np, torch
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
import paper_1908_04489_b200 as P
from paper_1908_04489_b200.batch import solve_batch
rng = np.random.default_rng(123)
bad = 0
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 24):
    d0 = int(rng.integers(3, 700)); d1 = int(rng.integers(3, 700))
    a = float(rng.uniform(-30, -10)); b = float(rng.uniform(10, 30))
    grids = [(a, b, d0), (a - 1.0, b + 1.0, d1)]
    n = int(rng.integers(2, 9))
    specs = [(float(rng.uniform(0.05, 1.0)), float(rng.choice([3.0, 5.0, 7.0]))) for _ in range(n)]
    cfg = P.SolverConfig(max_rounds=int(rng.integers(1, 4)), search_radius=float(rng.choice([0.2, 0.5, 1.5])))
    got = solve_batch([P.Witsenhausen(k=k, sigma=s, grids=grids) for k, s in specs], cfg)
    for (k, s), r in zip(specs, got):
        ref = P.solve(P.Witsenhausen(k=k, sigma=s, grids=grids), cfg)
        ok = (r.final_objective == ref.final_objective and len(r.rounds) == len(ref.rounds) and
              all(np.array_equal(np.asarray(r.controllers.values(m)).view(np.uint64),
                                 np.asarray(ref.controllers.values(m)).view(np.uint64)) for m in (0, 1)))
        if not ok:
            bad += 1
            print("MISMATCH", trial, grids, k, s, cfg.max_rounds, cfg.search_radius, r.final_objective, ref.final_objective)
print("soak done, mismatches:", bad)
