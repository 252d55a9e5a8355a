"""Small cases that drive every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per gpurun call).

    compute-sanitizer --tool racecheck --error-exitcode 99 python tools/sanitize_cases.py [case ...]

Cases (default: all), each checked against the oracle where cheap so a
sanitizer run is also a parity run:
  smoke    d=201 local + exhaustion + objective (latency walks, k_mom_fused, graph-free)
  block    d=201 full solve (graph-replayed blocks, deferred objective, PDL chain)
  walk     d=8192, 39-node windows: throughput-mode walks (tail exit, k_vsuf),
           both exhaustion phases, both local phases, objective
  moments  d=8192 stage-1 local update with the persistent k_moments
           (UCP_FUSED_MAX_QUERIES=0 is set by this script for that case: run it
           in its own process, e.g. ``... sanitize_cases.py moments``)
  batch    solve_many of 6 instances at d=201 (batched engine work queues)
  c5       ZeroDelay and Inventory M=3 (small and ~2k-4k grids), two rounds each, and the
           uniform-noise kernels vs the oracle
  mc       Philox Monte-Carlo objective, 2^16 samples
  table    d=2^15 exhaustion in the opt-in table arithmetic (k_ex_cells +
           ex_moments) vs the reference arithmetic: picks equal but for near-ties;
           d=2^19 local updates of both stages (cells; k_mom_fgt)
  tz       the chunked exact trapezoid (k_tz_*) on 2^17-sample sequences with
           ties, sign changes and binade crossings vs the oracle's serial sum
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CASES = ("smoke", "block", "walk", "moments", "batch", "c5", "mc", "table", "tz")


def main(argv):
    cases = argv or list(CASES)
    if "moments" in cases:
        if len(cases) > 1:
            raise SystemExit("run the 'moments' case in its own process (it sets UCP_FUSED_MAX_QUERIES)")
        os.environ["UCP_FUSED_MAX_QUERIES"] = "0"
    import numpy as np
    import torch

    import __graft_entry__ as g
    import paper_1908_04489_b200 as P
    from oracle import oracle as orc

    torch.cuda.set_device(0)
    orc.build()

    def same(a, b, what):
        a = np.asarray(a, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        assert a.tobytes() == b.tobytes(), what

    for case in cases:
        if case == "smoke":
            g.smoke()
        elif case == "block":
            prob = P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
            res = P.solve(prob, P.SolverConfig(max_rounds=4))
            p = orc.OracleWitsenhausen(grid0=(-25.0, 25.0, 201), grid1=(-25.0, 25.0, 201), f0=prob._f0,
                                       fw0=prob._fw0)
            u0, u1, J, rounds, term = orc.solve(p, orc.OracleConfig(max_rounds=4))
            same(res.controllers.values(0), u0, "block u0")
            same(res.final_objective, J, "block J")
        elif case in ("walk", "moments"):
            d = 8192
            prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
            h = prob.grids[0].spacing
            y = prob.grids[0].points
            rng = np.random.default_rng(5)
            u0 = -0.9 * y + 0.05 * rng.standard_normal(d)
            u1 = 0.8 * y + 0.05 * rng.standard_normal(d)
            U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
            cfg = P.SolverConfig(search_radius=19.5 * h)
            p = orc.OracleWitsenhausen(grid0=(-25.0, 25.0, d), grid1=(-25.0, 25.0, d), f0=prob._f0, fw0=prob._fw0)
            ocfg = orc.OracleConfig(search_radius=19.5 * h)
            pts = np.array([0, 1, 77, d // 3, d // 2, d - 2, d - 1], dtype=np.int64)
            phases = [("local", 1)] if case == "moments" else [("local", 0), ("local", 1),
                                                              ("exhaustion", 0), ("exhaustion", 1)]
            for kind, m in phases:
                if kind == "local":
                    got = P.local_update_phase(prob, m, U, cfg)
                    want = orc.local_update_phase(p, m, u0, u1, ocfg, points=pts)
                else:
                    got = P.partial_exhaustion_phase(prob, m, U, cfg)
                    want = orc.partial_exhaustion_phase(p, m, u0, u1, ocfg, points=pts)
                same(got[pts], want, f"{case} {kind}{m}")
            if case == "walk":
                terms = prob.device_objective_terms(U).cpu().numpy()
                same(terms[pts], p.cost_batch(0, u0[pts], pts, u0, u1), "walk objective terms")
        elif case == "batch":
            sweep = [(0.05 + 0.19 * i, (3.0, 5.0, 7.0)[i % 3]) for i in range(6)]
            probs = [P.Witsenhausen(k=k, sigma=s, grids=[(-25.0, 25.0, 201)] * 2) for k, s in sweep]
            res = P.solve_many(probs, P.SolverConfig(max_rounds=3))
            for (k, s), r, pr in zip(sweep, res, probs):
                p = orc.OracleWitsenhausen(k=k, sigma=s, grid0=(-25.0, 25.0, 201), grid1=(-25.0, 25.0, 201),
                                           f0=pr._f0, fw0=pr._fw0)
                u0, u1, J, rounds, term = orc.solve(p, orc.OracleConfig(max_rounds=3))
                same(r.final_objective, J, f"batch J k={k} sigma={s}")
        elif case == "c5":
            for prob in (P.ZeroDelay(grids=[(-5.0, 5.0, 257), (-6.0, 6.0, 257)]),
                         P.Inventory(stages=3, grids=[(-3.0, 3.0, 129)] * 3),
                         P.ZeroDelay(grids=[(-5.0, 5.0, 3000), (-6.0, 6.0, 2048)]),
                         P.Inventory(stages=3, grids=[(-3.0, 3.0, 1500)] * 3)):
                P.solve(prob, P.SolverConfig(max_rounds=2))
            # the uniform-noise kernels (producer/consumer form) vs the oracle, many stages per CTA
            rng = np.random.default_rng(9)
            d, a, h = 4096, -3.0, 6.0 / 4095
            x = np.sort(rng.uniform(-4.0, 4.0, 3000))
            x[rng.choice(3000, 40, replace=False)] = rng.uniform(-4.0, 4.0, 40)  # out of order
            masses = rng.uniform(0.0, 1.0, 3000)
            same(P.kernels.unif_propagate(masses, x, a, h, d, 1.0), orc.unif_propagate(masses, x, a, h, d, 1.0),
                 "unif_propagate")
            y = rng.uniform(-3.2, 3.2, 5000)
            vals = rng.normal(0.0, 2.0, 3000)
            got = P.kernels.unif_moments_points(y, x, masses, vals, a, h, d, 1.0)
            want = orc.unif_moments_points(y, x, masses, vals, a, h, d, 1.0)
            for k in range(3):
                same(got[k], want[k], f"unif_moments_points {k}")
        elif case == "mc":
            prob = P.Witsenhausen(grids=[(-25.0, 25.0, 2001)] * 2)
            P.device_monte_carlo_objective(prob, prob.identity_controllers(), 1 << 16, seed=3)
        elif case == "table":
            d = 1 << 15
            res = P.solve(P.Witsenhausen(), P.SolverConfig(max_rounds=2))
            yc, y = np.linspace(-25, 25, 2000), np.linspace(-25, 25, d)
            u0 = np.interp(y, yc, res.controllers.values(0))
            u1 = np.interp(y, yc, res.controllers.values(1))
            outs = []
            for arith in ("reference", "table"):
                prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2, arithmetic=arith)
                U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
                cfg = P.SolverConfig(search_radius=19.5 * prob.grids[0].spacing)
                outs.append(P.partial_exhaustion_phase(prob, 0, U, cfg))
            ndiff = int(np.count_nonzero(outs[0] != outs[1]))
            assert ndiff <= d // 1000, f"table picks differ at {ndiff} points"
            # the local update on the cells (stage 0) and, at h1 <= 1e-4, the
            # stage-1 expansion moments (k_mom_fgt, grid ends exact)
            d = 1 << 19
            y = np.linspace(-25, 25, d)
            u0 = np.interp(y, yc, res.controllers.values(0))
            u1 = np.interp(y, yc, res.controllers.values(1))
            outs = []
            for arith in ("reference", "table"):
                prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2, arithmetic=arith)
                U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
                cfg = P.SolverConfig(search_radius=19.5 * prob.grids[0].spacing)
                outs.append((P.local_update_phase(prob, 0, U, cfg), P.local_update_phase(prob, 1, U, cfg)))
            assert np.isfinite(outs[1][0]).all()
            assert np.max(np.abs(outs[1][1] - outs[0][1])) <= 2e-6, "table stage-1 local update"
        elif case == "tz":
            rng = np.random.default_rng(17)
            n = 1 << 17
            seqs = [rng.normal(0, 1, n), np.concatenate([[2.0 ** 54], rng.integers(-7, 8, n - 1).astype(float)]),
                    np.concatenate([rng.uniform(0, 1, n // 2), -rng.uniform(0, 1, n - n // 2)]),
                    rng.uniform(0, 0.3, n)]
            for x in seqs:
                same(P.kernels.trapezoid_sum(x, 0.01), orc.trapezoid_sum(x, 0.01), "chunked trapezoid")
        else:
            raise SystemExit(f"unknown case {case!r}; one of {CASES}")
        torch.cuda.synchronize()
        print(f"case {case}: ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
