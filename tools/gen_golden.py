"""Generate the golden parity fixtures under tests/golden/ by running the
reference package itself (``/root/reference/pkg/src/ucpsolve``, numba
backend) in this container.

The reference cannot travel to the GPU box, so its outputs are frozen here
as small .npz fixtures together with every host-computed input they depend
on (NumPy-exp densities f0/fw0 included), and the tests replay them against
the oracle (CPU) and the CUDA path (GPU).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/gen_golden.py [--skip-big]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("UCPSOLVE_BACKEND", "numba")
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402

from ucpsolve import kernels  # noqa: E402
from ucpsolve.grids import ControllerSet, SampledController, nearest_indices  # noqa: E402
from ucpsolve.numerics import pdf  # noqa: E402
from ucpsolve.problems import Inventory, Witsenhausen, ZeroDelay  # noqa: E402
from ucpsolve.solver import (  # noqa: E402
    SolverConfig,
    local_update_phase,
    partial_exhaustion_phase,
    solve,
)

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"
assert kernels.BACKEND == "numba", kernels.BACKEND


def perturbed(problem, seed=0, scale=0.5):
    # same recipe as the reference's tests/conftest.py:37-44
    rng = np.random.default_rng(seed)
    return ControllerSet(tuple(
        SampledController(g, problem.project(m, g.points + scale * rng.uniform(-1.0, 1.0, g.d)))
        for m, g in enumerate(problem.grids)))


def kernels_fixture():
    rng = np.random.default_rng(0)
    out = {}
    for tag, (a, b, d, n) in {"k307": (-9.0, 9.0, 307, 900), "k2": (-1.0, 1.0, 2, 40),
                              "k64": (-25.0, 25.0, 64, 300)}.items():
        h = (b - a) / (d - 1)
        vals = rng.normal(0, 3, d)
        weights = np.abs(rng.normal(0, 1, d)) * h
        centers = rng.uniform(a - 14, b + 14, n)
        # edge centres: exact grid nodes, the cut boundary, far outside
        extra = np.array([a, b, a - 12.0, b + 12.0, a - 13.0, b + 30.0, a + 12.0, b - 12.0,
                          0.5 * (a + b), a + 0.5 * h])
        centers = np.concatenate([centers, extra])
        queries = np.concatenate([rng.uniform(a - 1, b + 1, n), np.linspace(a, b, d)[:8],
                                  np.array([a, b, a - 5.0, b + 5.0])])
        xs = rng.uniform(a - 14, b + 14, d)
        special = np.array([a, b, 0.5 * (a + b)])[: min(3, d)]
        xs[: special.size] = special
        t = kernels.gauss_moments_grid(centers, vals, a, h, d)
        p = kernels.gauss_moments_points(queries, xs, weights, a, h, d)
        out.update({f"{tag}_a": a, f"{tag}_h": h, f"{tag}_d": d, f"{tag}_vals": vals,
                    f"{tag}_weights": weights, f"{tag}_centers": centers, f"{tag}_queries": queries,
                    f"{tag}_xs": xs, f"{tag}_grid_t0": t[0], f"{tag}_grid_t1": t[1],
                    f"{tag}_grid_t2": t[2], f"{tag}_pts_0": p[0], f"{tag}_pts_1": p[1],
                    f"{tag}_pts_2": p[2]})
    # trapezoid / argmin / flatten
    samples = rng.normal(size=1001)
    out["trap_samples"] = samples
    out["trap_value"] = kernels.trapezoid_sum(samples, 0.37)
    costs = np.round(rng.normal(size=500), 1)  # many ties
    offs = np.concatenate([[0], np.sort(rng.choice(np.arange(1, 500), 60, replace=False)), [500]])
    out["argmin_costs"], out["argmin_offsets"] = costs, offs.astype(np.int64)
    out["argmin_out"] = kernels.segmented_argmin(costs, offs.astype(np.int64))
    vals = np.round(rng.normal(size=300), 0)
    lo = np.clip(np.arange(300) - 7, 0, 299).astype(np.int64)
    hi = np.clip(np.arange(300) + 5, 0, 299).astype(np.int64)
    flat, foffs = kernels.flatten_windows(vals, lo, hi)
    out.update(flat_vals=vals, flat_lo=lo, flat_hi=hi, flat_out=flat, flat_offsets=foffs)
    np.savez_compressed(OUT / "kernels.npz", **out)


def wc_phase_fixture(d, tag):
    prob = Witsenhausen(grids=[(-25.0, 25.0, d), (-25.0, 25.0, d)])
    g0, g1 = prob.grids
    cfg = SolverConfig()
    out = {"d": d, "f0": pdf(prob._state_density, g0.points), "fw0": prob._fw0}
    sets = {"ident": prob.identity_controllers(), "pert0": perturbed(prob, 0, 0.5),
            "pert1": perturbed(prob, 1, 2.0)}
    for name, U in sets.items():
        u0, u1 = U.values(0), U.values(1)
        out[f"{name}_u0"], out[f"{name}_u1"] = u0, u1
        out[f"{name}_J"] = prob.objective(U)
        for m in (0, 1):
            g = prob.grids[m]
            u = U.values(m)
            out[f"{name}_c{m}"] = prob.marginal_cost_batch(m, u, g.points, U)
            out[f"{name}_c{m}_up"] = prob.marginal_cost_batch(m, u + 0.37, g.points, U)
            out[f"{name}_lu{m}"] = local_update_phase(prob, m, U, cfg)
            out[f"{name}_ex{m}"] = partial_exhaustion_phase(prob, m, U, cfg)
            small = SolverConfig(search_radius=3.5 * g.spacing)
            out[f"{name}_exs{m}"] = partial_exhaustion_phase(prob, m, U, small)
        # a full local and exhaustion iteration over both stages (phase chaining)
        V = U
        for ph in (local_update_phase, partial_exhaustion_phase):
            for m in (0, 1):
                V = V.replace(m, V[m].with_values(ph(prob, m, V, cfg)))
        out[f"{name}_it_u0"], out[f"{name}_it_u1"] = V.values(0), V.values(1)
        out[f"{name}_it_J"] = prob.objective(V)
    # segmented m=0 / m=1 with multi-candidate segments (per-candidate f0 repeat)
    rng = np.random.default_rng(5)
    U = sets["pert0"]
    seg_idx = np.sort(rng.choice(d, 25, replace=False)).astype(np.int64)
    counts = rng.integers(1, 9, seg_idx.size)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    u_flat = rng.uniform(-30, 30, int(offs[-1]))
    out.update(seg_idx=seg_idx, seg_offsets=offs, seg_u=u_flat)
    for m in (0, 1):
        out[f"seg_c{m}"] = prob.marginal_cost_segmented(m, u_flat, offs, prob.grids[m].points[seg_idx], U)
    np.savez_compressed(OUT / f"wc_{tag}.npz", **out)


def wc_solve_fixture(d, tag):
    prob = Witsenhausen(grids=[(-25.0, 25.0, d), (-25.0, 25.0, d)])
    t0 = time.perf_counter()
    res = solve(prob, SolverConfig())
    wall = time.perf_counter() - t0
    rounds = np.array([[r.round_index, r.objective, r.local_gain, r.exhaustion_gain, r.local_iters,
                        r.exhaustion_iters, r.objective_after_local] for r in res.rounds])
    np.savez_compressed(OUT / f"wc_solve_{tag}.npz", d=d, rounds=rounds, final_J=res.final_objective,
                        u0=res.controllers.values(0), u1=res.controllers.values(1),
                        termination=res.termination, wall_s=wall,
                        f0=pdf(prob._state_density, prob.grids[0].points), fw0=prob._fw0)
    return res, wall


def fine_fixture(res2000, log2d=20, n_centres=384, n_queries=12):
    """Sampled 2^20 kernels on warm controllers (C1-converged, nearest-resampled)."""
    d = 1 << log2d
    prob = Witsenhausen(grids=[(-25.0, 25.0, d), (-25.0, 25.0, d)])
    g0, g1 = prob.grids
    coarse = res2000.controllers
    cg = coarse.grid(0)
    u0 = coarse.values(0)[nearest_indices(cg, g0.points)]
    u1 = coarse.values(1)[nearest_indices(coarse.grid(1), g1.points)]
    rng = np.random.default_rng(11)
    idx = np.sort(rng.choice(d, n_centres, replace=False))
    idx = np.concatenate([[0, 1, d - 2, d - 1], idx])
    s = g0.points[idx] + u0[idx]
    t = kernels.gauss_moments_grid(s, u1, g1.a, g1.spacing, g1.d)
    q_idx = np.concatenate([[0, d - 1], np.sort(rng.choice(d, n_queries, replace=False))])
    x1 = g0.points + u0
    p = kernels.gauss_moments_points(g1.points[q_idx], x1, prob._fw0, g1.a, g1.spacing, g1.d)
    np.savez_compressed(OUT / f"wc_fine_2p{log2d}.npz", d=d, idx=idx, s=s, t0=t[0], t1=t[1], t2=t[2],
                        q_idx=q_idx, m0=p[0], m1=p[1], m2=p[2])


def generic_fixture(prob, tag, solve_too=True, extra=None):
    """Phases, objective and (optionally) a full solve of a config-5 problem."""
    cfg = SolverConfig()
    out = {"specs": np.array([[g.a, g.b, g.d] for g in prob.grids])}
    if extra:
        out.update(extra)
    sets = {"ident": prob.identity_controllers(), "pert0": perturbed(prob, 0, 0.3), "pert1": perturbed(prob, 1, 1.0)}
    # the solver starts from projected controllers (solver.py:241-248)
    for name, U in sets.items():
        for m in range(prob.M):
            U = U.replace(m, U[m].with_values(prob.project(m, U.values(m))))
        for m in range(prob.M):
            out[f"{name}_u{m}"] = U.values(m)
        out[f"{name}_J"] = prob.objective(U)
        for m in range(prob.M):
            g = prob.grids[m]
            out[f"{name}_c{m}"] = prob.marginal_cost_batch(m, U.values(m), g.points, U)
            out[f"{name}_lu{m}"] = local_update_phase(prob, m, U, cfg)
            out[f"{name}_ex{m}"] = partial_exhaustion_phase(prob, m, U, cfg)
        V = U
        for ph in (local_update_phase, partial_exhaustion_phase):
            for m in range(prob.M):
                V = V.replace(m, V[m].with_values(ph(prob, m, V, cfg)))
        for m in range(prob.M):
            out[f"{name}_it_u{m}"] = V.values(m)
        out[f"{name}_it_J"] = prob.objective(V)
    if solve_too:
        t0 = time.perf_counter()
        res = solve(prob, cfg)
        out["solve_wall_s"] = time.perf_counter() - t0
        out["solve_rounds"] = np.array([[r.round_index, r.objective, r.local_gain, r.exhaustion_gain,
                                         r.local_iters, r.exhaustion_iters, r.objective_after_local]
                                        for r in res.rounds])
        out["solve_J"] = res.final_objective
        out["solve_termination"] = res.termination
        for m in range(prob.M):
            out[f"solve_u{m}"] = res.controllers.values(m)
    np.savez_compressed(OUT / f"{tag}.npz", **out)


def config5_fixtures():
    zd = ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)])
    generic_fixture(zd, "zd_small", extra={"f0": pdf(zd._source, zd.grids[0].points), "fw0": zd._fw0, "pw": 2.0})
    zd2 = ZeroDelay(power_weight=0.7, grids=[(-5.0, 5.0, 400), (-6.0, 6.0, 333)])
    generic_fixture(zd2, "zd_pw07", solve_too=True,
                    extra={"f0": pdf(zd2._source, zd2.grids[0].points), "fw0": zd2._fw0, "pw": 0.7})
    inv = Inventory(grids=[(-3.0, 3.0, 241)] * 2)
    generic_fixture(inv, "inv_m2", extra={"stages": 2, "stage_cost": "piecewise_linear"})
    inv3 = Inventory(stages=3, grids=[(-3.0, 3.0, 121)] * 3)
    generic_fixture(inv3, "inv_m3", extra={"stages": 3, "stage_cost": "piecewise_linear"})
    invq = Inventory(stages=3, stage_cost="quadratic", order_cost=0.3, grids=[(-3.0, 3.0, 97), (-2.5, 3.5, 131),
                                                                               (-3.0, 2.0, 111)])
    generic_fixture(invq, "inv_m3q", extra={"stages": 3, "stage_cost": "quadratic", "order_cost": 0.3})
    inv1 = Inventory(stages=1, grids=[(-3.0, 3.0, 151)])
    generic_fixture(inv1, "inv_m1", extra={"stages": 1, "stage_cost": "piecewise_linear"})
    # default-grid solves (config 5 headline sizes)
    zdd = ZeroDelay()
    generic_fixture(zdd, "zd_default", extra={"f0": pdf(zdd._source, zdd.grids[0].points), "fw0": zdd._fw0,
                                              "pw": 2.0})
    generic_fixture(Inventory(), "inv_default", extra={"stages": 2, "stage_cost": "piecewise_linear"})


class _Recorder:
    """Wraps a NumPy Generator and records what simulate_cost draws."""

    def __init__(self, rng):
        self.rng, self.draws = rng, []

    def normal(self, *a):
        self.draws.append(self.rng.normal(*a))
        return self.draws[-1]

    def uniform(self, *a):
        self.draws.append(self.rng.uniform(*a))
        return self.draws[-1]


def mc_fixture():
    """simulate_cost / monte_carlo_objective (oracle.py:98-105) on small
    problems: the recorded draws, per-sample costs and (estimate, stderr)."""
    from ucpsolve.oracle import OracleConfig, monte_carlo_objective

    out = {}
    cases = {"wc": Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2),
             "zd": ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)]),
             "inv": Inventory(grids=[(-3.0, 3.0, 241)] * 2),
             "inv3q": Inventory(stages=3, stage_cost="quadratic", order_cost=0.3,
                                grids=[(-3.0, 3.0, 97), (-2.5, 3.5, 131), (-3.0, 2.0, 111)])}
    for i, (tag, prob) in enumerate(cases.items()):
        U = perturbed(prob, seed=30 + i, scale=0.4)
        for m in range(prob.M):
            out[f"{tag}_u{m}"] = U.values(m)
        rec = _Recorder(np.random.default_rng(90 + i))
        out[f"{tag}_costs"] = prob.simulate_cost(U, rec, 2000)
        out[f"{tag}_draws"] = np.stack(rec.draws)
        for n, seed in ((2000, 90 + i), (100_000, 7)):
            est, se = monte_carlo_objective(prob, U, OracleConfig(mc_samples=n, seed=seed))
            out[f"{tag}_mc_{n}_{seed}"] = np.array([est, se])
        out[f"{tag}_J"] = prob.objective(U)
    np.savez_compressed(OUT / "mc.npz", **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-big", action="store_true", help="skip the d=2000 solve and 2^20 samples")
    ap.add_argument("--only", choices=["mc"], help="regenerate one fixture file only")
    args = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    if args.only == "mc":
        mc_fixture()
        return
    meta = {"numpy": np.__version__, "backend": kernels.BACKEND}
    import numba

    meta["numba"] = numba.__version__
    kernels_fixture()
    config5_fixtures()
    mc_fixture()
    wc_phase_fixture(201, "d201")
    wc_phase_fixture(2000, "d2000")
    _, w201 = wc_solve_fixture(201, "d201")
    meta["solve_d201_wall_s"] = w201
    if not args.skip_big:
        res, wall = wc_solve_fixture(2000, "d2000")
        meta["solve_d2000_wall_s"] = wall
        fine_fixture(res)
    try:
        meta["cpu"] = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")][0]
    except Exception:  # pragma: no cover
        pass
    (OUT / "META.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
