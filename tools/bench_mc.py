"""Monte-Carlo objective throughput: device estimator
(Philox draws, costs and fixed-order reduction in HBM) at large sample
counts, the reference-semantics estimator (host PCG64 draws, device costs),
and the CPU restatement (NumPy, oracle) beside them.  One JSON line per case.

    python tools/bench_mc.py [--samples 1073741824] [--cases wc,zd,inv3]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1908_04489_b200 as P  # noqa: E402
from paper_1908_04489_b200 import _lib  # noqa: E402


def make(tag):
    if tag == "wc":
        return P.Witsenhausen(grids=[(-25.0, 25.0, 2 ** 20)] * 2)
    if tag == "zd":
        return P.ZeroDelay()
    return P.Inventory(stages=3)


def oracle_make(orc, tag):
    if tag == "wc":
        return orc.OracleWitsenhausen(grid0=(-25.0, 25.0, 2 ** 20), grid1=(-25.0, 25.0, 2 ** 20))
    if tag == "zd":
        return orc.OracleZeroDelay()
    return orc.OracleInventory(stages=3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=2 ** 30)
    ap.add_argument("--cases", default="wc,zd,inv3")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    from oracle import oracle as orc

    for tag in args.cases.split(","):
        prob = make(tag)
        U = prob.identity_controllers()
        J = prob.objective(U)
        P.device_monte_carlo_objective(prob, U, 1 << 20, seed=1)  # warm-up
        torch.cuda.synchronize()
        n = args.samples
        times = []
        for r in range(args.reps):
            l0 = _lib.launch_count()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sums = P.device_monte_carlo_objective(prob, U, n, seed=100 + r, return_device=True)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            launches = _lib.launch_count() - l0
        est, se = P.device_monte_carlo_objective(prob, U, n, seed=100)
        t = float(np.median(times))
        # reference-semantics estimator: PCG64 on the host, costs on the device
        nref = 10 ** 7
        t0 = time.perf_counter()
        rest, rse = P.monte_carlo_objective(prob, U, P.OracleConfig(mc_samples=nref, seed=8))
        tref = time.perf_counter() - t0
        # CPU restatement (NumPy): draws + costs, bounded sample
        ncpu = 10 ** 7
        p = oracle_make(orc, tag)
        Us = [U.values(m) for m in range(prob.M)]
        from paper_1908_04489_b200.montecarlo import _host_draws

        t0 = time.perf_counter()
        costs = orc.simulate_cost(p, Us, _host_draws(prob, np.random.default_rng(8), ncpu))
        float(np.mean(costs))
        tcpu = time.perf_counter() - t0
        print(json.dumps({
            "case": tag, "grids": [g.d for g in prob.grids], "controllers": "identity", "J_quadrature": J,
            "device": {"samples": n, "s": t, "samples_per_s": n / t, "estimate": est, "stderr": se,
                       "z": (est - J) / se, "launches": launches, "passes": 2},
            "reference_estimator": {"samples": nref, "s": tref, "samples_per_s": nref / tref, "estimate": rest,
                                    "stderr": rse, "note": "host NumPy PCG64 draws (bitwise the reference), device costs"},
            "cpu_numpy": {"samples": ncpu, "s": tcpu, "samples_per_s": ncpu / tcpu, "cores": 1,
                          "kind": "port (oracle.simulate_cost, NumPy)"},
        }), flush=True)


if __name__ == "__main__":
    main()
