"""A/B of the walk's no-op tail exit (UCP_TAIL_EXIT, csrc walk_tail_noop) on the
bench snapshot: the d=2000 solution interpolated onto a 2^log2d grid, every
stage-0/1 phase once + the objective.  Writes the phase outputs to --out (npz)
and prints one JSON line of event-timed phase milliseconds.  Run it once with
UCP_TAIL_EXIT=0 and once with 1 (the switch is read at library load) and
compare the npz files bitwise (tests/test_gpu_tail_exit.py does exactly that).
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2d", type=int, default=17)
    ap.add_argument("--window-nodes", type=int, default=39)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--out", required=True)
    ap.add_argument("--perturb", choices=["none", "spike", "identity", "huge"], default="none",
                    help="adversarial stage-1 controller: far-tail spikes (large finite addends after the "
                         "peak), u1 = y (odd: acc1 ~ 0 near s = 0), one 1e200 value (v*v overflows)")
    args = ap.parse_args()

    import torch

    import bench
    import paper_1908_04489_b200 as P

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    d = 1 << args.log2d
    res = P.solve(P.Witsenhausen(k=bench.K_WC, sigma=bench.SIGMA), P.SolverConfig())
    u0h = bench.resample(res.controllers.values(0), d)
    u1h = bench.resample(res.controllers.values(1), d)
    y = np.linspace(bench.SPAN[0], bench.SPAN[1], d)
    if args.perturb == "spike":
        u1h[d - 3] = 1e6
        u1h[d // 2 + d // 7] = -3e5
        u1h[d // 5] = 2e4
    elif args.perturb == "identity":
        u1h = y.copy()
    elif args.perturb == "huge":
        u1h[d // 2 + d // 9] = 1e200
    prob = P.Witsenhausen(k=bench.K_WC, sigma=bench.SIGMA, grids=[(*bench.SPAN, d), (*bench.SPAN, d)])
    h = prob.grids[0].spacing
    cfg = P.SolverConfig(search_radius=(args.window_nodes / 2.0) * h)
    U = P.ControllerSet(tuple(P.SampledController(prob.grids[m], torch.from_numpy(u).to(dev))
                              for m, u in ((0, u0h), (1, u1h))))
    sh = P.LOCAL
    stream = torch.cuda.current_stream(dev)
    outs, ms = {}, {}
    for rep in range(args.reps + 1):  # rep 0 warms up (lazy loading, workspace growth)
        for name, kind, m in bench.PHASES:
            sweep = prob.device_local_update if kind == "local" else prob.device_exhaustion
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            try:
                r = sweep(m, U, cfg, sh)
            except Exception as exc:  # the error (type and text) must match too
                r = np.frombuffer(f"{type(exc).__name__}: {exc}".encode(), dtype=np.uint8)
            e1.record(stream)
            torch.cuda.synchronize()
            if rep:
                ms[name] = ms.get(name, 0.0) + e0.elapsed_time(e1) / args.reps
            outs[name] = np.asarray(r.cpu().numpy() if hasattr(r, "cpu") else np.asarray(r))
        try:
            outs["J"] = np.array([float(prob.device_objective(U, sh))])
        except Exception as exc:
            outs["J"] = np.frombuffer(f"{type(exc).__name__}: {exc}".encode(), dtype=np.uint8)
    np.savez(args.out, **outs)
    print(json.dumps({"log2d": args.log2d, "perturb": args.perturb, "phase_ms": ms,
                      "J": float(outs["J"][0]) if outs["J"].dtype == np.float64 else bytes(outs["J"]).decode()}))


if __name__ == "__main__":
    main()
