"""Cross-check of bench.py's CPU baseline extrapolation (the reference's
algorithm -- the oracle's C/OpenMP port -- timed on bounded samples of every
phase, scaled by d/n): at grid sizes where a FULL CPU step is affordable, time
the full step phase by phase next to the sampled estimate and report the error.
(A single uniform sample -- the same few hundred points in every phase,
value = sampled evaluations / seconds -- was tried: per-call overheads of the
cheap phases put it 57% off at 2^16, so each phase keeps its own sample size.)

    python tools/cpu_extrapolation_check.py [--log2d 14 16] [--cpu-seconds 8]

One JSON line per size.  The full step also checks the sampled outputs: the
oracle's sampled results equal the full run's at those points (same code).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2d", type=int, nargs="+", default=[14, 16])
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--window-nodes", type=int, default=39)
    args = ap.parse_args()
    orc.build()
    orc.set_threads(os.cpu_count() or 1)
    sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
    for lg in args.log2d:
        d = 1 << lg
        u0, u1 = bench.resample(sol["u0"], d), bench.resample(sol["u1"], d)
        p = orc.OracleWitsenhausen(k=bench.K_WC, sigma=bench.SIGMA, grid0=(*bench.SPAN, d), grid1=(*bench.SPAN, d))
        r = (args.window_nodes / 2.0) * p.h0
        cfg = orc.OracleConfig(search_radius=r)
        counts = bench.workload_counts(u0, u1, d, r)
        q = bench.cpu_sample_step(orc, p, u0, u1, d, r, counts, args.cpu_seconds)
        est, thr, sample, outs = q["step_s_extrapolated"], q["threads"], q["sample"], q["outs"]
        est_phase = q["phase_s"]
        full, full_out = {}, {}
        for name, fn in (("local0", lambda: orc.local_update_phase(p, 0, u0, u1, cfg)),
                         ("local1", lambda: orc.local_update_phase(p, 1, u0, u1, cfg)),
                         ("exh0", lambda: orc.partial_exhaustion_phase(p, 0, u0, u1, cfg)),
                         ("exh1", lambda: orc.partial_exhaustion_phase(p, 1, u0, u1, cfg)),
                         ("objective", lambda: p.cost_batch(0, u0, np.arange(d, dtype=np.int64), u0, u1))):
            t = time.perf_counter()
            full_out[name] = fn()
            full[name] = time.perf_counter() - t
        same = all(np.array_equal(full_out[k][idx].view(np.uint64), np.asarray(v).view(np.uint64))
                   for k, (idx, v) in outs.items())
        tot = sum(full.values())
        print(json.dumps({
            "grid_points": d, "threads": thr, "host": orc.host_cpu_description(),
            "full_step_s": tot, "sampled_estimate_s": est, "rel_error": (est - tot) / tot,
            "phase_full_s": full, "phase_estimate_s": est_phase,
            "phase_rel_error": {k: (est_phase[k] - full[k]) / full[k] for k in full},
            "sample": sample, "sampled_outputs_equal_full_run": bool(same)}), flush=True)


if __name__ == "__main__":
    main()
