"""Reference vs fast (arithmetic="fma") arithmetic on the bench snapshot: one
step of every phase per mode, event-timed, plus how the outputs differ.

    python tools/fast_mode_ab.py [--log2d 18]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1908_04489_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2d", type=int, default=18)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
d = 1 << args.log2d
sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
u0, u1 = bench.resample(sol["u0"], d), bench.resample(sol["u1"], d)
out = {}
MODES = ("reference", "fma", "table")
for mode in MODES:
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2, arithmetic=mode)
    cfg = P.SolverConfig(search_radius=19.5 * prob.grids[0].spacing)
    U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
    ms, res = {}, {}
    for rep in range(args.reps + 1):
        for name, kind, m in bench.PHASES:
            sweep = prob.device_local_update if kind == "local" else prob.device_exhaustion
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = sweep(m, U, cfg)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                ms[name] = ms.get(name, 0.0) + e0.elapsed_time(e1) / args.reps
            res[name] = r.cpu().numpy()
        res["J"] = prob.device_objective(U)
    out[mode] = (ms, res)
ref = out["reference"][1]
# the objective (reference arithmetic) of each mode's new controller after
# each phase (the other stage's snapshot fixed): do rounding-ambiguous decisions move J?
jprob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)


def J_of(u_new, m):
    v = (u_new, u1) if m == 0 else (u0, u_new)
    return jprob.objective(P.ControllerSet((P.SampledController(jprob.grids[0], v[0]),
                                            P.SampledController(jprob.grids[1], v[1]))))


PH = ("local0", "local1", "exh0", "exh1")
J_after = {m: {ph: J_of(out[m][1][ph], int(ph[-1])) for ph in PH} for m in MODES}
line = {"log2d": args.log2d, "ms_reference": out["reference"][0]}
for mode in MODES[1:]:
    fast = out[mode][1]
    line[mode] = {"ms": out[mode][0], "speedup": {k: out["reference"][0][k] / out[mode][0][k] for k in out[mode][0]},
                  "points_differing": {k: int(np.count_nonzero(ref[k] != fast[k]))
                                       for k in ("local0", "local1", "exh0", "exh1")},
                  "J": fast["J"], "J_rel_diff": abs(fast["J"] - ref["J"]) / ref["J"],
                  "J_after_phase_rel_diff": {ph: (J_after[mode][ph] - J_after["reference"][ph]) / J_after["reference"][ph]
                                             for ph in PH},
                  "max_abs_diff": {k: float(np.max(np.abs(fast[k] - ref[k]))) for k in PH},
                  "local0_points_rel_diff_above_1e-9": int(np.count_nonzero(
                      np.abs(fast["local0"] - ref["local0"]) > 1e-9 * np.maximum(np.abs(ref["local0"]), 1e-300))),
                  "max_rel_diff_local0": float(np.max(np.abs(fast["local0"] - ref["local0"]) /
                                                      np.maximum(np.abs(ref["local0"]), 1e-300)))}
line["J_reference"] = ref["J"]
print(json.dumps(line), flush=True)
