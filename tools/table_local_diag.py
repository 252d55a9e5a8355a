"""Diagnostic: stage-0 local update, reference vs table arithmetic, on the
bench snapshot; saves both outputs for host-side analysis.

    python tools/table_local_diag.py --log2d 18 --out gpurun_out/tl18.npz
"""
import argparse
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
ap.add_argument("--out", default="gpurun_out/tl.npz")
args = ap.parse_args()
d = 1 << args.log2d
sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
u0, u1 = bench.resample(sol["u0"], d), bench.resample(sol["u1"], d)
res = {}
for mode in ("reference", "table"):
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2, arithmetic=mode)
    cfg = P.SolverConfig(search_radius=19.5 * prob.grids[0].spacing)
    U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
    res[mode] = P.local_update_phase(prob, 0, U, cfg)
    torch.cuda.synchronize()
np.savez(args.out, ref=res["reference"], table=res["table"], u0=u0, u1=u1)
print("saved", args.out, int(np.count_nonzero(res["reference"] != res["table"])))
