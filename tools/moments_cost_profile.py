"""Stage-1 moments cost along the grid (bench snapshot at 2^20): event-timed
k_moments over consecutive 32,768-query slices, next to the modelled work
(live-tile pairs, Witsenhausen._moments_weights) -- how well the shard
weights predict the kernel's time."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1908_04489_b200 as P  # noqa: E402
from paper_1908_04489_b200.witsenhausen import Witsenhausen  # noqa: E402

d = 1 << 20
sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
u0 = bench.resample(sol["u0"], d)
prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
y = torch.from_numpy(prob.grids[0].points).cuda()
x1 = y + torch.from_numpy(u0).cuda()
w = torch.from_numpy(prob._fw0).cuda()
model = Witsenhausen._moments_weights(x1, y).double()
P.kernels.gauss_moments_points(y[:40000], x1, w, -25.0, prob.grids[0].spacing, d)
S = 32768
rows = []
for b in range(0, d, S):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        P.kernels.gauss_moments_points(y[b:b + S], x1, w, -25.0, prob.grids[0].spacing, d)
    e1.record()
    torch.cuda.synchronize()
    rows.append((b, e0.elapsed_time(e1) / 3, float(model[b:b + S].sum())))
t = np.array([r[1] for r in rows]); m = np.array([r[2] for r in rows])
print(json.dumps({"slice": S, "ms": t.round(3).tolist(), "model_pairs_1e9": (m / 1e9).round(3).tolist(),
                  "ns_per_pair": (t * 1e6 / m).round(4).tolist()}))
