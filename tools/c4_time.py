"""Config 4 wall time (64 instances, d=2000, to convergence, batched engine):
median of --reps sweeps.  Used to compare library variants:

    UCP_B200_LIB=variants/x.so python tools/c4_time.py
"""
import argparse
import gc
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

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--instances", type=int, default=64)
args = ap.parse_args()
torch.cuda.set_device(0)
sweep = [(0.05 + 0.95 * i / (args.instances - 1), (3.0, 5.0, 7.0)[i % 3]) for i in range(args.instances)]
P.solve_many([P.Witsenhausen(k=k, sigma=s) for k, s in sweep], P.SolverConfig(max_rounds=1))
walls, Js = [], None
for _ in range(args.reps):
    probs = [P.Witsenhausen(k=k, sigma=s) for k, s in sweep]
    gc.collect()
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = P.solve_many(probs, P.SolverConfig())
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t)
    Js = [r.final_objective for r in res]
print(json.dumps({"lib": os.environ.get("UCP_B200_LIB", "default"), "wall_s_median": float(np.median(walls)),
                  "walls_s": [round(w, 4) for w in walls],
                  "J_bits_hash": hash(tuple(np.array(Js).view(np.uint64).tolist()))}), flush=True)
