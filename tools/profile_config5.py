"""Kernel-time breakdown (CUPTI) of config-5 solves (ZeroDelay d=16384,
Inventory M=3 d=4096), for ncu target selection and profiles/.

    python tools/profile_config5.py [zd_16384,inv3_4096,inv8_601]
"""
import json
import sys
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1908_04489_b200 as P  # noqa: E402

cases = {"zd_16384": lambda: P.ZeroDelay(grids=[(-5.0, 5.0, 16384), (-6.0, 6.0, 16384)]),
         "inv3_4096": lambda: P.Inventory(stages=3, grids=[(-3.0, 3.0, 4096)] * 3),
         "inv8_601": lambda: P.Inventory(stages=8, grids=[(-3.0, 3.0, 601)] * 8)}
pick = sys.argv[1].split(",") if len(sys.argv) > 1 else ["zd_16384", "inv3_4096"]
for name, mk in ((k, cases[k]) for k in pick):
    P.solve(mk(), P.SolverConfig(max_rounds=1))
    torch.cuda.synchronize()
    agg = defaultdict(lambda: [0, 0.0])
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.solve(mk(), P.SolverConfig())
        torch.cuda.synchronize()
    for e in prof.events():
        if e.device_type.name == "CUDA":
            n = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:48]
            agg[n][0] += 1
            agg[n][1] += e.device_time_total / 1e3
    tot = sum(v[1] for v in agg.values())
    top = sorted(agg.items(), key=lambda kv: -kv[1][1])[:8]
    print(json.dumps({"case": name, "kernel_ms": round(tot, 2),
                      "top": {k: [v[0], round(v[1], 2), round(100 * v[1] / tot, 1)] for k, v in top}}), flush=True)
