import sys, time, json
from collections import defaultdict
sys.path.insert(0, '/root/repo')
import torch
from torch.profiler import ProfilerActivity, profile
import paper_1908_04489_b200 as P
p = P.Witsenhausen(grids=[(-25.0, 25.0, 14000)] * 2)
P.solve(p, P.SolverConfig(max_rounds=1)); torch.cuda.synchronize()
p = P.Witsenhausen(grids=[(-25.0, 25.0, 14000)] * 2)
agg = defaultdict(lambda: [0, 0.0])
t = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = P.solve(p, P.SolverConfig()); torch.cuda.synchronize()
wall = time.perf_counter() - t
for e in prof.events():
    if e.device_type.name == "CUDA":
        n = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:40]
        agg[n][0] += 1; agg[n][1] += e.device_time_total / 1e3
busy = sum(v[1] for v in agg.values())
print(json.dumps({"wall_under_profiler": wall, "busy_ms": busy, "rounds": r.total_rounds,
                  "top": {k: [v[0], round(v[1], 1)] for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]}}, separators=(",", ":")))
