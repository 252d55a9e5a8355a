"""Time (and, under ncu, list the launches of) the default-grid C1 solve."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1908_04489_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = P.Witsenhausen()
p.objective(p.identity_controllers())
torch.cuda.synchronize()
for _ in range(n):
    t = time.perf_counter()
    r = P.solve(p)
    torch.cuda.synchronize()
    print("C1 solve s", round(time.perf_counter() - t, 4), r.total_rounds, repr(r.final_objective), flush=True)

# per-iteration device time of each block kind at the converged snapshot
cfg = P.SolverConfig()
U = r.controllers
for kind in ("local", "exhaustion"):
    P.run_block(p, U, cfg, 2, kind)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.run_block(p, U, cfg, 10, kind)
    e1.record()
    torch.cuda.synchronize()
    print(f"{kind} iteration (both stages): {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
for _ in range(2):
    t = time.perf_counter()
    p.objective(U)
    print(f"objective (incl. D2H sync): {(time.perf_counter() - t) * 1e6:.1f} us")

def tphase(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for m in (0, 1):
    print(f"local m={m}: {tphase(lambda: p.device_local_update(m, U, cfg)):.1f} us;  "
          f"exhaustion m={m}: {tphase(lambda: p.device_exhaustion(m, U, cfg)):.1f} us", flush=True)
p.flush_errors()
