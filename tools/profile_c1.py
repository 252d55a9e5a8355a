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
