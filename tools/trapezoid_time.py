"""Time of the objective's trapezoid (bitwise serial sum) at 2^20 and 2^22:
the chunked exact form (default) vs the serial kernel (UCP_TZ_PARALLEL=0).

    python tools/trapezoid_time.py; UCP_TZ_PARALLEL=0 python tools/trapezoid_time.py
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1908_04489_b200 as P  # noqa: E402

res = {"parallel": os.environ.get("UCP_TZ_PARALLEL", "1") != "0"}
for lg in (20, 22):
    x = torch.rand(1 << lg, dtype=torch.float64, device="cuda") * 0.3
    P.kernels.trapezoid_sum(x, 1e-3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        P.kernels.trapezoid_sum(x, 1e-3)  # (includes the 8-byte read-back per call)
    e1.record()
    torch.cuda.synchronize()
    res[f"ms_2p{lg}"] = e0.elapsed_time(e1) / 5
print(json.dumps(res))
