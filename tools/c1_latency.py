"""Why does C1 (d=2000, 22 rounds) time-to-converge vary from solve to solve?

Runs N solves of fresh problems in each of several modes and prints one JSON
line per mode with the wall times, the per-round host times, and the SM clock
sampled (nvidia-smi, 50 ms) during the solves:

  fresh      a new Witsenhausen per solve (new device context + graph captures)
  same       the same problem re-solved (graphs and workspace warm)
  prewarm    fresh problems, each solve preceded by ~100 ms of device work
             (the SM clock ramps up before the latency-bound solve starts)
  nographs   fresh problems with UCP_GRAPHS=0 semantics (graphs=False blocks)

    python tools/c1_latency.py [--n 9]
"""
from __future__ import annotations

import argparse
import gc
import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1908_04489_b200 as P  # noqa: E402
from paper_1908_04489_b200 import _lib, witsenhausen  # noqa: E402
from paper_1908_04489_b200._device import ptr  # noqa: E402


class Clocks:
    def __init__(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=timestamp,clocks.sm,power.draw",
                                   "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                  stderr=subprocess.DEVNULL)

    def stop(self):
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 2]
        return {"sm_mhz_median": float(np.median(sm)) if sm else None, "sm_mhz_min": min(sm) if sm else None,
                "sm_mhz_max": max(sm) if sm else None, "samples": len(sm)}


def busy(ms=100.0):
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.empty(sms * 8 * 256, dtype=torch.float64, device="cuda")
    t = time.perf_counter()
    while (time.perf_counter() - t) * 1e3 < ms:
        _lib.call("ucp_fp64_probe", sms * 8, 256, 512, ptr(sink), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=9)
    ap.add_argument("--modes", default="fresh,same,prewarm,nographs,fresh")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    P.solve(P.Witsenhausen(), P.SolverConfig(max_rounds=1))
    same = P.Witsenhausen()
    P.solve(same, P.SolverConfig())
    for mode in args.modes.split(","):
        witsenhausen.GRAPH_BLOCKS = mode != "nographs"
        walls, rounds_ms = [], []
        clk = Clocks()
        for _ in range(args.n):
            pr = same if mode == "same" else P.Witsenhausen()
            pr.objective(pr.identity_controllers())
            gc.collect()
            if mode == "prewarm":
                busy()
            torch.cuda.synchronize()
            t = time.perf_counter()
            res = P.solve(pr, P.SolverConfig())
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t)
            rounds_ms.append([round(r.wall_ms, 2) for r in res.rounds])
        c = clk.stop()
        witsenhausen.GRAPH_BLOCKS = True
        print(json.dumps({"mode": mode, "wall_s_median": float(np.median(walls)), "wall_s_min": min(walls),
                          "wall_s_max": max(walls), "walls_s": [round(w, 5) for w in walls], "clocks": c,
                          "rounds_ms_first": rounds_ms[0], "rounds_ms_slowest":
                              rounds_ms[int(np.argmax(walls))]}), flush=True)


def profile_fresh(n=5):
    """cProfile of n fresh-problem solves vs n re-solves of one problem: where
    the fresh solves' extra host time goes (top functions by own time)."""
    import cProfile
    import pstats

    torch.cuda.set_device(0)
    P.solve(P.Witsenhausen(), P.SolverConfig(max_rounds=1))
    same = P.Witsenhausen()
    P.solve(same, P.SolverConfig())
    for mode in ("fresh", "same"):
        pr_ = cProfile.Profile()
        for _ in range(n):
            pr = same if mode == "same" else P.Witsenhausen()
            pr.objective(pr.identity_controllers())
            gc.collect()
            torch.cuda.synchronize()
            pr_.enable()
            P.solve(pr, P.SolverConfig())
            torch.cuda.synchronize()
            pr_.disable()
        print(f"==== {mode}: {n} solves, top 25 by own time", flush=True)
        pstats.Stats(pr_).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    if "--profile" in sys.argv:
        profile_fresh()
    else:
        main()
