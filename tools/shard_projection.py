"""Multi-GPU projection from one B200: every rank's shard of the bench step,
timed on its own.

This run has one GPU, so the 2/4/8-GPU step cannot be measured.  What CAN be
measured is the work each rank would do: for N = 1, 2, 4, 8 and every rank r,
the four phases and the objective run on rank r's shard of the
work-balanced plans (Witsenhausen._plan; the collectives are stubbed, so a
phase is exactly rank r's kernels), event-timed on this GPU.  Each phase of
the real run ends in an all-gather, so the projected N-GPU step is
sum over phases of max over ranks, plus the exchange (8 MiB per phase at 2^20,
~10-20 us over NVLink 5: reported, not measured).  No kernel waits on another
rank here (B200_PROFILING.md: ranks are never emulated as concurrent launches).

    python tools/shard_projection.py [--log2d 20] [--ns 1 2 4 8]
"""
from __future__ import annotations

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


class Rank(P.Sharding):
    """Rank r of an N-rank plan with the exchanges stubbed (single-GPU timing)."""

    def allgather_(self, buf):
        pass

    def allgather_uneven_(self, buf, bounds):
        pass

    def allreduce_min_(self, t):
        pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2d", type=int, default=20)
    ap.add_argument("--ns", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--window-nodes", type=int, default=39)
    ap.add_argument("--no-rank-warmup", action="store_true",
                    help="skip the untimed pass per rank (large grids; the plan read-back is then timed, ~ms)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    d = 1 << args.log2d
    sol = np.load(ROOT / "tests" / "golden" / "wc_solve_d2000.npz")
    u0, u1 = bench.resample(sol["u0"], d), bench.resample(sol["u1"], d)
    prob = P.Witsenhausen(k=bench.K_WC, sigma=bench.SIGMA, grids=[(*bench.SPAN, d)] * 2)
    cfg = P.SolverConfig(search_radius=(args.window_nodes / 2.0) * prob.grids[0].spacing)
    U = P.ControllerSet(tuple(P.SampledController(prob.grids[m], u) for m, u in ((0, u0), (1, u1))))
    names = [p[0] for p in bench.PHASES] + ["objective"]

    def rank_step(sh, timed):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        ev[0].record()
        for k, (_, kind, m) in enumerate(bench.PHASES):
            (prob.device_local_update if kind == "local" else prob.device_exhaustion)(m, U, cfg, sh)
            ev[k + 1].record()
        prob.device_objective(U, sh)
        ev[-1].record()
        torch.cuda.synchronize()
        return [ev[k].elapsed_time(ev[k + 1]) for k in range(len(names))] if timed else None

    rank_step(Rank(rank=0, world=1), False)  # warm-up: lazy loading, workspace growth
    base = None
    for n in args.ns:
        per_rank = []
        for r in range(n):
            sh = Rank(rank=r, world=n)
            if not args.no_rank_warmup:
                rank_step(sh, False)  # plan cache + warm
            per_rank.append(rank_step(sh, True))
        t = np.array(per_rank)  # [rank, phase] ms
        step = float(t.max(axis=0).sum())
        base = step if n == 1 else base
        print(json.dumps({
            "n_gpus": n, "grid_points": d, "projected_step_ms": step,
            "efficiency_vs_1": None if base is None else base / (n * step),
            "speedup_vs_1": None if base is None else base / step,
            "phase_ms_max_over_ranks": dict(zip(names, t.max(axis=0).round(3).tolist())),
            "imbalance_max_over_mean": dict(zip(names, (t.max(axis=0) / t.mean(axis=0)).round(4).tolist())),
            "rank_step_ms": t.sum(axis=1).round(2).tolist(),
            "rank_phase_ms": t.round(2).tolist(),
            "exchange": f"not included: one all-gather of {d * 8 / 2**20:.0f} MiB per phase over NVLink 5",
        }), flush=True)


if __name__ == "__main__":
    main()
