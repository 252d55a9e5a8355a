"""Config 5: the paper's additional examples (multi-stage inventory, zero-delay
coding) solved on the GPU, with the CPU reference algorithm (oracle port)
timed beside them.  One JSON line per case.

    python tools/bench_config5.py [--cpu-rounds 2] [--cases inv3_601,zd_2000,...]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1908_04489_b200 as P  # noqa: E402

CASES = {
    "inv3_601": ("inventory", 3, 601), "inv4_601": ("inventory", 4, 601), "inv8_601": ("inventory", 8, 601),
    "inv3_4096": ("inventory", 3, 4096), "zd_2000": ("zero_delay", None, 2000),
    "zd_16384": ("zero_delay", None, 16384),
}


def make(kind, M, d, lib):
    if kind == "inventory":
        if lib == "gpu":
            return P.Inventory(stages=M, grids=[(-3.0, 3.0, d)] * M)
        from oracle import oracle as orc

        return orc.OracleInventory(stages=M, grids=[(-3.0, 3.0, d)] * M)
    if lib == "gpu":
        return P.ZeroDelay(grids=[(-5.0, 5.0, d), (-6.0, 6.0, d)])
    from oracle import oracle as orc

    return orc.OracleZeroDelay(grid0=(-5.0, 5.0, d), grid1=(-6.0, 6.0, d))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--cpu-rounds", type=int, default=1, help="rounds of the CPU oracle per case (0: skip)")
    ap.add_argument("--reps", type=int, default=5, help="timed solves per case (median reported)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for name in args.cases.split(","):
        kind, M, d = CASES[name]
        prob = make(kind, M, d, "gpu")
        P.solve(prob, P.SolverConfig(max_rounds=1))  # context + first launches
        walls = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            res = P.solve(prob, P.SolverConfig())
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t)
        wall = float(sorted(walls)[len(walls) // 2])
        line = {"case": name, "problem": kind, "stages": prob.M, "d": d, "gpu_solve_s": wall,
                "gpu_solve_s_all": [round(w, 5) for w in walls],
                "rounds": res.total_rounds, "J": res.final_objective, "termination": res.termination,
                "gpu_s_per_round": wall / res.total_rounds}
        if args.cpu_rounds > 0:
            from oracle import oracle as orc

            p = make(kind, M, d, "cpu")
            t = time.perf_counter()
            _, J1, rounds, _ = orc.solve_generic(p, orc.OracleConfig(max_rounds=args.cpu_rounds))
            cpu = time.perf_counter() - t
            g1 = P.solve(prob, P.SolverConfig(max_rounds=args.cpu_rounds))
            line.update(cpu_s_per_round=cpu / len(rounds), cpu_cores=orc.num_threads(),
                        cpu_solve_s_extrapolated=cpu / len(rounds) * res.total_rounds,
                        parity_first_rounds=bool(g1.final_objective == J1))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
