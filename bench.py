#!/usr/bin/env python
"""Benchmark: marginal-cost evaluations/s of the Witsenhausen hot path at 2^20.

Workload (BASELINE.json configs[1]): Witsenhausen k=0.2, sigma=5 on two
2^20-point grids over [-25, 25], FP64.  Controllers: the converged
default-grid (d=2000) solution, linearly interpolated onto the fine grid
(deterministic; every value distinct, like controllers after a local sweep).
SolverConfig(search_radius=19.5 h): 39-node exhaustion windows.

One *step* = every hot-path phase once on that controller snapshot:
    local_update(m=0), local_update(m=1), exhaustion(m=0), exhaustion(m=1), J.
Every step reads the same snapshot, so all steps do identical work.  ``value`` counts the marginal-cost evaluations the REFERENCE performs
for that step (5 per point per stage for a local sweep, one per distinct
window candidate for an exhaustion sweep, one per point for J) divided by
the device time; both arms use this same count, so their ratio is a pure
time ratio.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun): points of every stage are sharded across ranks and the new
controller is all-gathered over NCCL after each phase (strong scaling on the
fixed 2^20 grid); device time is the max over ranks.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "marginal-cost evals/sec & time-to-converge (s), Witsenhausen k=0.2 σ=5, 1/2/4/8 GPU"
K_WC, SIGMA = 0.2, 5.0
SPAN = (-25.0, 25.0)
C1_D = 2000
C1_SOLVES = 7
PAPER_SOLVES = 3
C4_SWEEPS = 3
FAST_STEPS = 2
DP_OPS_PER_NODE = 8  # kernels.py:430-439: 3 mul + 3 add accumulate, 2 mul recurrence
# kernels.py:466-482 per in-cutoff pair: sub, 2 compares, 2 mul (-0.5*diff*diff), exp (12 DP
# instructions in the device port of glibc's __exp_fma: 8 FMA + 1 sub + 1 add + 2 mul),
# *factor, *INV, != 0, *w, 3 add, 2 mul (wp*x, (wp*x)*x) = 26; out of the cutoff: sub +
# compares = 3
DP_OPS_PER_PAIR = 26
DP_OPS_PER_PAIR_OUT = 3
# FP64-pipe instructions k_moments executes per in-cutoff pair (ncu
# sm__sass_thread_inst_executed_op_fp64_pred_on.sum = 6.634e11 over 2.875e10 in-cutoff pairs at 2^18,
# profiles/r2_fp64_inst_2p18.csv)
DP_INST_PER_PAIR_EXEC = 23.07


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--log2d", type=int, default=20)
    ap.add_argument("--window-nodes", type=int, default=39)
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target CPU seconds of the cpu_baseline sample (ours) / per step (reference)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fast", action="store_true", help="skip the supplementary fast-arithmetic step")
    ap.add_argument("--backend", default="nccl", help="process-group backend for N>1 (gloo: plumbing tests only)")
    ap.add_argument("--same-device", action="store_true",
                    help="all ranks on cuda:0 (multi-rank plumbing test on a one-GPU box, gloo only)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def grid_points(d):
    return np.linspace(SPAN[0], SPAN[1], d), (SPAN[1] - SPAN[0]) / (d - 1)


def resample(u_coarse, d):
    """Linear interpolation of a d=2000 controller onto the fine grid."""
    y, _ = grid_points(d)
    yc, _ = grid_points(u_coarse.size)
    return np.ascontiguousarray(np.interp(y, yc, u_coarse))


def walk_nodes(s, a, h, d):
    """Visited nodes of the stage-0 walk at centres s (kernels.py:416-421)."""
    jlo = np.maximum(np.ceil(((s - 12.0) - a) / h), 0)
    jhi = np.minimum(np.floor(((s + 12.0) - a) / h), d - 1)
    return np.maximum(jhi - jlo + 1, 0)


def window_candidates(u, lo, hi):
    """Distinct-by-run candidates per window (== the reference's dedup count for staircases)."""
    flags = np.concatenate([[0], (u[1:] != u[:-1]).astype(np.int64)])
    pref = np.cumsum(flags)
    return 1 + pref[hi] - pref[lo]


def window_bounds(d, r):
    y, h = grid_points(d)
    lo = np.ceil((y - r - SPAN[0]) / h - 1e-9).astype(np.int64)
    hi = np.floor((y + r - SPAN[0]) / h + 1e-9).astype(np.int64)
    ic = np.clip(np.ceil((y - SPAN[0]) / h - 0.5).astype(np.int64), 0, d - 1)
    return np.maximum(0, np.minimum(lo, ic)), np.minimum(d - 1, np.maximum(hi, ic))


def exhaustion_nodes(u0, y, lo, hi, h, d):
    """Visited walk nodes of all exhaustion candidates (run-start dedup, as the kernels)."""
    total = 0.0
    flags = np.concatenate([[True], u0[1:] != u0[:-1]])
    for k in range(int((hi - lo).max()) + 1):
        j = lo + k
        ok = j <= hi
        jj = np.minimum(j, d - 1)
        first = ok & ((k == 0) | flags[jj])
        total += float(walk_nodes(y[first] + u0[jj[first]], SPAN[0], h, d).sum())
    return total


def moments_pairs(x1, yq):
    """In-range (|y - x| <= 12) support pairs of the stage-1 moments."""
    xs = np.sort(x1)
    return float((np.searchsorted(xs, yq + 12.0, side="right") - np.searchsorted(xs, yq - 12.0)).sum())


def workload_counts(u0, u1, d, r, fd_step=1e-4):
    """Reference evaluation count per step and algorithmic work of the kernels."""
    y, h = grid_points(d)
    lo, hi = window_bounds(d, r)
    cand0_pp = window_candidates(u0, lo, hi)
    cand1_pp = window_candidates(u1, lo, hi)
    cand0, cand1 = int(cand0_pp.sum()), int(cand1_pp.sum())
    evals = 5 * d + 5 * d + cand0 + cand1 + d
    hh = fd_step * (1.0 + np.abs(u0))
    s = y + u0
    nodes = (walk_nodes(s + hh, SPAN[0], h, d) + 2 * walk_nodes(s, SPAN[0], h, d) + walk_nodes(s - hh, SPAN[0], h, d))
    ex_nodes = exhaustion_nodes(u0, y, lo, hi, h, d)
    pairs = moments_pairs(y + u0, y)
    return {"evals": evals, "cand0": cand0, "cand1": cand1, "cand0_pp": cand0_pp, "cand1_pp": cand1_pp,
            "lu0_nodes": float(nodes.sum()),
            "lu0_dp_ops": float(nodes.sum()) * DP_OPS_PER_NODE, "ex0_nodes": ex_nodes,
            "ex0_dp_ops": ex_nodes * DP_OPS_PER_NODE, "moment_pairs": pairs,
            "moment_dp_ops": pairs * DP_OPS_PER_PAIR}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [ln.split(",") for ln in Path(self.f.name).read_text().splitlines() if ln.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for k, name in enumerate(names):
                if len(r) > 5 + k and "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------ CPU (oracle) timing
def cpu_sample_step(orc, p, u0, u1, d, r, counts, target_s, seed=0):
    """One bounded sample of the step on the CPU: the reference's algorithm (the
    oracle port, all host threads) on random points of every phase (both grid
    ends included), each phase's sample sized to about target_s / 5 seconds
    so per-call overheads stay negligible.  Each phase's time is scaled by
    d / n to the full step (the per-point work is independent, so the scaling
    is unbiased; tools/cpu_extrapolation_check.py measured -1.5% against a
    full CPU step at 2^16).  Returns the measured seconds, the extrapolated
    full-step seconds and rate (the reference's evaluations of the full step
    over them), per-phase seconds and every phase's outputs (parity check)."""
    cfg = orc.OracleConfig(search_radius=r)
    thr = orc.num_threads()
    W = float(np.mean(walk_nodes(grid_points(d)[0] + u0, SPAN[0], p.h1, d)))
    node_rate, pair_rate = 4.0e8 * thr, 1.5e8 * thr  # rough per-thread rates to size samples
    per = target_s / 5.0
    cpp = counts["cand0"] / d
    sizes = {"local0": int(np.clip(per * node_rate / (5 * W), 16, d)),
             "local1": int(np.clip(per * pair_rate / (5 * d), 4, d)),
             "exh0": int(np.clip(per * node_rate / (cpp * W), 16, d)),
             "exh1": int(np.clip(per * pair_rate / d, 4, d)),
             "objective": int(np.clip(per * node_rate / W, 16, d))}
    rng = np.random.default_rng(seed)
    phases = (("local0", lambda i: orc.local_update_phase(p, 0, u0, u1, cfg, points=i)),
              ("local1", lambda i: orc.local_update_phase(p, 1, u0, u1, cfg, points=i)),
              ("exh0", lambda i: orc.partial_exhaustion_phase(p, 0, u0, u1, cfg, points=i)),
              ("exh1", lambda i: orc.partial_exhaustion_phase(p, 1, u0, u1, cfg, points=i)),
              ("objective", lambda i: p.cost_batch(0, u0[i], i, u0, u1)))
    times, full, outs = {}, {}, {}
    for name, fn in phases:
        idx = rng.choice(d, max(sizes[name] - 2, 1), replace=False).astype(np.int64)
        idx = np.unique(np.concatenate([idx, [0, d - 1]]))  # the grid ends: every phase's edge cases
        t = time.perf_counter()
        outs[name] = (idx, fn(idx))
        times[name] = time.perf_counter() - t
        full[name] = times[name] * d / idx.size
    step_s = sum(full.values())
    return {"seconds": sum(times.values()), "rate": counts["evals"] / step_s, "step_s_extrapolated": step_s,
            "phase_s": full, "outs": outs, "threads": thr,
            "sample": ("random points per phase, both grid ends included: "
                       + ", ".join(f"{k}={v[0].size}" for k, v in outs.items())
                       + f" of {d}; each phase's time scaled x d/n to the full step")}


def parity_vs_oracle(outs, gpu, J, orc, h):
    """Bitwise mismatches of the GPU step against the oracle's outputs on the
    sampled points (the cpu_baseline leg's own results): the four phases, the
    objective integrand, and J re-summed from the device integrand by the
    oracle's serial trapezoid (kernels.py:136-144)."""
    par = {}
    for name, (idx, want) in outs.items():
        got = gpu[name][idx]
        par[name] = int(np.count_nonzero(got.view(np.uint64) != np.ascontiguousarray(want, np.float64).view(np.uint64)))
    par["J_from_terms"] = int(np.float64(orc.trapezoid_sum(gpu["objective"], h)).view(np.uint64)
                              != np.float64(J).view(np.uint64))
    par["points"] = {name: int(idx.size) for name, (idx, _) in outs.items()}
    par["what"] = ("bitwise mismatches, GPU step vs the oracle (reference-order C restatement, pinned to the "
                   "reference's goldens) on the cpu_baseline sample points, grid ends included")
    return par


def c1_oracle_solve(orc):
    p = orc.OracleWitsenhausen(k=K_WC, sigma=SIGMA, grid0=(*SPAN, C1_D), grid1=(*SPAN, C1_D))
    t = time.perf_counter()
    u0, u1, J, rounds, term = orc.solve(p)
    return u0, u1, {"wall_s": time.perf_counter() - t, "rounds": len(rounds), "J": J, "termination": term}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc

    orc.build()
    orc.set_threads(os.cpu_count() or 1)  # torchrun exports OMP_NUM_THREADS=1; use every host core
    d = 1 << args.log2d
    u0c, u1c, c1 = c1_oracle_solve(orc)
    u0, u1 = resample(u0c, d), resample(u1c, d)
    p = orc.OracleWitsenhausen(k=K_WC, sigma=SIGMA, grid0=(*SPAN, d), grid1=(*SPAN, d))
    r = (args.window_nodes / 2.0) * p.h0
    counts = workload_counts(u0, u1, d, r)
    per_step = max(args.cpu_seconds, 2.0)
    for w in range(args.warmup):
        cpu_sample_step(orc, p, u0, u1, d, r, counts, per_step / 4, seed=1000 + w)
    samples = [cpu_sample_step(orc, p, u0, u1, d, r, counts, per_step, seed=k) for k in range(args.steps)]
    sec = float(np.mean([q["seconds"] for q in samples]))  # measured: one bounded sample per step
    value = counts["evals"] / float(np.mean([q["step_s_extrapolated"] for q in samples]))
    last = samples[-1]
    host = orc.host_cpu_description()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, d, counts),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": last["threads"], "kind": "port",
                         "sample": last["sample"], "host": host, "phase_s": last["phase_s"],
                         "step_s_extrapolated": float(np.mean([q["step_s_extrapolated"] for q in samples]))},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step": "one bounded sample of the step per step (cpu_baseline.sample; ms_per_step is its measured "
                "time); value = the full step's reference evaluations / the sample's per-phase times scaled "
                "x d/n (cpu_baseline.step_s_extrapolated)",
        "time_to_converge": {"config": f"d={C1_D} default SolverConfig, identity init", **c1},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, d, counts):
    return {"workload": f"witsenhausen k={K_WC} sigma={SIGMA} grids 2x{d} on [-25,25], controllers = "
                        f"d=2000 solution linearly interpolated, search_radius={args.window_nodes / 2}h; step = every "
                        "phase once on that snapshot: local(m=0,1) + exhaustion(m=0,1) + objective",
            "grid_points": d, "window_nodes": args.window_nodes,
            "evals_per_step": counts["evals"], "exhaustion_candidates": [counts["cand0"], counts["cand1"]],
            "l2": "inputs re-read each step; L2 flushed between steps (256 MiB memset inside timed region)"}


# ------------------------------------------------------------ our B200 arm
PHASES = (("local0", "local", 0), ("local1", "local", 1), ("exh0", "exhaustion", 0), ("exh1", "exhaustion", 1))


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if args.backend == "nccl":
            # communicator init lines (ranks, NVLS/P2P transport) in the log, so every rank is checkable
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.backend)
    import paper_1908_04489_b200 as P
    from paper_1908_04489_b200 import _lib
    from paper_1908_04489_b200._device import ptr

    sh = P.from_process_group() if world > 1 else P.LOCAL
    d = 1 << args.log2d

    # time-to-converge at the default grid (C1) on the GPU(s); it also gives the snapshot.
    # One round on a throw-away problem first (lazy module loading and the first launch
    # of every kernel are one-time process costs), then C1_SOLVES solves, each of a fresh
    # problem (new device context, graph captures included) as a user would run them:
    # median, min and max reported.  At N>1 the small solves run as replicas on every rank
    # (a d=2000 phase is latency-bound: sharding it only adds collectives).
    warm = P.Witsenhausen(k=K_WC, sigma=SIGMA)
    P.solve(warm, P.SolverConfig(max_rounds=1))
    del warm  # its workspace goes to the pool every later problem draws from

    def timed_solves(make, n):
        walls, res = [], None
        for _ in range(n):
            pr = make()
            pr.objective(pr.identity_controllers())  # context creation (allocations) outside the clock
            gc.collect()  # no collector pass (or context teardown) inside a timed region
            torch.cuda.synchronize()
            t = time.perf_counter()
            res = P.solve(pr, P.SolverConfig())
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t)
            del pr
        return res, {"wall_s": float(np.median(walls)), "wall_s_min": min(walls), "wall_s_max": max(walls),
                     "solves": n, "walls_s": [round(w, 5) for w in walls]}

    res, c1w = timed_solves(lambda: P.Witsenhausen(k=K_WC, sigma=SIGMA), C1_SOLVES)
    c1 = {"config": f"d={C1_D} default SolverConfig, identity init; median of {C1_SOLVES} solves of fresh "
                    "problems" + (" (replica on every rank)" if world > 1 else ""), **c1w,
          "rounds": res.total_rounds, "J": res.final_objective, "termination": res.termination}
    u0h, u1h = resample(res.controllers.values(0), d), resample(res.controllers.values(1), d)
    # the paper's grid size (d=14000): the reference needs 1,437 s on 8 cores
    rp, pw = timed_solves(lambda: P.Witsenhausen(k=K_WC, sigma=SIGMA, grids=[(*SPAN, 14000), (*SPAN, 14000)]),
                          PAPER_SOLVES)
    paper = {"config": f"d=14000 (paper size) default SolverConfig, identity init; median of {PAPER_SOLVES} "
                       "solves" + (" (replica on every rank)" if world > 1 else ""), **pw,
             "rounds": rp.total_rounds, "J": rp.final_objective,
             "termination": rp.termination, "reference_cpu_s": 1437.4,
             "reference_cpu": "numba reference, 8-core Xeon (SURVEY.md Appendix B)"}
    del rp
    # config 4: 64 independent instances (k in [0.05, 1], sigma in {3, 5, 7}) at d=2000 to
    # convergence -- the batched engine (one kernel over (instance, point) per step);
    # instances k % world per rank ("replicas only")
    sweep = [(0.05 + 0.95 * i / 63, (3.0, 5.0, 7.0)[i % 3]) for i in range(64)]
    # first launches of the batched kernels and the engine for this shape (a
    # reusable resource, cached per shape like a workspace)
    P.solve_many([P.Witsenhausen(k=k, sigma=s_) for k, s_ in sweep], P.SolverConfig(max_rounds=1), sharding=sh)
    swalls = []
    for _ in range(C4_SWEEPS):
        sprobs = [P.Witsenhausen(k=k, sigma=s_) for k, s_ in sweep]
        gc.collect()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        sres = P.solve_many(sprobs, P.SolverConfig(), sharding=sh)
        torch.cuda.synchronize()
        sw = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(sw, op=dist.ReduceOp.MAX)
        swalls.append(float(sw.item()))
    swall = float(np.median(swalls))
    config4 = {"config": "64 Witsenhausen instances, k = 0.05 + 0.95 i/63, sigma = (3, 5, 7)[i % 3], d=2000, "
                         f"default SolverConfig, to convergence; instances k % world per rank; median of "
                         f"{C4_SWEEPS} sweeps (max over ranks each)",
               "wall_s": swall, "wall_s_min": min(swalls), "wall_s_max": max(swalls),
               "solves_per_s": 64 / swall, "engine": "batched (csrc/ucp_batch.cuh)",
               "rounds_max": max(r.total_rounds for r in sres if r is not None),
               "reference_cpu_s_per_instance": 7.5,
               "reference_cpu": "oracle port on 16 cores, profiles/r1_sweep_c4.json"}
    del sprobs, sres

    prob = P.Witsenhausen(k=K_WC, sigma=SIGMA, grids=[(*SPAN, d), (*SPAN, d)])
    h = prob.grids[0].spacing
    cfg = P.SolverConfig(search_radius=(args.window_nodes / 2.0) * h)
    U0 = P.ControllerSet(tuple(P.SampledController(prob.grids[m], torch.from_numpy(u).to(dev))
                               for m, u in ((0, u0h), (1, u1h))))
    counts = workload_counts(u0h, u1h, d, cfg.radius_for(prob.grids[0]))
    begin, end = sh.bounds(d)
    frac_rank = (end - begin) / d

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]

    def step(U, evs=None):
        flush.zero_()
        if evs:
            evs[0].record(stream)
        outs = []
        for k, (_, kind, m) in enumerate(PHASES):
            sweep = prob.device_local_update if kind == "local" else prob.device_exhaustion
            outs.append(sweep(m, U, cfg, sh))
            if evs:
                evs[k + 1].record(stream)
        J = prob.device_objective(U, sh)
        if evs:
            evs[5].record(stream)
        return outs, J

    # FP64 pipe peak of this GPU (DMUL/DADD, no FMA) -- the roofline denominator
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.empty(sms * 8 * 256, dtype=torch.float64, device=dev)
    iters = 4096
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        if rep == 2:
            e0.record(stream)
        _lib.call("ucp_fp64_probe", sms * 8, 256, iters, ptr(sink), stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    fp64_peak = sms * 8 * 256 * iters * 16 / (e0.elapsed_time(e1) * 1e-3)

    for _ in range(args.warmup):
        step(U0)
    gc.collect()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = _lib.launch_count()
    for k in range(args.steps):
        step(U0, ev[k])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count() - n_launch0
    clk = clocks.stop()
    ms = ev[0][0].elapsed_time(ev[-1][5])
    phase_ms = np.array([[e[q].elapsed_time(e[q + 1]) for q in range(5)] for e in ev]).mean(axis=0)
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_step = float(tmax.item()) / args.steps

    # end to end through the public API: host controllers in, every phase's
    # new host controller + J out, each step
    e2e = None
    if not args.no_e2e:
        hu = [torch.from_numpy(u0h).pin_memory(), torch.from_numpy(u1h).pin_memory()]
        ho = [torch.empty(d, dtype=torch.float64).pin_memory() for _ in PHASES]

        def e2e_step():
            flush.zero_()
            U = P.ControllerSet(tuple(P.SampledController(prob.grids[m], hu[m].to(dev, non_blocking=True))
                                      for m in (0, 1)))
            outs, J = step(U)
            for o, hbuf in zip(outs, ho):
                hbuf.copy_(o, non_blocking=True)
            stream.synchronize()
            return J

        e2e_step()
        e2e_steps = max(1, min(args.steps, 2))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        t1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item()) / e2e_steps
        e2e = {"value": counts["evals"] / (e2e_ms * 1e-3), "unit": "evals/s", "ms_per_step": e2e_ms,
               "steps": e2e_steps, "h2d_bytes_per_step": 2 * d * 8,
               "d2h_bytes_per_step": len(PHASES) * d * 8 + 16,
               "path": "public API: SampledController from pinned host arrays -> 4 device sweeps + objective "
                       "-> new controllers copied back to pinned host buffers, J to host"}

    # executed walk nodes: the no-op tail exit (csrc walk_tail_noop) visits fewer nodes than
    # the reference's windows, so the roofline counts what the kernels actually walked --
    # one untimed, instrumented pass of the two stage-0 phases on this rank's shard
    ctr = torch.zeros(1, dtype=torch.int64, device=dev)
    visited = {}
    for key, kind in (("lu0", "local"), ("ex0", "exhaustion")):
        ctr.zero_()
        torch.cuda.synchronize()
        _lib.call("ucp_walk_node_counter", ptr(ctr))
        try:
            (prob.device_local_update if kind == "local" else prob.device_exhaustion)(0, U0, cfg, sh)
            torch.cuda.synchronize()
        finally:
            _lib.call("ucp_walk_node_counter", None)
        visited[key] = float(ctr.item())
        if visited[key] == 0:  # latency-mode walks (small grids) are not instrumented: full windows
            visited[key] = counts[f"{key}_nodes"] * frac_rank

    # the opt-in fast arithmetics (Witsenhausen(arithmetic=...), NOT bitwise --
    # tolerance stated in DESIGN.md §2b and tests/test_gpu_fast_mode.py) on the
    # same snapshot: supplementary figures, never the headline
    fast = None
    fast_outs = {}
    if not args.no_fast:
        fast = {}
        for arith in ("fma", "table"):
            fprob = P.Witsenhausen(k=K_WC, sigma=SIGMA, grids=[(*SPAN, d), (*SPAN, d)], arithmetic=arith)
            FU = P.ControllerSet(tuple(P.SampledController(fprob.grids[m], U0[m]._dev, _trusted_device=True)
                                       for m in (0, 1)))

            def fstep():
                outs = [(fprob.device_local_update if kind == "local" else fprob.device_exhaustion)(m, FU, cfg, sh)
                        for _, kind, m in PHASES]
                return outs, fprob.device_objective(FU, sh)

            fstep()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            f0_, f1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0_.record(stream)
            for _ in range(FAST_STEPS):
                flush.zero_()
                fouts, fJ = fstep()
            f1_.record(stream)
            torch.cuda.synchronize()
            tf = torch.tensor([f0_.elapsed_time(f1_) / FAST_STEPS], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(tf, op=dist.ReduceOp.MAX)
            fast[arith] = {"value": counts["evals"] / (float(tf.item()) * 1e-3), "unit": "evals/s",
                           "ms_per_step": float(tf.item()), "steps": FAST_STEPS, "J": fJ}
            fast_outs[arith] = [o.cpu().numpy() for o in fouts]
            del fprob, FU, fouts
        fast["what"] = ("opt-in arithmetic, NOT bitwise (tolerance stated in DESIGN.md §2b and "
                        "tests/test_gpu_fast_mode.py): 'fma' = FMA walk; 'table' = stage-0 window sums from per-cell "
                        "Taylor expansions (objective included; the reference walk's rounding bias reproduced) + "
                        "per-tile Taylor-expansion stage-1 moments, grids with h1 <= 2e-3")

    # the step's outputs on the host (one untimed step on the same snapshot): the
    # parity check against the oracle's results on the cpu_baseline sample points
    outs_dev, J_dev = step(U0)
    gpu_out = {name: o.cpu().numpy() for (name, _, _), o in zip(PHASES, outs_dev)}
    for arith, fo_list in fast_outs.items():
        fast[arith]["J_rel_diff_vs_reference_arithmetic"] = abs(fast[arith].pop("J") - J_dev) / abs(J_dev)
        fast[arith]["points_differing"] = {name: int(np.count_nonzero(gpu_out[name] != fo))
                                           for (name, _, _), fo in zip(PHASES, fo_list)}
    gpu_out["objective"] = prob.device_objective_terms(U0, sh).cpu().numpy()

    # roofline: every kernel family, and the dominant one.  Two work counts per
    # family (this rank's share): "algorithmic" = SURVEY.md §8(d)'s per-unit figure
    # over the reference's full windows / all pairs; "executed" = what the kernels
    # actually ran (walk nodes counted on the device: the no-op tail exit skips the
    # rest; moment pairs inside the cutoff, FP64 instructions per pair from ncu).
    # Two denominators: the nominal FP64 issue rate SMs x 64 x the SM clock sampled
    # during the timed region (§8(d)), and the DMUL/DADD probe measured above.
    clk_mhz = clk.get("sm_mhz") or 1965.0
    p_nominal = sms * 64 * clk_mhz * 1e6
    mom_pairs = counts["moment_pairs"] * frac_rank
    mom_all = float(d) * float(d) * frac_rank
    kernels = {
        "exh0": ("k_ex0_eval (stage-0 exhaustion candidates)", phase_ms[2],
                 counts["ex0_nodes"] * frac_rank * DP_OPS_PER_NODE, visited["ex0"] * DP_OPS_PER_NODE),
        "local0": ("k_lu0_probe + k_lu0_finish (stage-0 local update)", phase_ms[0],
                   counts["lu0_nodes"] * frac_rank * DP_OPS_PER_NODE, visited["lu0"] * DP_OPS_PER_NODE),
        "local1": ("k_moments (u1 estimator) + k_lu1", phase_ms[1],
                   mom_pairs * DP_OPS_PER_PAIR + (mom_all - mom_pairs) * DP_OPS_PER_PAIR_OUT,
                   mom_pairs * DP_INST_PER_PAIR_EXEC),
    }
    fam = {}
    for k, (kname, ms_k, alg, exe) in kernels.items():
        s_k = ms_k * 1e-3
        fam[k] = {"kernel": kname, "ms": ms_k, "ops_algorithmic": alg, "ops_executed": exe,
                  "tflops_algorithmic": alg / s_k / 1e12, "tflops_executed": exe / s_k / 1e12,
                  "frac_algorithmic": alg / s_k / p_nominal, "frac_executed": exe / s_k / p_nominal,
                  "frac_algorithmic_probe": alg / s_k / fp64_peak, "frac_executed_probe": exe / s_k / fp64_peak}
    top = max(kernels, key=lambda k: kernels[k][1])
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"dram_bytes_per_launch_2p{args.log2d}", {}).get(top)
        except Exception:
            traffic = None
    roofline = {"bound": "fp64", "kernel": kernels[top][0], "achieved": fam[top]["tflops_algorithmic"],
                "peak": p_nominal / 1e12, "unit": "TFLOP/s", "frac": fam[top]["frac_algorithmic"],
                "frac_executed": fam[top]["frac_executed"],
                "frac_algorithmic_probe": fam[top]["frac_algorithmic_probe"],
                "frac_executed_probe": fam[top]["frac_executed_probe"], "traffic": traffic,
                "peak_source": f"nominal FP64 issue rate {sms} SMs x 64 DP lanes x {clk_mhz:.0f} MHz (median SM "
                               f"clock sampled during the timed region; SURVEY.md §8(d)); probe = ucp_fp64_probe "
                               f"DMUL+DADD throughput measured on this GPU at bench start: "
                               f"{fp64_peak / 1e12:.3f} T instr/s",
                "work": f"achieved/frac = algorithmic work (SURVEY.md §8(d)): {DP_OPS_PER_NODE} DP ops per node of "
                        f"the reference's full clamped walk windows ({counts['ex0_nodes']:.4g} nodes in exh0, "
                        f"{counts['lu0_nodes']:.4g} in local0); frac_executed counts the nodes the kernels walked "
                        f"(device counter: {visited['ex0']:.4g} / {visited['lu0']:.4g} on this rank; the no-op tail "
                        f"exit skips the rest, result-invariant). Moments: {DP_OPS_PER_PAIR} DP ops per in-cutoff "
                        f"pair + {DP_OPS_PER_PAIR_OUT} per out-of-cutoff pair algorithmic, {DP_INST_PER_PAIR_EXEC} "
                        f"FP64 instructions per in-cutoff pair executed (ncu, profiles/README.md); exp/erf/setup "
                        f"outside the loops excluded",
                "walk_nodes": {"executed": visited, "reference": {"ex0": counts["ex0_nodes"] * frac_rank,
                                                                   "lu0": counts["lu0_nodes"] * frac_rank}},
                "families": fam}

    if rank == 0:
        value = counts["evals"] / (ms_step * 1e-3)
        cpu, parity = None, None
        if not args.no_cpu_baseline and world == 1:
            from oracle import oracle as orc

            orc.build()
            orc.set_threads(os.cpu_count() or 1)
            p = orc.OracleWitsenhausen(k=K_WC, sigma=SIGMA, grid0=(*SPAN, d), grid1=(*SPAN, d),
                                       f0=prob._f0, fw0=prob._fw0)
            q = cpu_sample_step(orc, p, u0h, u1h, d, cfg.radius_for(prob.grids[0]), counts, args.cpu_seconds)
            cpu = {"value": q["rate"], "unit": "evals/s", "cores": q["threads"], "kind": "port",
                   "sample": q["sample"], "sample_s": q["seconds"], "step_s_extrapolated": q["step_s_extrapolated"],
                   "phase_s": q["phase_s"], "host": orc.host_cpu_description()}
            parity = parity_vs_oracle(q["outs"], gpu_out, J_dev, orc, prob.grids[0].spacing)
        elif not args.no_cpu_baseline:
            # N>1: the same check on a smaller sample (parity only; the CPU baseline is an N=1 figure)
            from oracle import oracle as orc

            orc.build()
            orc.set_threads(os.cpu_count() or 1)
            p = orc.OracleWitsenhausen(k=K_WC, sigma=SIGMA, grid0=(*SPAN, d), grid1=(*SPAN, d),
                                       f0=prob._f0, fw0=prob._fw0)
            q = cpu_sample_step(orc, p, u0h, u1h, d, cfg.radius_for(prob.grids[0]), counts,
                                min(args.cpu_seconds, 3.0))
            parity = parity_vs_oracle(q["outs"], gpu_out, J_dev, orc, prob.grids[0].spacing)
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(args, d, counts),
            "roofline": roofline, "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "clocks": clk, "gpu_launches": launches,
            "phase_ms": dict(zip(["local0", "local1", "exh0", "exh1", "objective"], phase_ms.round(3).tolist())),
            "time_to_converge": c1, "time_to_converge_paper_size": paper, "config4_sweep": config4,
            "fast_mode": fast, "gpu": torch.cuda.get_device_name(dev),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
