"""bench.py keeps the driver's JSON contract (a small, fast configuration):
one line, every required key, consistent units, the reference arm too."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(*args):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=str(ROOT), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "1", "--warmup", "3", "--log2d", "12", "--cpu-seconds", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["unit"] == "evals/s" and d["value"] > 0 and d["dtype"] == "f64" and d["data"] == "synthetic"
    assert "workload" in d["config"]
    r = d["roofline"]
    assert set(("bound", "achieved", "peak", "unit", "frac", "traffic")) <= set(r) and 0 < r["frac"] <= 1.0
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] > 0 and c["unit"] == d["unit"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["gpu_launches"] > 0
    assert d["time_to_converge"]["J"] == 0.16692114286407383  # C1, bitwise the reference


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--log2d", "12", "--cpu-seconds", "1")
    assert d["impl"] == "reference" and d["unit"] == "evals/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["value"] == d["value"]


def _run_torchrun(world, *args):
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
                        "--gpus", str(world), *args], cwd=str(ROOT), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_line_contract_two_ranks():
    """The driver's N>1 launch (torchrun, one rank per GPU) on a one-GPU box: gloo, both
    ranks on cuda:0 — plumbing only (barriers, max-over-ranks timing, one JSON line)."""
    d = _run_torchrun(2, "--steps", "1", "--warmup", "3", "--log2d", "12", "--no-cpu-baseline",
                      "--backend", "gloo", "--same-device")
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["time_to_converge"]["J"] == 0.16692114286407383  # sharded C1 solve, bitwise the reference



def test_bench_two_ranks_balanced_plans_with_parity():
    """2 ranks at 2^15 points (above UCP_BALANCE_MIN_POINTS: work-balanced,
    uneven shards and the uneven all-gather) with the N>1 parity check and
    the fast-arithmetic field: every sampled point of every phase bitwise the
    oracle's, on the path the driver's multi-GPU run takes."""
    d = _run_torchrun(2, "--steps", "1", "--warmup", "3", "--log2d", "15", "--cpu-seconds", "2",
                      "--backend", "gloo", "--same-device")
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["cpu_baseline"] is None  # the CPU baseline is an N=1 figure
    par = d["parity"]
    assert all(par[k] == 0 for k in ("local0", "local1", "exh0", "exh1", "objective", "J_from_terms")), par
    assert min(par["points"].values()) >= 16
    for arith in ("fma", "table"):
        f = d["fast_mode"][arith]
        assert f["value"] > 0 and f["J_rel_diff_vs_reference_arithmetic"] < 1e-12 and f["points_differing"]["exh1"] == 0
