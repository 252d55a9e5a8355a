"""CUDA path vs the reference (golden vectors) and vs the oracle, bitwise.

Bar (BASELINE.json north_star): argmin choices / controller values bit-exact
in reference order, J within 1e-9 relative -- these tests demand bitwise
equality for everything, J included.
"""
import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

from parity_util import assert_bitwise

pytestmark = pytest.mark.gpu

NATIVE = Path(__file__).resolve().parent / "native"


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def _wc(P, g, d=None):
    d = int(g["d"]) if d is None else d
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, d), (-25.0, 25.0, d)])
    prob._override_host_constants(g["f0"], g["fw0"])
    return prob


def _U(P, prob, u0, u1):
    return P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))


# ------------------------------------------------------------------ libm port
@pytest.fixture(scope="module")
def host_libm():
    subprocess.run(["make", "-s", "-C", str(NATIVE)], check=True)
    L = ctypes.CDLL(str(NATIVE / "_build" / "liblibm_port_check.so"))
    for f in ("host_exp", "host_erf"):
        getattr(L, f).restype = ctypes.c_double
        getattr(L, f).argtypes = [ctypes.c_double]
    return L


@pytest.mark.parametrize("which,lo,hi", [("exp", -75.0, 1.0), ("exp", -1e-3, 1e-3), ("exp", -745.0, 709.0),
                                         ("erf", -9.0, 9.0), ("erf", -1.3, 1.3)])
def test_device_libm(P, host_libm, which, lo, hi):
    rng = np.random.default_rng(7)
    x = rng.uniform(lo, hi, 200_000)
    x[:4] = [lo, hi, 0.0, -0.0]
    got = P.kernels.device_libm(which, x)
    f = host_libm.host_exp if which == "exp" else host_libm.host_erf
    want = np.array([f(float(v)) for v in x])
    assert_bitwise(got, want, f"device {which}")


def test_device_phi_cdf(P, oracle_mod):
    z = np.concatenate([np.random.default_rng(3).uniform(-13, 13, 20_000), [-12.0, 12.0, -11.999, 0.0]])
    want = np.array([oracle_mod.phi_cdf(v) for v in z])
    assert_bitwise(P.kernels.device_libm("phi_cdf", z), want, "phi_cdf")


# -------------------------------------------------------- kernels.py surface
@pytest.mark.parametrize("tag", ["k307", "k2", "k64"])
def test_kernels_vs_golden(P, golden, tag):
    g = golden("kernels")
    a, h, d = g[f"{tag}_a"], g[f"{tag}_h"], int(g[f"{tag}_d"])
    t = P.kernels.gauss_moments_grid(g[f"{tag}_centers"], g[f"{tag}_vals"], a, h, d)
    for k in range(3):
        assert_bitwise(t[k], g[f"{tag}_grid_t{k}"], f"{tag} T{k}")
    p = P.kernels.gauss_moments_points(g[f"{tag}_queries"], g[f"{tag}_xs"], g[f"{tag}_weights"], a, h, d)
    for k in range(3):
        assert_bitwise(p[k], g[f"{tag}_pts_{k}"], f"{tag} M{k}")


def test_small_kernels_vs_golden(P, golden):
    g = golden("kernels")
    assert_bitwise(P.kernels.trapezoid_sum(g["trap_samples"], 0.37), g["trap_value"], "trapezoid")
    np.testing.assert_array_equal(P.kernels.segmented_argmin(g["argmin_costs"], g["argmin_offsets"]),
                                  g["argmin_out"])


# ----------------------------------------------------- Witsenhausen phases
@pytest.mark.parametrize("tag", ["d201", "d2000"])
@pytest.mark.parametrize("name", ["ident", "pert0", "pert1"])
def test_phases_vs_golden(P, golden, tag, name):
    g = golden(f"wc_{tag}")
    prob = _wc(P, g)
    cfg = P.SolverConfig()
    U = _U(P, prob, g[f"{name}_u0"], g[f"{name}_u1"])
    assert_bitwise(prob.objective(U), g[f"{name}_J"], "J")
    for m in (0, 1):
        pts = prob.grids[m].points
        u = U.values(m)
        assert_bitwise(prob.marginal_cost_batch(m, u, pts, U), g[f"{name}_c{m}"], f"C{m}")
        assert_bitwise(prob.marginal_cost_batch(m, u + 0.37, pts, U), g[f"{name}_c{m}_up"], f"C{m}+")
        assert_bitwise(P.local_update_phase(prob, m, U, cfg), g[f"{name}_lu{m}"], f"LU{m}")
        assert_bitwise(P.partial_exhaustion_phase(prob, m, U, cfg), g[f"{name}_ex{m}"], f"EX{m}")
        small = P.SolverConfig(search_radius=3.5 * prob.grids[m].spacing)
        assert_bitwise(P.partial_exhaustion_phase(prob, m, U, small), g[f"{name}_exs{m}"], f"EXs{m}")
    V = P.run_block(prob, U, cfg, 1, "local")
    V = P.run_block(prob, V, cfg, 1, "exhaustion")
    assert_bitwise(V.values(0), g[f"{name}_it_u0"], "it u0")
    assert_bitwise(V.values(1), g[f"{name}_it_u1"], "it u1")
    assert_bitwise(prob.objective(V), g[f"{name}_it_J"], "it J")


@pytest.mark.parametrize("tag", ["d201", "d2000"])
def test_segmented_vs_golden(P, golden, tag):
    g = golden(f"wc_{tag}")
    prob = _wc(P, g)
    U = _U(P, prob, g["pert0_u0"], g["pert0_u1"])
    for m in (0, 1):
        y = prob.grids[m].points[g["seg_idx"]]
        got = prob.marginal_cost_segmented(m, g["seg_u"], g["seg_offsets"], y, U)
        assert_bitwise(got, g[f"seg_c{m}"], f"seg C{m}")


@pytest.mark.parametrize("tag", ["d201", "d2000"])
def test_full_solve_vs_golden(P, golden, tag):
    g = golden(f"wc_solve_{tag}")
    prob = _wc(P, g)
    res = P.solve(prob, P.SolverConfig())
    assert res.termination == str(g["termination"])
    got = np.array([[r.round_index, r.objective, r.local_gain, r.exhaustion_gain, r.local_iters,
                     r.exhaustion_iters, r.objective_after_local] for r in res.rounds])
    assert got.shape == g["rounds"].shape
    assert_bitwise(got[:, 1], g["rounds"][:, 1], "per-round J")
    assert_bitwise(got[:, 6], g["rounds"][:, 6], "J after local")
    np.testing.assert_array_equal(got[:, 4:6], g["rounds"][:, 4:6])
    assert_bitwise(res.final_objective, g["final_J"], "final J")
    assert_bitwise(res.controllers.values(0), g["u0"], "u0")
    assert_bitwise(res.controllers.values(1), g["u1"], "u1")


# ------------------------------------------------------------ fine grid 2^20
@pytest.fixture(scope="module")
def fine(golden, oracle_mod):
    f = golden("wc_fine_2p20")
    sol = golden("wc_solve_d2000")
    d = int(f["d"])
    y, h = oracle_mod.linspace_grid(-25.0, 25.0, d)
    _, ch = oracle_mod.linspace_grid(-25.0, 25.0, 2000)
    near = np.clip(np.ceil((y - (-25.0)) / ch - 0.5).astype(np.int64), 0, 1999)
    return dict(f=f, d=d, y=y, h=h, u0=sol["u0"][near], u1=sol["u1"][near])


def test_fine_stage0_walks_vs_golden(P, fine):
    f = fine["f"]
    t = P.kernels.gauss_moments_grid(f["s"], fine["u1"], -25.0, fine["h"], fine["d"])
    for k in range(3):
        assert_bitwise(t[k], f[f"t{k}"], f"T{k} (W=503,316)")


def test_fine_stage1_moments_vs_oracle(P, fine, oracle_mod):
    p = oracle_mod.OracleWitsenhausen(grid0=(-25.0, 25.0, fine["d"]), grid1=(-25.0, 25.0, fine["d"]))
    q = fine["f"]["q_idx"]
    x1 = fine["y"] + fine["u0"]
    want = oracle_mod.gauss_moments_points(fine["y"][q], x1, p.fw0, -25.0, fine["h"], fine["d"])
    got = P.kernels.gauss_moments_points(fine["y"][q], x1, p.fw0, -25.0, fine["h"], fine["d"])
    for k in range(3):
        assert_bitwise(got[k], want[k], f"M{k}")


def test_fine_local_update_sample_vs_oracle(P, fine, oracle_mod):
    """A full 2^20 stage-0 local-update sweep on device, checked on 64 sampled points."""
    d = fine["d"]
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
    U = _U(P, prob, fine["u0"], fine["u1"])
    cfg = P.SolverConfig()
    new0 = P.local_update_phase(prob, 0, U, cfg)
    p = oracle_mod.OracleWitsenhausen(grid0=(-25.0, 25.0, d), grid1=(-25.0, 25.0, d), f0=prob._f0,
                                      fw0=prob._fw0)
    pts = np.sort(np.random.default_rng(2).choice(d, 64, replace=False))
    pts[0], pts[-1] = 0, d - 1
    want = oracle_mod.local_update_phase(p, 0, fine["u0"], fine["u1"], oracle_mod.OracleConfig(), points=pts)
    assert_bitwise(new0[pts], want, "LU0 @2^20")


# ------------------------------------------------- randomized vs the oracle
@pytest.mark.parametrize("seed,d0,d1", [(0, 333, 517), (1, 1024, 97), (2, 64, 64)])
def test_random_grids_vs_oracle(P, oracle_mod, seed, d0, d1):
    rng = np.random.default_rng(seed)
    g0, g1 = (-7.0 - seed, 9.0, d0), (-11.0, 6.5 + seed, d1)
    prob = P.Witsenhausen(k=0.3 + 0.1 * seed, sigma=2.0 + seed, grids=[g0, g1])
    p = oracle_mod.OracleWitsenhausen(k=prob.k, sigma=prob.sigma, grid0=g0, grid1=g1, f0=prob._f0,
                                      fw0=prob._fw0)
    u0 = np.round(prob.grids[0].points + rng.uniform(-2, 2, d0), 1)  # repeats -> dedup paths
    u1 = prob.grids[1].points * rng.uniform(0.5, 1.5) + rng.normal(0, 0.3, d1)
    U = _U(P, prob, u0, u1)
    ocfg, cfg = oracle_mod.OracleConfig(search_radius=0.9), P.SolverConfig(search_radius=0.9)
    assert_bitwise(prob.objective(U), oracle_mod.objective(p, u0, u1), "J")
    for m in (0, 1):
        assert_bitwise(P.local_update_phase(prob, m, U, cfg),
                       oracle_mod.local_update_phase(p, m, u0, u1, ocfg), f"LU{m}")
        assert_bitwise(P.partial_exhaustion_phase(prob, m, U, cfg),
                       oracle_mod.partial_exhaustion_phase(p, m, u0, u1, ocfg), f"EX{m}")


# ------------------------------------------------------------- error paths
def test_nonfinite_raises_like_reference(P, oracle_mod, golden):
    g = golden("wc_d201")
    prob = _wc(P, g)
    p = oracle_mod.OracleWitsenhausen(grid0=(-25.0, 25.0, 201), grid1=(-25.0, 25.0, 201), f0=g["f0"],
                                      fw0=g["fw0"])
    u0, u1 = g["pert0_u0"].copy(), g["pert0_u1"].copy()
    u1[150] = 1e200  # (s - u1)^2 overflows -> inf/NaN costs around it
    U = _U(P, prob, u0, u1)
    cfg = P.SolverConfig()
    for fn_dev, fn_orc in ((P.local_update_phase, oracle_mod.local_update_phase),
                           (P.partial_exhaustion_phase, oracle_mod.partial_exhaustion_phase)):
        with pytest.raises(P.NumericError) as e_dev:
            fn_dev(prob, 0, U, cfg)
        with pytest.raises(oracle_mod.OracleNumericError) as e_orc:
            fn_orc(p, 0, u0, u1, oracle_mod.OracleConfig())
        assert str(e_dev.value) == str(e_orc.value)
    with pytest.raises(P.NumericError) as e_dev:
        prob.objective(U)
    with pytest.raises(oracle_mod.OracleNumericError) as e_orc:
        oracle_mod.objective(p, u0, u1)
    assert str(e_dev.value) == str(e_orc.value)


def test_no_cpu_fallback_and_launches(P):
    from paper_1908_04489_b200 import _lib

    n0 = _lib.launch_count()
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, 101)] * 2)
    prob.objective(prob.identity_controllers())
    assert _lib.launch_count() > n0
    assert _lib.LIB_PATH.exists()


@pytest.mark.parametrize("nq,m", [(8000, 4096), (8704, 257), (10_000, 4096), (9000, 257), (20_000, 4096),
                                  (17_000, 257), (3, 5000)])
def test_moments_direct_path_vs_oracle(P, oracle_mod, nq, m):
    """Both moments kernels on unsorted queries: up to 8,704 queries (the
    default UCP_FUSED_MAX_QUERIES) the fused producer/consumer kernel, above
    it the persistent tiled kernel (tile skipping, edge blocks, work queue);
    bitwise vs the oracle."""
    rng = np.random.default_rng(nq)
    a, b = -20.0, 20.0
    h = (b - a) / (m - 1)
    x = np.sort(rng.uniform(-35, 35, m)) + rng.normal(0, 0.5, m)  # mostly increasing, some disorder
    x[::97] = x[::97][::-1]
    w = np.abs(rng.normal(0, 1, m)) * h
    y = np.concatenate([[a, b, a - 1.0, b + 1.0], rng.uniform(a - 2, b + 2, max(nq - 4, 0))])[:nq]
    got = P.kernels.gauss_moments_points(y, x, w, a, h, m)
    want = oracle_mod.gauss_moments_points(y, x, w, a, h, m)
    for k in range(3):
        assert_bitwise(got[k], want[k], f"M{k}")


def test_solve_many_matches_individual_solves(P):
    """Concurrent instances (streams + threads) give each instance's solo result bitwise."""
    pars = [(0.2, 5.0), (0.5, 3.0), (0.9, 7.0), (0.05, 5.0), (0.3, 3.0)]
    grids = [(-25.0, 25.0, 301)] * 2
    cfg = P.SolverConfig(max_rounds=4)
    many = P.solve_many([P.Witsenhausen(k=k, sigma=s, grids=grids) for k, s in pars], cfg, concurrency=3)
    for (k, s), r in zip(pars, many):
        solo = P.solve(P.Witsenhausen(k=k, sigma=s, grids=grids), cfg)
        assert r.final_objective == solo.final_objective
        assert [x.objective for x in r.rounds] == [x.objective for x in solo.rounds]
        np.testing.assert_array_equal(np.asarray(r.controllers.values(0)), np.asarray(solo.controllers.values(0)))


def test_exhaustion_sync_and_syncfree_paths_agree(P, golden, monkeypatch):
    """ucp_wc_exhaustion with a host candidate bound (no stream sync) and
    without one (count read back) give the reference's result."""
    from paper_1908_04489_b200.device_problem import DeviceContext

    g = golden("wc_d201")
    cfg = P.SolverConfig()
    for bound_off in (False, True):
        prob = _wc(P, g)
        if bound_off:
            monkeypatch.setattr(DeviceContext, "candidate_bound", lambda *a, **k: 0)
        U = _U(P, prob, g["pert1_u0"], g["pert1_u1"])
        assert_bitwise(P.partial_exhaustion_phase(prob, 0, U, cfg), g["pert1_ex0"], f"EX0 bound_off={bound_off}")
        V = P.run_block(prob, U, cfg, 1, "local")
        V = P.run_block(prob, V, cfg, 1, "exhaustion")
        assert_bitwise(V.values(0), g["pert1_it_u0"], "it u0")


@pytest.mark.parametrize("kind", ["local", "exhaustion"])
def test_graph_replayed_blocks_bitwise_and_errors(P, golden, kind):
    """Blocks replayed from CUDA graphs give the eager result bit for bit, and a
    failure inside one raises exactly the eager (reference) error."""
    g = golden("wc_d201")
    prob = _wc(P, g)
    cfg = P.SolverConfig()
    U = _U(P, prob, g["pert1_u0"], g["pert1_u1"])
    a = prob.device_run_block(kind, 4, U, cfg, graphs=True)
    b = prob.device_run_block(kind, 4, U, cfg, graphs=False)
    a2 = prob.device_run_block(kind, 3, a, cfg, graphs=True)  # graph reuse with new inputs
    b2 = prob.device_run_block(kind, 3, b, cfg, graphs=False)
    for m in (0, 1):
        assert_bitwise(a2.values(m), b2.values(m), f"{kind} u{m}")
    prob.flush_errors()
    u1 = g["pert0_u1"].copy()
    u1[150] = 1e200
    bad = _U(P, prob, g["pert0_u0"], u1)
    msgs = []
    for graphs in (True, False):
        prob.device_run_block(kind, 3, bad, cfg, graphs=graphs)
        with pytest.raises(P.NumericError) as e:
            prob.flush_errors()
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


@pytest.mark.gpu
def test_concurrent_graph_capture_with_workspace_churn():
    """solve_many: graph captures in some host threads while others grow or
    destroy workspaces (device-synchronising calls) -- results stay bitwise
    the sequential solves'."""
    import gc

    import paper_1908_04489_b200 as P

    cfg = P.SolverConfig(max_rounds=4)
    specs = [(0.05 + 0.1 * i, (3.0, 5.0, 7.0)[i % 3], 301 + 97 * (i % 5)) for i in range(24)]
    probs = [P.Witsenhausen(k=k, sigma=s, grids=[(-25.0, 25.0, d)] * 2) for k, s, d in specs]
    got = P.solve_many(probs, cfg, concurrency=12)
    del probs
    gc.collect()
    for (k, s, d), r in zip(specs, got):
        ref = P.solve(P.Witsenhausen(k=k, sigma=s, grids=[(-25.0, 25.0, d)] * 2), cfg)
        assert r.final_objective == ref.final_objective
        for m in range(2):
            assert np.array_equal(np.asarray(r.controllers.values(m)), np.asarray(ref.controllers.values(m)))


@pytest.mark.parametrize("nq,m,special", [(100, 1, None), (64, 2, None), (300, 300, "nan"), (300, 513, "dup"),
                                          (20_000, 300, "nan")])
def test_moments_edge_inputs_vs_oracle(P, oracle_mod, nq, m, special):
    """Tiny support sets, a NaN support point (its tile is never skipped and
    NaN reaches every query that sees the tails or the pdf), duplicated
    support points -- fused and persistent kernels, bitwise vs the oracle."""
    rng = np.random.default_rng(m + nq)
    a, b = -10.0, 10.0
    d = 401
    h = (b - a) / (d - 1)
    x = rng.uniform(-30, 30, m)
    if special == "nan":
        x[m // 3] = np.nan
    if special == "dup":
        x[1::2] = x[0::2][: x[1::2].size]
    w = np.abs(rng.normal(0, 1, m)) * h
    y = np.concatenate([[a, b], rng.uniform(a - 3, b + 3, nq - 2)])
    got = P.kernels.gauss_moments_points(y, x, w, a, h, d)
    want = oracle_mod.gauss_moments_points(y, x, w, a, h, d)
    for k in range(3):
        assert_bitwise(got[k], want[k], f"M{k}")


def test_deferred_objective_value_and_error_order(P):
    """The post-local objective is queued without a synchronisation: its value
    is bitwise the synchronous one, and a failure is raised (with the
    reference's message) before anything queued after it."""
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
    g0, g1 = prob.grids
    rng = np.random.default_rng(5)
    U = P.ControllerSet((P.SampledController(g0, g0.points + rng.uniform(-1, 1, g0.d)),
                         P.SampledController(g1, g1.points)))
    V = prob.identity_controllers()
    want = prob.device_objective(U)
    h = prob.device_objective_deferred(U)
    other = prob.device_objective(V, deferred=[h])
    assert h[1] == [want] and other == prob.device_objective(V)
    bad = P.ControllerSet((P.SampledController(g0, np.full(g0.d, 1e200)), P.SampledController(g1, g1.points)))
    with pytest.raises(P.NumericError) as sync_err:
        prob.device_objective(bad)
    h = prob.device_objective_deferred(bad)
    with pytest.raises(P.NumericError) as got:
        prob.device_objective(V, deferred=[h])
    assert str(got.value) == str(sync_err.value)


def test_nccl_comm_single_rank(P):
    """The library's NCCL communicator (ucp_comm_*) on one rank: the equal and
    uneven in-place all-gathers and the MIN all-reduce leave the data as is,
    bad arguments are rejected, and a solve sharded over the communicator is
    bitwise the unsharded one (multi-rank runs need one GPU per rank)."""
    uid = P.NcclComm.unique_id()
    comm = P.NcclComm(1, 0, uid)
    x = torch.arange(10, dtype=torch.float64, device="cuda")
    comm.allgather_(x)
    comm.allgatherv_(x, (0, 10))
    e = torch.tensor([5, 3, 9], dtype=torch.int64, device="cuda")
    comm.allreduce_min_(e)
    torch.cuda.synchronize()
    assert x.cpu().tolist() == list(map(float, range(10))) and e.cpu().tolist() == [5, 3, 9]
    with pytest.raises(ValueError):
        comm.allgatherv_(x, (4, 2))
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
    got = P.solve(prob, P.SolverConfig(max_rounds=3), sharding=comm.sharding())
    want = P.solve(P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2), P.SolverConfig(max_rounds=3))
    assert got.final_objective == want.final_objective
    comm.close()
    with pytest.raises(ValueError):
        P.NcclComm(2, 5, uid)
