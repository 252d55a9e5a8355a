"""Config 5 on the device: ZeroDelay and Inventory (M = 1, 2, 3) vs the
reference's goldens, and the uniform-noise kernels vs the oracle, bitwise."""
import numpy as np
import pytest
import torch

from parity_util import assert_bitwise
from test_oracle_config5 import FIXTURES, oracle_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available()
    return P


def device_problem(P, g):
    specs = [tuple(float(v) if k < 2 else int(v) for k, v in enumerate(row)) for row in g["specs"]]
    if "pw" in g:
        prob = P.ZeroDelay(power_weight=float(g["pw"]), grids=specs)
        prob._override_host_constants(g["f0"], g["fw0"])
        return prob
    return P.Inventory(stages=int(g["stages"]), stage_cost=str(g["stage_cost"]),
                       order_cost=float(g["order_cost"]) if "order_cost" in g else 0.1, grids=specs)


def _U(P, prob, us):
    return P.ControllerSet(tuple(P.SampledController(g, u) for g, u in zip(prob.grids, us)))


@pytest.mark.parametrize("tag", FIXTURES)
def test_config5_device_vs_golden(P, golden, tag):
    g = golden(tag)
    prob = device_problem(P, g)
    cfg = P.SolverConfig()
    for name in ("ident", "pert0", "pert1"):
        U = _U(P, prob, [g[f"{name}_u{m}"] for m in range(prob.M)])
        assert_bitwise(prob.objective(U), g[f"{name}_J"], f"{name} J")
        for m in range(prob.M):
            pts = prob.grids[m].points
            assert_bitwise(prob.marginal_cost_batch(m, U.values(m), pts, U), g[f"{name}_c{m}"], f"{name} C{m}")
            assert_bitwise(P.local_update_phase(prob, m, U, cfg), g[f"{name}_lu{m}"], f"{name} LU{m}")
            assert_bitwise(P.partial_exhaustion_phase(prob, m, U, cfg), g[f"{name}_ex{m}"], f"{name} EX{m}")
        V = P.run_block(prob, U, cfg, 1, "local")
        V = P.run_block(prob, V, cfg, 1, "exhaustion")
        for m in range(prob.M):
            assert_bitwise(V.values(m), g[f"{name}_it_u{m}"], f"{name} it u{m}")
        assert_bitwise(prob.objective(V), g[f"{name}_it_J"], f"{name} it J")
    if "solve_J" in g:
        res = P.solve(prob, cfg)
        assert res.termination == str(g["solve_termination"])
        assert_bitwise(np.array([r.objective for r in res.rounds]), g["solve_rounds"][:, 1], "per-round J")
        assert_bitwise(res.final_objective, g["solve_J"], "J")
        for m in range(prob.M):
            assert_bitwise(res.controllers.values(m), g[f"solve_u{m}"], f"u{m}")


def test_inventory_forward_density_vs_oracle(P, golden, oracle_mod):
    g = golden("inv_m3")
    prob = device_problem(P, g)
    p = oracle_problem(oracle_mod, g)
    us = [g[f"pert1_u{m}"] for m in range(3)]
    U = _U(P, prob, us)
    for m in range(3):
        assert_bitwise(prob.forward_density(m, U), p.forward_density(m, us), f"f_{m}")


@pytest.mark.parametrize("seed", [0, 1])
def test_uniform_kernels_vs_oracle(P, oracle_mod, seed):
    from paper_1908_04489_b200 import _lib, config5
    from paper_1908_04489_b200._device import ptr, stream_ptr

    config5._bind()
    rng = np.random.default_rng(seed)
    a, b, d = -4.0, 3.5, 257 + seed * 100
    h = (b - a) / (d - 1)
    v = rng.normal(0, 2, d)
    x = np.concatenate([rng.uniform(a - 3, b + 3, 999), [a, b, a - 1.0, b + 1.0, 0.5 * (a + b)]])
    dev = torch.device("cuda", 0)
    keep = []  # device copies must outlive the (asynchronous) calls that read them

    def T(z):
        t = torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64)).to(dev)
        keep.append(t)
        return t

    s = stream_ptr(dev)
    for rad in (1.0, 0.37):
        outs = [torch.empty(x.size, dtype=torch.float64, device=dev) for _ in range(3)]
        _lib.call("ucp_unif_moments_grid", ptr(T(x)), x.size, ptr(T(v)), a, h, d, rad, *(ptr(o) for o in outs), s)
        want = oracle_mod.unif_moments_grid(x, v, a, h, d, rad)
        for k in range(3):
            assert_bitwise(outs[k].cpu().numpy(), want[k], f"unif_moments_grid s{k}")
        out = torch.empty(x.size, dtype=torch.float64, device=dev)
        _lib.call("ucp_unif_ball_sum", ptr(T(x)), x.size, ptr(T(v)), a, h, d, rad, ptr(out), s)
        assert_bitwise(out.cpu().numpy(), oracle_mod.unif_ball_sum(x, v, a, h, d, rad), "ball_sum")
        masses = np.abs(rng.normal(0, 1, x.size))
        out = torch.empty(d, dtype=torch.float64, device=dev)
        _lib.call("ucp_unif_propagate", ptr(T(masses)), ptr(T(x)), x.size, a, h, d, rad, ptr(out), s)
        assert_bitwise(out.cpu().numpy(), oracle_mod.unif_propagate(masses, x, a, h, d, rad), "propagate")
        w, vals = np.abs(rng.normal(0, 1, x.size)), rng.normal(0, 3, x.size)
        q = rng.uniform(a - 1, b + 1, 500)
        outs = [torch.empty(q.size, dtype=torch.float64, device=dev) for _ in range(3)]
        _lib.call("ucp_unif_moments_points", ptr(T(q)), q.size, ptr(T(x)), ptr(T(w)), ptr(T(vals)), x.size, a, h, d,
                  rad, *(ptr(o) for o in outs), s)
        want = oracle_mod.unif_moments_points(q, x, w, vals, a, h, d, rad)
        for k in range(3):
            assert_bitwise(outs[k].cpu().numpy(), want[k], f"unif_moments_points m{k}")


def test_inventory_reuse_across_calls_is_result_identical(P):
    """Densities / costs-to-go reused across calls (content keys) give the
    bits of the no-reuse path, in any call order, and an in-place change of a
    controller tensor (version bump) is never served from the cache."""
    rng = np.random.default_rng(7)
    M, d = 5, 97
    specs = [(-3.0, 3.0, d)] * M
    keyed, plain = P.Inventory(stages=M, grids=specs), P.Inventory(stages=M, grids=specs)
    plain.reuse = False
    pts = keyed.grids[0].points
    sets = [[np.maximum(0.0, 0.5 - 0.3 * pts + 0.2 * rng.uniform(-1, 1, d)) for _ in range(M)] for _ in range(3)]
    cfg = P.SolverConfig()
    # the keyed side reuses its controller objects (stable keys: cache hits)
    ctrl = [[P.SampledController(keyed.grids[k], sets[s][k]) for k in range(M)] for s in range(3)]
    from paper_1908_04489_b200 import _lib

    launches = [0, 0]
    for step in range(24):
        pick = [int(rng.integers(3)) for _ in range(M)]  # stages drawn from different sets
        us = [sets[pick[k]][k] for k in range(M)]
        m = int(rng.integers(M))
        Uk = P.ControllerSet(tuple(ctrl[pick[k]][k] for k in range(M)))
        Up = _U(P, plain, us)
        n0 = _lib.launch_count()
        a = P.local_update_phase(keyed, m, Uk, cfg)
        n1 = _lib.launch_count()
        b = P.local_update_phase(plain, m, Up, cfg)
        launches[0] += n1 - n0
        launches[1] += _lib.launch_count() - n1
        assert_bitwise(a, b, f"LU{m} {step}")
        assert_bitwise(keyed.forward_density(m, Uk), plain.forward_density(m, Up), f"f{m} {step}")
        if step % 4 == 0:
            assert_bitwise(P.partial_exhaustion_phase(keyed, m, Uk, cfg),
                           P.partial_exhaustion_phase(plain, m, Up, cfg), f"EX{m} {step}")
    assert launches[0] < launches[1], launches  # reuse happened
    # in-place change of stage 0's device values after they were cached
    us = sets[0]
    Uk = P.ControllerSet(tuple(ctrl[0]))
    P.local_update_phase(keyed, M - 1, Uk, cfg)
    t = Uk.device_values(0, torch.device("cuda"))
    t.add_(0.125)
    changed = [us[0] + 0.125] + list(us[1:])
    for m in (M - 1, 1):
        assert_bitwise(P.local_update_phase(keyed, m, Uk, cfg),
                       P.local_update_phase(plain, m, _U(P, plain, changed), cfg), f"LU{m} after in-place change")


@pytest.mark.parametrize("n", [0, 1, 31, 33, 255, 257, 1000])
def test_uniform_source_compaction_edges(P, oracle_mod, n):
    """k_unif_propagate / k_unif_moments_points skip sources out of a warp's
    reach: source counts around the 32-lane and 256-source batch boundaries,
    clustered / far-away / infinite / NaN centres, bitwise vs the oracle."""
    from paper_1908_04489_b200 import _lib, config5
    from paper_1908_04489_b200._device import ptr, stream_ptr

    config5._bind()
    rng = np.random.default_rng(n)
    a, b, d = -2.0, 2.0, 301
    h = (b - a) / (d - 1)
    x = np.concatenate([rng.uniform(-0.1, 0.1, n // 2), rng.uniform(a - 6, b + 6, n - n // 2)])
    rng.shuffle(x)
    if n >= 31:
        x[3], x[7], x[11], x[30] = np.inf, -np.inf, np.nan, 50.0
    masses = np.abs(rng.normal(0, 1, n))
    w, vals = np.abs(rng.normal(0, 1, n)), rng.normal(0, 3, n)
    q = np.concatenate([np.linspace(a - 0.5, b + 0.5, 77), [a, b, a - 3.0, b + 3.0]])
    dev = torch.device("cuda", 0)
    keep = []

    def T(z):
        t = torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64)).to(dev)
        keep.append(t)
        return t

    s = stream_ptr(dev)
    for rad in (1.0, 0.05):
        out = torch.empty(d, dtype=torch.float64, device=dev)
        _lib.call("ucp_unif_propagate", ptr(T(masses)), ptr(T(x)), n, a, h, d, rad, ptr(out), s)
        assert_bitwise(out.cpu().numpy(), oracle_mod.unif_propagate(masses, x, a, h, d, rad), f"propagate n={n}")
        outs = [torch.empty(q.size, dtype=torch.float64, device=dev) for _ in range(3)]
        _lib.call("ucp_unif_moments_points", ptr(T(q)), q.size, ptr(T(x)), ptr(T(w)), ptr(T(vals)), n, a, h, d,
                  rad, *(ptr(o) for o in outs), s)
        want = oracle_mod.unif_moments_points(q, x, w, vals, a, h, d, rad)
        for k in range(3):
            assert_bitwise(outs[k].cpu().numpy(), want[k], f"unif_moments_points m{k} n={n}")
