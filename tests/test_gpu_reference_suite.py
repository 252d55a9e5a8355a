"""The reference's own unit tests for the hot path (pkg/tests/test_solver.py,
test_problems.py, test_problem_core.py), restated against the device package
with the same inputs and assertions.  Tests of the out-of-scope Quadratic toy
problem and of non-device plugin problems (FlatCost, Poisoned) are omitted."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available()
    return P


def small_witsenhausen(P):  # conftest.py:8-9
    return P.Witsenhausen(grids=[(-25.0, 25.0, 201), (-25.0, 25.0, 201)])


def small_zero_delay(P):
    return P.ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)])


def small_inventory(P):
    return P.Inventory(grids=[(-3.0, 3.0, 241)] * 2)


def perturbed_controllers(P, problem, seed=0, scale=0.5):  # conftest.py:37-44
    rng = np.random.default_rng(seed)
    return P.ControllerSet(tuple(P.SampledController(g, problem.project(m, g.points + scale * rng.uniform(-1.0, 1.0, g.d)))
                                 for m, g in enumerate(problem.grids)))


# ---------------------------------------------------------- test_solver.py
def test_witsenhausen_closed_form_interior(P):  # test_solver.py:135-145
    wc = small_witsenhausen(P)
    new = P.local_update_phase(wc, 0, wc.zero_controllers(), P.SolverConfig(newton_cap=1e9))
    g = wc.grids[0]
    interior = np.abs(g.points) <= 12.0
    want = -g.points / (1.0 + wc.k ** 2)
    assert np.max(np.abs(new[interior] - want[interior])) <= 5e-3


def test_inventory_projection(P):  # :147-152
    inv = small_inventory(P)
    assert P.local_update_phase(inv, 0, inv.zero_controllers(), P.SolverConfig()).min() >= 0.0


def test_never_raises_pointwise_cost(P):  # :154-162
    wc = small_witsenhausen(P)
    U = perturbed_controllers(P, wc, seed=21)
    g = wc.grids[0]
    before = wc.marginal_cost_batch(0, U.values(0), g.points, U)
    new = P.local_update_phase(wc, 0, U, P.SolverConfig())
    after = wc.marginal_cost_batch(0, new, g.points, U)
    assert np.all(after <= before)


def test_constant_controller_unchanged(P):  # :165-171
    wc = small_witsenhausen(P)
    U = wc.zero_controllers()
    vals = np.full(wc.grids[1].d, 0.75)
    U = U.replace(1, U[1].with_values(vals))
    assert np.array_equal(P.partial_exhaustion_phase(wc, 1, U, P.SolverConfig()), vals)


def test_degenerate_window_unchanged(P):  # :173-178
    wc = small_witsenhausen(P)
    U = perturbed_controllers(P, wc, seed=22)
    cfg = P.SolverConfig(search_radius=wc.grids[0].spacing / 4.0)
    assert np.array_equal(P.partial_exhaustion_phase(wc, 0, U, cfg), U.values(0))


def test_matches_windowed_oracle(P):  # :180-189
    wc = small_witsenhausen(P)
    U = wc.zero_controllers()
    U = U.replace(1, U[1].with_values(np.sin(wc.grids[1].points) * 3.0))
    cfg = P.SolverConfig()
    new = P.partial_exhaustion_phase(wc, 1, U, cfg)
    g = wc.grids[1]
    r = cfg.radius_for(g)
    for i in range(0, g.d, 17):
        assert new[i] == P.windowed_argmin(wc, 1, float(g.points[i]), U, r)


def test_never_increases_objective(P):  # :191-200
    for problem in (small_witsenhausen(P), small_inventory(P)):
        U = perturbed_controllers(P, problem, seed=23)
        J = problem.objective(U)
        for m in range(problem.M):
            new = P.partial_exhaustion_phase(problem, m, U, P.SolverConfig())
            U = U.replace(m, U[m].with_values(new))
            J2 = problem.objective(U)
            assert J2 <= J + 1e-9 * (1 + abs(J))
            J = J2


def test_round_report_invariants(P):  # :213-221
    res = P.solve(small_witsenhausen(P), P.SolverConfig(workers=1, max_rounds=6))
    for r in res.rounds:
        assert r.local_iters + r.exhaustion_iters == 20
        assert 1 <= r.local_iters <= 19
        assert r.local_gain >= 0 and r.exhaustion_gain >= 0
    assert res.rounds[0].local_iters == 10


def test_fixed_split_schedule(P):  # :223-227
    res = P.solve(small_witsenhausen(P), P.SolverConfig(workers=1, max_rounds=3, fixed_local_iters=19))
    assert res.termination == "max_rounds"
    assert all(r.local_iters == 19 and r.exhaustion_iters == 1 for r in res.rounds)


def test_worker_count_does_not_change_results(P):  # :229-234
    a = P.solve(small_witsenhausen(P), P.SolverConfig(workers=1, max_rounds=3))
    b = P.solve(small_witsenhausen(P), P.SolverConfig(workers=2, max_rounds=3))
    for m in range(2):
        assert np.array_equal(a.controllers.values(m), b.controllers.values(m))
    assert a.final_objective == b.final_objective


def test_monotone_exhaustion_blocks(P):  # :236-239
    res = P.solve(small_witsenhausen(P), P.SolverConfig(workers=1, max_rounds=8))
    for r in res.rounds:
        assert r.objective <= r.objective_after_local + 1e-9 * (1 + abs(r.objective))


def test_initial_controllers_validated(P):  # :255-259
    wc = small_witsenhausen(P)
    other = small_zero_delay(P).identity_controllers()
    with pytest.raises(ValueError):
        P.solve(wc, P.SolverConfig(workers=1), initial=other)


def test_infeasible_initial_is_projected(P):  # :261-265
    inv = small_inventory(P)
    res = P.solve(inv, P.SolverConfig(workers=1, max_rounds=2))
    for m in range(inv.stages):
        assert res.controllers.values(m).min() >= 0.0


# -------------------------------------------------------- test_problems.py
def test_objective_zero_controllers(P):  # test_problems.py:37-39
    wc = small_witsenhausen(P)
    assert wc.objective(wc.zero_controllers()) == pytest.approx(25.0, abs=0.01)


def test_objective_cancelling_first_stage(P):  # :41-45
    wc = small_witsenhausen(P)
    U = wc.zero_controllers()
    U = U.replace(0, U[0].with_values(-wc.grids[0].points))
    assert wc.objective(U) == pytest.approx(1.0, abs=0.01)


def test_stage0_argmin_closed_form(P):  # :47-53
    wc = small_witsenhausen(P)
    got = P.exhaustive_argmin(wc, 0, 5.0, wc.zero_controllers(), P.OracleConfig(-10.0, 0.0, 20001))
    assert got == pytest.approx(-5.0 / 1.04, abs=3e-3)


def test_stage1_argmin_symmetric(P):  # :55-60
    wc = small_witsenhausen(P)
    got = P.exhaustive_argmin(wc, 1, 0.0, wc.zero_controllers(), P.OracleConfig(-5.0, 5.0, 20001))
    assert got == 0.0


def test_pinned_stage1_cost(P):  # :62-72 (PINNED["wc_stage1_cost"], production tolerance)
    wc = P.Witsenhausen()
    got = wc.marginal_cost(1, 0.5, 1.0, wc.zero_controllers())
    assert got == pytest.approx(0.09014577594859935, rel=1e-9)


def test_zero_delay_objective_zero_controllers(P):  # :82-84
    zd = small_zero_delay(P)
    assert zd.objective(zd.zero_controllers()) == pytest.approx(1.0, abs=0.01)


# ---------------------------------------------------- test_problem_core.py
def test_default_objective_matches_stage0_quadrature(P):  # test_problem_core.py:165-174
    wc = small_witsenhausen(P)
    U = perturbed_controllers(P, wc, seed=10)
    g = wc.grids[0]
    costs = wc.marginal_cost_batch(0, U.values(0), g.points, U)
    wts = np.full(g.d, g.spacing)
    wts[0] *= 0.5
    wts[-1] *= 0.5
    assert wc.objective(U) == pytest.approx(float(costs @ wts), rel=1e-12)


def test_batch_matches_scalar_fd(P):  # :129-142
    wc = small_witsenhausen(P)
    U = perturbed_controllers(P, wc, seed=9)
    g = wc.grids[0]
    idx = [10, 50, 120]
    u = U.values(0)[idx]
    y = g.points[idx]
    h = 1e-4 * (1.0 + np.abs(u))
    c1, c2 = wc.derivatives_batch(0, u, y, U, h)
    for t in range(len(idx)):
        want1 = wc.marginal_cost_d1(0, float(u[t]), float(y[t]), U, float(h[t]))
        want2 = wc.marginal_cost_d2(0, float(u[t]), float(y[t]), U, float(h[t]))
        assert c1[t] == pytest.approx(want1, rel=1e-12, abs=1e-15)
        assert c2[t] == pytest.approx(want2, rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("name", ["witsenhausen", "zero_delay"])
def test_odd_controllers_give_even_cost(P, name):  # :179-196
    problem = small_witsenhausen(P) if name == "witsenhausen" else small_zero_delay(P)
    U = problem.identity_controllers()
    for m, g in enumerate(problem.grids):
        vals = np.tanh(g.points) * (1.5 + 0.5 * np.sin(g.points))
        odd = 0.5 * (vals - vals[::-1])
        U = U.replace(m, U[m].with_values(odd))
    rng = np.random.default_rng(12)
    for m in range(problem.M):
        for _ in range(6):
            y = float(rng.uniform(-3, 3))
            u = float(rng.uniform(-2, 2))
            lhs = problem.marginal_cost(m, u, y, U)
            rhs = problem.marginal_cost(m, -u, -y, U)
            assert lhs == pytest.approx(rhs, rel=1e-9, abs=1e-15)


def test_check_controllers(P):  # :115-127
    for problem in (small_witsenhausen(P), small_zero_delay(P), small_inventory(P)):
        problem.check_controllers(problem.identity_controllers())
        wrong = P.ControllerSet(tuple(P.SampledController(P.make_grid(-1, 1, 7), np.zeros(7))
                                      for _ in range(problem.M)))
        with pytest.raises(ValueError):
            problem.check_controllers(wrong)


@pytest.mark.parametrize("name", ["witsenhausen", "zero_delay", "inventory"])
def test_batched_windowed_rule_matches_every_swept_point(P, name):
    """verify.windowed_argmin_many re-derives the partial-exhaustion rule at
    EVERY grid point in one batched device evaluation (oracle.py:70-95's rule,
    independent of the sweep kernels' candidate lists and argmin): equal to
    the device sweep everywhere, and to the one-point form."""
    prob = {"witsenhausen": P.Witsenhausen(grids=[(-25.0, 25.0, 301)] * 2),
            "zero_delay": P.ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)]),
            "inventory": P.Inventory(grids=[(-3.0, 3.0, 241)] * 2)}[name]
    rng = np.random.default_rng(3)
    U = P.ControllerSet(tuple(P.SampledController(g, prob.project(m, np.round(g.points + rng.uniform(-1, 1, g.d), 1)))
                              for m, g in enumerate(prob.grids)))
    cfg = P.SolverConfig()
    for m, g in enumerate(prob.grids):
        swept = P.partial_exhaustion_phase(prob, m, U, cfg)
        best = P.windowed_argmin_many(prob, m, g.points, U, cfg.radius_for(g))
        np.testing.assert_array_equal(prob.project(m, best), swept)
        i = g.d // 3
        assert P.windowed_argmin(prob, m, float(g.points[i]), U, cfg.radius_for(g)) == best[i]


def test_batched_exhaustive_argmin(P):
    wc = P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
    U = wc.zero_controllers()
    oc = P.OracleConfig(-10.0, 10.0, 2001)
    ys = [-5.0, 0.0, 5.0, 12.5]
    many = P.exhaustive_argmin_many(wc, 0, ys, U, oc)
    assert [P.exhaustive_argmin(wc, 0, y, U, oc) for y in ys] == many.tolist()
