"""Batched multi-instance engine (config 4): every
instance's result is bitwise its single-instance solve's (controllers, J,
round reports), across schedules that diverge between instances."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available()
    return P


def _same(P, a, b):
    assert a.termination == b.termination
    assert np.float64(a.final_objective).view(np.uint64) == np.float64(b.final_objective).view(np.uint64)
    assert len(a.rounds) == len(b.rounds)
    for ra, rb in zip(a.rounds, b.rounds):
        assert (ra.objective, ra.objective_after_local, ra.local_gain, ra.exhaustion_gain, ra.local_iters,
                ra.exhaustion_iters) == (rb.objective, rb.objective_after_local, rb.local_gain, rb.exhaustion_gain,
                                         rb.local_iters, rb.exhaustion_iters)
    for m in range(2):
        va, vb = np.asarray(a.controllers.values(m)), np.asarray(b.controllers.values(m))
        assert np.array_equal(va.view(np.uint64), vb.view(np.uint64)), m


def _sweep(P, n, d):
    return [P.Witsenhausen(k=0.05 + 0.95 * i / max(n - 1, 1), sigma=(3.0, 5.0, 7.0)[i % 3],
                           grids=[(-25.0, 25.0, d)] * 2) for i in range(n)]


@pytest.mark.parametrize("d", [301, 200])
def test_batch_matches_single_solves(P, d):
    from paper_1908_04489_b200.batch import solve_batch

    cfg = P.SolverConfig(max_rounds=6)
    probs = _sweep(P, 10, d)
    got = solve_batch(probs, cfg)
    for p, r in zip(_sweep(P, 10, d), got):
        _same(P, r, P.solve(p, cfg))


def test_batch_default_grid_to_convergence(P):
    """config-4 instances at d = 2000, default solver, run to convergence."""
    from paper_1908_04489_b200.batch import solve_batch

    probs = [P.Witsenhausen(k=k, sigma=s) for k, s in ((0.05, 3.0), (0.2, 5.0), (0.6, 7.0), (1.0, 5.0))]
    got = solve_batch(probs, P.SolverConfig())
    assert got[1].final_objective == 0.16692114286407383 and got[1].total_rounds == 22
    for (k, s), r in zip(((0.05, 3.0), (0.2, 5.0), (0.6, 7.0), (1.0, 5.0)), got):
        _same(P, r, P.solve(P.Witsenhausen(k=k, sigma=s), P.SolverConfig()))


def test_batch_fixed_split_and_initials(P):
    from paper_1908_04489_b200.batch import solve_batch

    cfg = P.SolverConfig(max_rounds=4, fixed_local_iters=7)
    probs = _sweep(P, 5, 257)
    rng = np.random.default_rng(4)
    inits = [P.ControllerSet(tuple(P.SampledController(g, g.points + 0.3 * rng.uniform(-1, 1, g.d)) for g in p.grids))
             for p in probs]
    got = solve_batch(probs, cfg, inits)
    for p, U, r in zip(probs, inits, got):
        _same(P, r, P.solve(p, cfg, U))


def test_solve_many_routes_to_batch(P):
    cfg = P.SolverConfig(max_rounds=3)
    got = P.solve_many(_sweep(P, 6, 301), cfg)
    for p, r in zip(_sweep(P, 6, 301), got):
        _same(P, r, P.solve(p, cfg))


def test_batch_numeric_error_is_the_single_solves(P):
    from paper_1908_04489_b200.batch import solve_batch

    probs = _sweep(P, 3, 201)
    g0, g1 = probs[1].grids
    bad = P.ControllerSet((P.SampledController(g0, np.full(g0.d, 1e200)), P.SampledController(g1, g1.points)))
    with pytest.raises(P.NumericError) as got:
        solve_batch(probs, P.SolverConfig(max_rounds=2), [None, bad, None])
    with pytest.raises(P.NumericError) as want:
        P.solve(probs[1], P.SolverConfig(max_rounds=2), bad)
    assert str(got.value) == str(want.value)


def _same_as_oracle(r, want):
    """A SolveResult vs oracle.solve's (u0, u1, J, rounds, termination), bitwise."""
    u0, u1, J, rounds, term = want
    assert r.termination == term
    assert np.float64(r.final_objective).view(np.uint64) == np.float64(J).view(np.uint64)
    assert len(r.rounds) == len(rounds)
    for got, (idx, after_exh, gl, ge, nl, ne, after_local) in zip(r.rounds, rounds):
        assert (got.round_index, got.local_iters, got.exhaustion_iters) == (idx, nl, ne)
        g = np.array([got.objective, got.objective_after_local, got.local_gain, got.exhaustion_gain])
        w = np.array([after_exh, after_local, gl, ge])
        assert np.array_equal(g.view(np.uint64), w.view(np.uint64)), (idx, g, w)
    for m, w in enumerate((u0, u1)):
        assert np.array_equal(np.asarray(r.controllers.values(m)).view(np.uint64), w.view(np.uint64)), m


@pytest.mark.parametrize("d", [201, 301])
def test_batch_vs_oracle_sweep(P, oracle_mod, d):
    """The batched engine against the oracle (not against itself): every
    (k, sigma) of k in {0.05, 0.2, 0.6, 1.0} x sigma in {3, 5, 7} solved to
    convergence in ONE solve_batch, each instance's trajectory (controllers,
    J, every RoundReport) bitwise the oracle's sequential solve
    (reference solver.py:234-290)."""
    from paper_1908_04489_b200.batch import solve_batch

    ks = [(k, s) for k in (0.05, 0.2, 0.6, 1.0) for s in (3.0, 5.0, 7.0)]
    probs = [P.Witsenhausen(k=k, sigma=s, grids=[(-25.0, 25.0, d)] * 2) for k, s in ks]
    got = solve_batch(probs, P.SolverConfig())
    assert len({r.total_rounds for r in got}) > 1  # schedules diverge between instances
    for (k, s), pr, r in zip(ks, probs, got):
        p = oracle_mod.OracleWitsenhausen(k=k, sigma=s, grid0=(-25.0, 25.0, d), grid1=(-25.0, 25.0, d),
                                          f0=pr._f0, fw0=pr._fw0)
        _same_as_oracle(r, oracle_mod.solve(p, oracle_mod.OracleConfig()))
