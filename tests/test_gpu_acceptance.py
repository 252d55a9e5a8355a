"""The reference's acceptance criteria (its
tests/test_acceptance.py) evaluated on the device path.  Criteria 8-9
(Monte Carlo, the Quadratic toy problem) are outside this package's scope
(DESIGN.md §9); criterion 2 is a documented xfail in the reference too."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available()
    return P


@pytest.fixture(scope="module")
def wc_full(P):
    prob = P.Witsenhausen()
    return prob, P.solve(prob, P.SolverConfig())


def test_criterion_1_witsenhausen_value_and_stretch(P, wc_full):
    _, res = wc_full
    assert res.termination == "converged" and res.final_objective <= 0.175
    big = P.solve(P.Witsenhausen(grids=[(-25.0, 25.0, 14000)] * 2), P.SolverConfig())
    assert 0.1665 <= big.final_objective <= 0.1680  # stretch goal at the paper's grid size
    assert big.final_objective == 0.1669226437644399  # the reference's bits


def test_criterion_3_zero_delay_value(P):
    res = P.solve(P.ZeroDelay(power_weight=2.0), P.SolverConfig())
    assert res.termination == "converged" and 0.885 <= res.final_objective <= 0.901


def test_criterion_4_adaptive_beats_fixed_split(P):
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, 1000)] * 2)

    def rounds_to(cfg):
        res = P.solve(prob, cfg)
        for r in res.rounds:
            if r.objective <= 0.20:
                return r.round_index
        return 10**9

    assert rounds_to(P.SolverConfig(max_rounds=40)) <= rounds_to(P.SolverConfig(max_rounds=40, fixed_local_iters=19))


def test_criterion_5_monotone_descent(wc_full):
    _, res = wc_full
    for r in res.rounds:
        assert r.objective - r.objective_after_local <= 1e-9 * (1.0 + abs(r.objective))


def test_criterion_6_oracle_equivalence(P, wc_full):
    """Partial-exhaustion output == windowed argmin with scalar evaluations, at
    100 random (stage, point) pairs on each device problem."""
    rng = np.random.default_rng(6)
    probs = [wc_full[0], P.ZeroDelay(grids=[(-5.0, 5.0, 401), (-6.0, 6.0, 481)]),
             P.Inventory(grids=[(-3.0, 3.0, 241)] * 2)]
    for prob in probs:
        U = prob.identity_controllers()
        U = P.ControllerSet(tuple(P.SampledController(g, prob.project(m, g.points + rng.uniform(-0.5, 0.5, g.d)))
                                  for m, g in enumerate(prob.grids)))
        cfg = P.SolverConfig()
        swept = [P.partial_exhaustion_phase(prob, m, U, cfg) for m in range(prob.M)]
        for _ in range(100):
            m = int(rng.integers(0, prob.M))
            g = prob.grids[m]
            i = int(rng.integers(0, g.d))
            best = P.windowed_argmin(prob, m, float(g.points[i]), U, cfg.radius_for(g))
            assert prob.project(m, np.array([best]))[0] == swept[m][i], (prob.name, m, i)


@pytest.mark.parametrize("name", ["witsenhausen", "zero_delay", "inventory"])
def test_criterion_7_consistency_50_points(P, name):
    prob = {"witsenhausen": P.Witsenhausen(grids=[(-25.0, 25.0, 301)] * 2),
            "zero_delay": P.ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)]),
            "inventory": P.Inventory(grids=[(-3.0, 3.0, 241)] * 2)}[name]
    rng = np.random.default_rng(7)
    U = P.ControllerSet(tuple(P.SampledController(g, prob.project(m, g.points + 0.5 * rng.uniform(-1, 1, g.d)))
                              for m, g in enumerate(prob.grids)))
    J = prob.objective(U)
    for _ in range(50):
        m = int(rng.integers(0, prob.M))
        g = prob.grids[m]
        i = int(rng.integers(0, g.d))
        y, u = float(g.points[i]), float(U.values(m)[i])
        vals = U.values(m).copy()
        vals[i] = u + 0.05
        J2 = prob.objective(U.replace(m, U[m].with_values(vals)))
        dC = prob.marginal_cost(m, u + 0.05, y, U) - prob.marginal_cost(m, u, y, U)
        assert abs((J2 - J) - dC * g.spacing) <= 1e-6 * (1.0 + abs(J))


def test_criterion_11_rank_determinism_via_cli_csv(P, tmp_path):
    """Controller CSVs are bitwise identical across runs (and, by
    test_distributed, across rank counts)."""
    from paper_1908_04489_b200 import cli

    base = ["solve", "--problem", "witsenhausen", "--grid=-25,25,400", "--solver", "max_rounds=4"]
    assert cli.main(base + ["--out", str(tmp_path / "a")]) == 0
    assert cli.main(base + ["--out", str(tmp_path / "b")]) == 0
    for m in (0, 1):
        assert (tmp_path / "a" / f"controller_{m}.csv").read_bytes() == \
            (tmp_path / "b" / f"controller_{m}.csv").read_bytes()


def test_criterion_12_inventory_properties(P):
    prob = P.Inventory()
    res = P.solve(prob, P.SolverConfig())
    assert all(np.asarray(res.controllers.values(m)).min() >= 0.0 for m in range(prob.M))
    for m in range(prob.M):
        mass = float(prob.forward_density(m, res.controllers).sum() * prob.grids[m].spacing)
        assert abs(mass - 1.0) <= 1e-6
    for r in res.rounds:
        assert r.objective - r.objective_after_local <= 1e-9 * (1.0 + abs(r.objective))
