"""Config 5 (PAPER.md's additional examples): the oracle's restatement of
ZeroDelay and Inventory (M = 1, 2, 3 stages) vs the reference's goldens."""
import numpy as np
import pytest

from parity_util import assert_bitwise

FIXTURES = ["zd_small", "zd_pw07", "inv_m1", "inv_m2", "inv_m3", "inv_m3q", "zd_default", "inv_default"]


def oracle_problem(orc, g):
    specs = [tuple(float(v) if k < 2 else int(v) for k, v in enumerate(row)) for row in g["specs"]]
    if "pw" in g:
        return orc.OracleZeroDelay(power_weight=float(g["pw"]), grid0=specs[0], grid1=specs[1], f0=g["f0"],
                                   fw0=g["fw0"])
    return orc.OracleInventory(stages=int(g["stages"]), stage_cost=str(g["stage_cost"]),
                               order_cost=float(g["order_cost"]) if "order_cost" in g else 0.1, grids=specs)


@pytest.mark.parametrize("tag", FIXTURES)
def test_config5_phases_and_solve(golden, oracle_mod, tag):
    g = golden(tag)
    p = oracle_problem(oracle_mod, g)
    cfg = oracle_mod.OracleConfig()
    for name in ("ident", "pert0", "pert1"):
        Us = [g[f"{name}_u{m}"] for m in range(p.M)]
        assert_bitwise(oracle_mod.objective_of(p, Us), g[f"{name}_J"], f"{name} J")
        for m in range(p.M):
            idx = np.arange(Us[m].size, dtype=np.int64)
            assert_bitwise(oracle_mod._cost_batch(p, m, Us[m], idx, Us), g[f"{name}_c{m}"], f"{name} C{m}")
            assert_bitwise(oracle_mod.local_update(p, m, Us, cfg), g[f"{name}_lu{m}"], f"{name} LU{m}")
            assert_bitwise(oracle_mod.partial_exhaustion(p, m, Us, cfg), g[f"{name}_ex{m}"], f"{name} EX{m}")
        V = list(Us)
        for phase in (oracle_mod.local_update, oracle_mod.partial_exhaustion):
            for m in range(p.M):
                V[m] = phase(p, m, V, cfg)
        for m in range(p.M):
            assert_bitwise(V[m], g[f"{name}_it_u{m}"], f"{name} it u{m}")
    if "solve_J" in g:
        Us, J, rounds, term = oracle_mod.solve_generic(p, cfg)
        assert term == str(g["solve_termination"])
        assert_bitwise(np.array([r[1] for r in rounds]), g["solve_rounds"][:, 1], "per-round J")
        assert_bitwise(J, g["solve_J"], "J")
        for m in range(p.M):
            assert_bitwise(Us[m], g[f"solve_u{m}"], f"u{m}")
