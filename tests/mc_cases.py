"""The Monte-Carlo fixture cases of tools/gen_golden.py:mc_fixture (tests/golden/mc.npz)."""
import numpy as np

CASES = ("wc", "zd", "inv", "inv3q")
SEEDS = {"wc": 90, "zd": 91, "inv": 92, "inv3q": 93}


def oracle_problem(orc, tag):
    if tag == "wc":
        return orc.OracleWitsenhausen(grid0=(-25.0, 25.0, 201), grid1=(-25.0, 25.0, 201))
    if tag == "zd":
        return orc.OracleZeroDelay(grid0=(-5.0, 5.0, 201), grid1=(-6.0, 6.0, 241))
    if tag == "inv":
        return orc.OracleInventory(grids=[(-3.0, 3.0, 241)] * 2)
    return orc.OracleInventory(stages=3, stage_cost="quadratic", order_cost=0.3,
                               grids=[(-3.0, 3.0, 97), (-2.5, 3.5, 131), (-3.0, 2.0, 111)])


def device_problem(P, tag):
    if tag == "wc":
        return P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
    if tag == "zd":
        return P.ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)])
    if tag == "inv":
        return P.Inventory(grids=[(-3.0, 3.0, 241)] * 2)
    return P.Inventory(stages=3, stage_cost="quadratic", order_cost=0.3,
                       grids=[(-3.0, 3.0, 97), (-2.5, 3.5, 131), (-3.0, 2.0, 111)])


def controllers(g, tag, M):
    return [g[f"{tag}_u{m}"] for m in range(M)]


class ReplayRng:
    """Stands in for a NumPy Generator, returning recorded draws in order."""

    def __init__(self, draws):
        self.draws = list(np.asarray(draws))

    def normal(self, loc, scale, n):
        return self.draws.pop(0)[:n]

    def uniform(self, lo, hi, n):
        return self.draws.pop(0)[:n]
