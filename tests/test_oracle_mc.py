"""Monte-Carlo objective: the oracle's restatement of
simulate_cost vs the reference's recorded costs, the host draw order of the
package, and the device generator's Philox restatement vs published
known-answer vectors.  CPU only."""
import math

import numpy as np
import pytest

from mc_cases import CASES, SEEDS, controllers, oracle_problem
from parity_util import assert_bitwise


@pytest.mark.parametrize("tag", CASES)
def test_simulate_cost_matches_reference(golden, oracle_mod, tag):
    g = golden("mc")
    p = oracle_problem(oracle_mod, tag)
    costs = oracle_mod.simulate_cost(p, controllers(g, tag, p.M), g[f"{tag}_draws"])
    assert_bitwise(costs, g[f"{tag}_costs"], f"{tag} costs")
    # the reference's estimator is np.mean / np.std(ddof=1) over these costs
    est, se = g[f"{tag}_mc_2000_{SEEDS[tag]}"]
    assert float(np.mean(costs)) == est
    assert float(np.std(costs, ddof=1) / math.sqrt(costs.size)) == se


@pytest.mark.parametrize("tag", CASES)
def test_host_draw_order_matches_reference(golden, tag):
    """montecarlo._host_draws calls the generator exactly as simulate_cost does."""
    import paper_1908_04489_b200 as P
    from mc_cases import device_problem
    from paper_1908_04489_b200.montecarlo import _host_draws

    g = golden("mc")
    draws = _host_draws(device_problem(P, tag), np.random.default_rng(SEEDS[tag]), 2000)
    assert_bitwise(np.stack(draws), g[f"{tag}_draws"], f"{tag} draws")


def test_philox_known_answers(oracle_mod):
    """Random123's published Philox4x32-10 vectors."""
    kat = [((0, 0, 0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 6, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for args, want in kat:
        got = tuple(int(v[()]) for v in oracle_mod.philox4x32_10(*args))
        assert got == want


def test_philox_uniform_range_and_moments(oracle_mod):
    u1, u2 = oracle_mod.philox_uniform01(12345, np.arange(200_000), 1)
    for u in (u1, u2):
        assert u.min() > 0.0 and u.max() < 1.0
        assert abs(u.mean() - 0.5) < 5 * math.sqrt(1 / 12 / u.size)


def test_fixed_order_reduction_restatement(oracle_mod):
    rng = np.random.default_rng(3)
    for n in (1, 4095, 4096, 4097, 3 * 4096 + 17, 1024 * 4096 + 5):
        x = rng.uniform(0, 10, n)
        parts = oracle_mod.mc_chunk_partials(x)
        assert parts.size == -(-n // 4096)
        total = oracle_mod.mc_reduce(parts)
        assert abs(total - math.fsum(x)) <= 1e-12 * abs(total)
