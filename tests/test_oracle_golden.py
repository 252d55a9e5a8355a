"""Pin the oracle (oracle/ucp_oracle.c + oracle/oracle.py) to the reference.

Every golden vector in tests/golden/ was produced by the reference package
itself (tools/gen_golden.py, numba backend).  The oracle must reproduce them
bit for bit on this host -- this is what licenses using it as the parity
checker for the CUDA path.
"""
import numpy as np
import pytest

from parity_util import assert_bitwise


@pytest.mark.parametrize("tag", ["k307", "k2", "k64"])
def test_gauss_moments_grid(golden, oracle_mod, tag):
    g = golden("kernels")
    t = oracle_mod.gauss_moments_grid(g[f"{tag}_centers"], g[f"{tag}_vals"], g[f"{tag}_a"],
                                      g[f"{tag}_h"], int(g[f"{tag}_d"]))
    for k in range(3):
        assert_bitwise(t[k], g[f"{tag}_grid_t{k}"], f"{tag} T{k}")


@pytest.mark.parametrize("tag", ["k307", "k2", "k64"])
def test_gauss_moments_points(golden, oracle_mod, tag):
    g = golden("kernels")
    p = oracle_mod.gauss_moments_points(g[f"{tag}_queries"], g[f"{tag}_xs"], g[f"{tag}_weights"],
                                        g[f"{tag}_a"], g[f"{tag}_h"], int(g[f"{tag}_d"]))
    for k in range(3):
        assert_bitwise(p[k], g[f"{tag}_pts_{k}"], f"{tag} M{k}")


def test_small_kernels(golden, oracle_mod):
    g = golden("kernels")
    assert_bitwise(oracle_mod.trapezoid_sum(g["trap_samples"], 0.37), g["trap_value"], "trapezoid")
    np.testing.assert_array_equal(
        oracle_mod.segmented_argmin(g["argmin_costs"], g["argmin_offsets"]), g["argmin_out"])
    flat, offs = oracle_mod.flatten_windows(g["flat_vals"], g["flat_lo"], g["flat_hi"])
    assert_bitwise(flat, g["flat_out"], "flatten")
    np.testing.assert_array_equal(offs, g["flat_offsets"])


def _problem(oracle_mod, g):
    d = int(g["d"])
    return oracle_mod.OracleWitsenhausen(grid0=(-25.0, 25.0, d), grid1=(-25.0, 25.0, d),
                                         f0=g["f0"], fw0=g["fw0"])


@pytest.mark.parametrize("tag", ["d201", "d2000"])
def test_host_constants(golden, oracle_mod, tag):
    """The oracle's own NumPy pdf reproduces the reference's f0/fw0 on this host."""
    g = golden(f"wc_{tag}")
    d = int(g["d"])
    p = oracle_mod.OracleWitsenhausen(grid0=(-25.0, 25.0, d), grid1=(-25.0, 25.0, d))
    assert_bitwise(p.f0, g["f0"], "f0")
    assert_bitwise(p.fw0, g["fw0"], "fw0")


@pytest.mark.parametrize("tag", ["d201", "d2000"])
@pytest.mark.parametrize("name", ["ident", "pert0", "pert1"])
def test_witsenhausen_phases(golden, oracle_mod, tag, name):
    g = golden(f"wc_{tag}")
    p = _problem(oracle_mod, g)
    cfg = oracle_mod.OracleConfig()
    u0, u1 = g[f"{name}_u0"], g[f"{name}_u1"]
    idx = np.arange(p.d0, dtype=np.int64)
    assert_bitwise(oracle_mod.objective(p, u0, u1), g[f"{name}_J"], "J")
    for m in (0, 1):
        u = u0 if m == 0 else u1
        assert_bitwise(p.cost_batch(m, u, idx, u0, u1), g[f"{name}_c{m}"], f"C{m}")
        assert_bitwise(p.cost_batch(m, u + 0.37, idx, u0, u1), g[f"{name}_c{m}_up"], f"C{m}+")
        assert_bitwise(oracle_mod.local_update_phase(p, m, u0, u1, cfg), g[f"{name}_lu{m}"], f"LU{m}")
        assert_bitwise(oracle_mod.partial_exhaustion_phase(p, m, u0, u1, cfg), g[f"{name}_ex{m}"],
                       f"EX{m}")
        small = oracle_mod.OracleConfig(search_radius=3.5 * (p.h0 if m == 0 else p.h1))
        assert_bitwise(oracle_mod.partial_exhaustion_phase(p, m, u0, u1, small), g[f"{name}_exs{m}"],
                       f"EXs{m}")
    v0, v1 = u0, u1
    for phase in (oracle_mod.local_update_phase, oracle_mod.partial_exhaustion_phase):
        v0 = phase(p, 0, v0, v1, cfg)
        v1 = phase(p, 1, v0, v1, cfg)
    assert_bitwise(v0, g[f"{name}_it_u0"], "it u0")
    assert_bitwise(v1, g[f"{name}_it_u1"], "it u1")
    assert_bitwise(oracle_mod.objective(p, v0, v1), g[f"{name}_it_J"], "it J")


@pytest.mark.parametrize("tag", ["d201", "d2000"])
def test_segmented_costs(golden, oracle_mod, tag):
    g = golden(f"wc_{tag}")
    p = _problem(oracle_mod, g)
    for m in (0, 1):
        got = p.cost_segmented(m, g["seg_u"], g["seg_offsets"], g["seg_idx"], g["pert0_u0"], g["pert0_u1"])
        assert_bitwise(got, g[f"seg_c{m}"], f"seg C{m}")


def test_full_solve_d201(golden, oracle_mod):
    g = golden("wc_solve_d201")
    p = _problem(oracle_mod, g)
    u0, u1, J, rounds, term = oracle_mod.solve(p)
    assert term == str(g["termination"])
    assert_bitwise(np.array([r[1] for r in rounds]), g["rounds"][:, 1], "per-round J")
    np.testing.assert_array_equal(np.array([r[4] for r in rounds]), g["rounds"][:, 4])
    assert_bitwise(u0, g["u0"], "u0")
    assert_bitwise(u1, g["u1"], "u1")
    assert_bitwise(J, g["final_J"], "J")


def test_fine_grid_samples(golden, oracle_mod):
    """2^20 grid, warm controllers: sampled stage-0 walks (W=503,316) and stage-1 moments."""
    fine = golden("wc_fine_2p20")
    sol = golden("wc_solve_d2000")
    d = int(fine["d"])
    p = oracle_mod.OracleWitsenhausen(grid0=(-25.0, 25.0, d), grid1=(-25.0, 25.0, d))
    cy, ch = oracle_mod.linspace_grid(-25.0, 25.0, 2000)
    near = np.clip(np.ceil((p.y0 - (-25.0)) / ch - 0.5).astype(np.int64), 0, 1999)
    u0, u1 = sol["u0"][near], sol["u1"][near]
    assert_bitwise(p.y0[fine["idx"]] + u0[fine["idx"]], fine["s"], "centres")
    sel = slice(0, 96)
    t = oracle_mod.gauss_moments_grid(fine["s"][sel], u1, p.a1, p.h1, d)
    for k in range(3):
        assert_bitwise(t[k], fine[f"t{k}"][sel], f"T{k}")
    q = fine["q_idx"][:6]
    m = oracle_mod.gauss_moments_points(p.y1[q], p.y0 + u0, p.fw0, p.a1, p.h1, d)
    for k in range(3):
        assert_bitwise(m[k], fine[f"m{k}"][:6], f"M{k}")


@pytest.mark.slow
def test_full_solve_d2000(golden, oracle_mod):
    g = golden("wc_solve_d2000")
    p = _problem(oracle_mod, g)
    u0, u1, J, rounds, term = oracle_mod.solve(p)
    assert len(rounds) == len(g["rounds"]) == 22
    assert_bitwise(J, g["final_J"], "J")
    assert_bitwise(u0, g["u0"], "u0")
