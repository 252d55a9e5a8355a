"""The objective's serial trapezoid (kernels.py:136-144) in its chunked exact
form (k_tz_*, n >= 32768): bitwise the serial sum on adversarial sequences --
ties at the running sum's half-ulp, sign changes, binade crossings both ways,
zero crossings, tiny/huge/subnormal addends, non-finite samples -- against the
oracle's serial C sum.  (The algorithm's host restatement passed the same
families: DESIGN.md §2c.)"""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available()
    return P


def _families(n, rng):
    yield "uniform", rng.uniform(0, 1, n)
    yield "normal", rng.normal(0, 1, n)
    yield "wide", rng.normal(5, 1, n) * 10.0 ** rng.integers(-5, 5, n)
    yield "ties 2^54", np.concatenate([[2.0 ** 54], rng.integers(-7, 8, n - 1).astype(float)])
    yield "ties 3*2^53", np.concatenate([[3 * 2.0 ** 53], rng.choice([-1.0, 1.0, 3.0, -3.0, 0.5, -0.5], n - 1)])
    yield "tiny", np.concatenate([[1.0], np.full(n - 1, 2.0 ** -53)])
    yield "tiny ties", np.concatenate([[1.0], rng.choice([2.0 ** -53, -2.0 ** -53, 2.0 ** -54,
                                                           -(2.0 ** -53 + 2.0 ** -80)], n - 1)])
    yield "walk", np.concatenate([[4.0], rng.choice([-1.0, 1.0], n - 1) * rng.uniform(0, 1e-3, n - 1)])
    yield "huge", np.concatenate([[0.0], rng.normal(0, 1e300, n - 1)])
    yield "subnormal", np.concatenate([[1e-300], rng.normal(0, 1e-310, n - 1)])
    yield "binade down", np.concatenate([[2.0 ** 52], np.full(n - 1, -1.0)])
    yield "negative ties", np.concatenate([[-(2.0 ** 53)], rng.integers(-3, 4, n - 1).astype(float)])
    yield "to zero", np.concatenate([rng.uniform(0, 1, n // 2), -rng.uniform(0, 1, n - n // 2)])
    x = rng.normal(0, 1, n)
    x[n // 3] = np.nan
    yield "nan", x
    x = rng.normal(0, 1, n)
    x[n - 5] = -np.inf
    yield "inf", x
    for t in range(12):
        x = rng.normal(rng.normal(), 10.0 ** rng.uniform(-3, 3), n) * rng.choice([1, 0.5, 2 ** -20, 3.0], n)
        if t % 3 == 0:
            x = np.round(x * 4) / 4
        yield f"random {t}", x


@pytest.mark.parametrize("n", [32768, 32769, 65536 + 1023, 1 << 20])
def test_chunked_trapezoid_bitwise(P, oracle_mod, n):
    rng = np.random.default_rng(n)
    for name, x in _families(n, rng):
        h = float(rng.uniform(1e-5, 1.0))
        got = P.kernels.trapezoid_sum(x, h)
        want = oracle_mod.trapezoid_sum(x, h)
        assert np.float64(got).tobytes() == np.float64(want).tobytes(), (name, got, want)


def test_chunked_trapezoid_objective_terms(P, golden):
    """The real input: the 2^20 bench snapshot's objective integrand."""
    from oracle import oracle as orc

    d = 1 << 20
    sol = golden("wc_solve_d2000")
    yc, y = np.linspace(-25, 25, 2000), np.linspace(-25, 25, d)
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
    U = P.ControllerSet((P.SampledController(prob.grids[0], np.interp(y, yc, sol["u0"])),
                         P.SampledController(prob.grids[1], np.interp(y, yc, sol["u1"]))))
    terms = prob.device_objective_terms(U).cpu().numpy()
    J = prob.objective(U)
    assert np.float64(J).tobytes() == np.float64(orc.trapezoid_sum(terms, prob.grids[0].spacing)).tobytes()


def test_chunked_trapezoid_first_nonfinite_index(P):
    from paper_1908_04489_b200 import _lib

    n = 1 << 17
    for bad in (0, 1, 5000, n - 2, n - 1):
        x = torch.ones(n, dtype=torch.float64, device="cuda")
        x[bad] = float("nan")
        x[min(bad + 7, n - 1)] = float("inf")
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        err = torch.full((1,), 2 ** 62, dtype=torch.int64, device="cuda")
        _lib.call("ucp_trapezoid_sum", x.data_ptr(), n, 0.5, out.data_ptr(), err.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert int(err.item()) == bad


def test_chunked_trapezoid_concurrent_streams(P, oracle_mod):
    """Per-stream scratch: interleaved calls on two streams, each bitwise."""
    from paper_1908_04489_b200 import _lib

    rng = np.random.default_rng(3)
    n = 1 << 18
    xs = [rng.normal(0, 1, n), rng.uniform(0, 0.3, n)]
    want = [oracle_mod.trapezoid_sum(x, 0.25) for x in xs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    dev = [torch.from_numpy(x).cuda() for x in xs]
    outs = [torch.empty(8, dtype=torch.float64, device="cuda") for _ in xs]
    torch.cuda.synchronize()
    for rep in range(8):
        for k in range(2):
            _lib.call("ucp_trapezoid_sum", dev[k].data_ptr(), n, 0.25, outs[k][rep:].data_ptr(), None,
                      streams[k].cuda_stream)
    torch.cuda.synchronize()
    for k in range(2):
        got = outs[k].cpu().numpy()
        assert all(np.float64(g).tobytes() == np.float64(want[k]).tobytes() for g in got), k
