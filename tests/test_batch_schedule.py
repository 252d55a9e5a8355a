"""Host logic of the batched engine (batch.schedule_rounds) on CPU: B
instances advanced in lock-step ticks, each on its own round schedule, with
an oracle-backed device stand-in.  Every instance's round reports, final J
and termination must equal the oracle's sequential solve of that instance
(solve_generic restates solver.py:234-290)."""
import numpy as np
import pytest

SPECS = [(0.2, 5.0), (0.05, 3.0), (0.6, 7.0), (1.0, 5.0)]


class OracleDev:
    def __init__(self, orc, probs, ocfg):
        self.orc, self.probs, self.ocfg = orc, probs, ocfg
        self.U = [[p.grid(0)[0].copy(), p.grid(1)[0].copy()] for p in probs]
        self.J = np.zeros((3, len(probs)))
        self.calls = []

    def iterate(self, kind, ids, iters):
        self.calls.append((kind, tuple(ids), iters))
        phase = self.orc.local_update if kind == 0 else self.orc.partial_exhaustion
        for i in ids:
            for _ in range(iters):
                for m in (0, 1):
                    self.U[i][m] = phase(self.probs[i], m, self.U[i], self.ocfg)

    def objective(self, lane, ids, row):
        for i in ids:
            self.J[row, i] = self.orc.objective_of(self.probs[i], self.U[i])

    def order(self):
        pass

    def read(self):
        from paper_1908_04489_b200.device_problem import NO_ERROR

        B = len(self.probs)
        return self.J.copy(), np.full((B, 6), NO_ERROR, dtype=np.int64), np.full(B, NO_ERROR, dtype=np.int64)

    def failed(self, i):
        raise AssertionError(f"instance {i} flagged")


@pytest.mark.parametrize("max_rounds", [1, 4])
def test_schedule_matches_sequential_solves(oracle_mod, max_rounds):
    import paper_1908_04489_b200 as P
    from paper_1908_04489_b200.batch import schedule_rounds

    orc = oracle_mod
    grids = ((-25.0, 25.0, 101), (-25.0, 25.0, 101))
    probs = [orc.OracleWitsenhausen(k=k, sigma=s, grid0=grids[0], grid1=grids[1]) for k, s in SPECS]
    ocfg = orc.OracleConfig(max_rounds=max_rounds)
    dev = OracleDev(orc, probs, ocfg)
    stats = {}
    current, reports, termination = schedule_rounds(dev, len(probs), P.SolverConfig(max_rounds=max_rounds), stats)
    for i, p in enumerate(probs):
        Us, J, rounds, term = orc.solve_generic(p, ocfg)
        assert termination[i] == term
        assert current[i] == J
        got = [(r.round_index, r.objective, r.local_gain, r.exhaustion_gain, r.local_iters, r.exhaustion_iters,
                r.objective_after_local) for r in reports[i]]
        assert got == rounds
        for m in (0, 1):
            assert np.array_equal(dev.U[i][m], Us[m])
    # one decision (sync) per round, not per block
    assert stats["decisions"] == max(len(r) for r in reports)
    # ticks run the local and exhaustion groups side by side once schedules diverge
    assert all(iters >= 1 for _, _, iters in dev.calls)


def test_schedule_fixed_split(oracle_mod):
    import paper_1908_04489_b200 as P
    from paper_1908_04489_b200.batch import schedule_rounds

    orc = oracle_mod
    probs = [orc.OracleWitsenhausen(k=k, sigma=s, grid0=(-25.0, 25.0, 61), grid1=(-25.0, 25.0, 61))
             for k, s in SPECS[:2]]
    dev = OracleDev(orc, probs, orc.OracleConfig())
    _, reports, termination = schedule_rounds(dev, 2, P.SolverConfig(max_rounds=3, fixed_local_iters=19))
    for rs, term in zip(reports, termination):
        assert term == "max_rounds" and len(rs) == 3
        assert all(r.local_iters == 19 and r.exhaustion_iters == 1 for r in rs)
