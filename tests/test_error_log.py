"""Lazy device error log (device_problem.ErrorLog) host logic on CPU tensors:
rows are read once at the next synchronisation point, the FIRST failing phase
in execution order raises the reference's error (solver.py:170-176,
218-221), and the objective's own scalars travel in the same transfer."""
import numpy as np
import pytest
import torch


class _Prob:
    name = "witsenhausen"

    def __init__(self):
        import paper_1908_04489_b200 as P

        self.grids = [P.make_grid(-25.0, 25.0, 11), P.make_grid(-25.0, 25.0, 11)]


_PROBLEMS = []  # the log holds its problem weakly


def _log():
    from paper_1908_04489_b200.device_problem import ErrorLog

    _PROBLEMS.append(_Prob())
    return ErrorLog(torch.device("cpu"), _PROBLEMS[-1], capacity=8)


def test_clean_rows_return_extra():
    from paper_1908_04489_b200.distributed import LOCAL

    log = _log()
    log.slot("local", 0, LOCAL)
    log.slot("exhaustion", 1, LOCAL)
    extra = torch.tensor([7, 9], dtype=torch.int64)
    assert log.flush(LOCAL, extra=extra).tolist() == [7, 9]
    assert log.meta == [] and log.flush(LOCAL) is None


def test_first_failing_phase_raises_in_order():
    import paper_1908_04489_b200 as P
    from paper_1908_04489_b200.distributed import LOCAL

    log = _log()
    log.slot("local", 0, LOCAL)
    r1 = log.slot("exhaustion", 1, LOCAL)
    r2 = log.slot("local", 1, LOCAL)
    r1[0] = 4   # partial exhaustion, stage 1, point 4
    r2[1] = 2   # a later phase's failure must not win
    with pytest.raises(P.NumericError, match=r"witsenhausen: non-finite marginal cost in partial-exhaustion phase at stage 1, grid point 4 \(y=np\.float64\(-5\.0\)\)"):
        log.flush(LOCAL, extra=torch.zeros(2, dtype=torch.int64))
    # the log is reset after a flush
    assert log.meta == [] and bool((log.rows == log.rows[0, 0]).all())


def test_non_finite_controller_value_is_a_value_error():
    from paper_1908_04489_b200.distributed import LOCAL

    log = _log()
    r = log.slot("local", 0, LOCAL)
    r[2] = 3  # the stepped value itself is not finite (grids.py: SampledController)
    with pytest.raises(ValueError, match="grid point 3 is not finite"):
        log.flush(LOCAL)


def test_capacity_overflow_flushes_early():
    from paper_1908_04489_b200.distributed import LOCAL

    log = _log()
    for _ in range(8):
        log.slot("local", 0, LOCAL)
    log.slot("local", 1, LOCAL)  # the 9th row forces a flush of the first 8
    assert len(log.meta) == 1
    rows = log.slots([("local", 0)] * 20, LOCAL)  # more than the capacity: the buffer grows
    assert rows.shape == (20, 3) and np.all(rows.numpy() == rows.numpy()[0, 0])
