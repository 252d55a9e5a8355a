"""CLI on the device path (reference cli.py): parsing and exit codes on CPU;
solve/export/report and the CSV round trip on the GPU."""
import json

import numpy as np
import pytest

from paper_1908_04489_b200 import cli


def test_config_errors_exit_1(tmp_path, capsys):
    assert cli.main(["solve", "--problem", "nope"]) == 1
    assert cli.main(["solve", "--solver", "bogus=1", "--out", str(tmp_path)]) == 1
    assert cli.main(["solve", "--grid", "1,2", "--out", str(tmp_path)]) == 1
    assert cli.main(["solve", "--mode", "fixed_split:x", "--out", str(tmp_path)]) == 1
    bad = tmp_path / "c.json"
    bad.write_text(json.dumps({"problem": "witsenhausen", "color": "red"}))
    assert cli.main(["solve", "--config", str(bad)]) == 1
    assert cli.main([]) == 1


def test_run_config_merging(tmp_path):
    cfgf = tmp_path / "c.json"
    cfgf.write_text(json.dumps({"problem": "zero_delay", "params": {"power_weight": 3.0},
                                "solver": {"max_rounds": 7}}))
    args = cli.build_parser().parse_args(["solve", "--config", str(cfgf), "--param", "power_weight=1.5",
                                          "--grid=1:-6,6,301", "--solver", "precision=1e-8",
                                          "--out", str(tmp_path / "o")])
    rc = cli.load_run_config(args)
    assert rc.problem == "zero_delay" and rc.params == {"power_weight": 1.5}
    assert rc.solver == {"max_rounds": 7, "precision": 1e-8}
    assert rc.grids == [(-5.0, 5.0, 2000), (-6.0, 6.0, 301)]
    prob, scfg = rc.build()
    assert prob.power_weight == 1.5 and scfg.max_rounds == 7


@pytest.mark.gpu
def test_solve_exports_bitwise_csv_and_report(tmp_path, golden):
    g = golden("wc_solve_d201")
    out = tmp_path / "run"
    assert cli.main(["solve", "--grid=-25,25,201", "--out", str(out)]) == 0
    rep = json.loads((out / "report.json").read_text())
    assert rep["termination"] == "converged" and rep["backend"] == "b200"
    assert rep["total_rounds"] == len(g["rounds"])
    # host NumPy densities equal the golden's on this host: the CSV must
    # reproduce the reference's controllers bit for bit after parsing
    import paper_1908_04489_b200 as P

    prob = P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
    if not np.array_equal(prob._fw0, g["fw0"]):
        pytest.skip("host NumPy exp differs from the golden host")
    U = cli.read_controllers(prob, out)
    assert np.array_equal(np.asarray(U.values(0)).view(np.uint64), g["u0"].view(np.uint64))
    assert np.array_equal(np.asarray(U.values(1)).view(np.uint64), g["u1"].view(np.uint64))
    assert np.float64(rep["final_objective"]).view(np.uint64) == np.float64(g["final_J"]).view(np.uint64)


def test_numeric_failure_exit_2(tmp_path, monkeypatch):
    from paper_1908_04489_b200.problem import NumericError

    def boom(*a, **k):
        raise NumericError("witsenhausen: non-finite marginal cost in local-update phase at stage 0, grid point 3")

    monkeypatch.setattr(cli, "solve", boom)
    assert cli.main(["solve", "--grid=-25,25,101", "--out", str(tmp_path)]) == 2


def test_cli_fast_arithmetic_param():
    """`--param arithmetic=fma` selects the opt-in fast walk;
    the default stays the reference's arithmetic, and a bad value is a config error."""
    from paper_1908_04489_b200 import cli

    args = cli.build_parser().parse_args(["solve", "--problem", "witsenhausen", "--param", "arithmetic=fma"])
    prob, _ = cli.load_run_config(args).build()
    assert prob.arithmetic == "fma"
    prob, _ = cli.load_run_config(cli.build_parser().parse_args(["solve", "--problem", "witsenhausen"])).build()
    assert prob.arithmetic == "reference"
    with pytest.raises(ValueError):
        cli.load_run_config(cli.build_parser().parse_args(
            ["solve", "--problem", "witsenhausen", "--param", "arithmetic=fp32"])).build()
