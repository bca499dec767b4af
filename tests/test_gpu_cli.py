"""`cli solve` on the reference's own demo documents (tests/golden/io) against
the reference's `watermpc solve` output (controlOutput.json): same
termination, same iteration count, u0 within the parity metric."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_err
from paper_1904_10548_b200 import cli
from paper_1904_10548_b200 import io as wio

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nominal", [False, True])
@pytest.mark.parametrize("kind", ["tank1", "net3"])
def test_cli_solve_matches_reference_control_output(kind, nominal, tmp_path, capsys):
    d = os.path.join(GOLDEN, "io", kind)
    extra = ["--nominal-prices"] if nominal else []
    rc = cli.main(["solve", "--network", os.path.join(d, "network.json"), "--tree", os.path.join(d, "scenarioTree.json"),
                   "--forecast", os.path.join(d, "forecaster.json"), "--config", os.path.join(d, "controllerconfig.json"),
                   "--state", os.path.join(d, "state.json"), "--out", str(tmp_path), "--threads", "4", *extra])
    assert rc == 0
    out = capsys.readouterr().out
    assert out.startswith("iters=") and "residual=" in out and "time_ms=" in out
    ours = wio.load_control_output(tmp_path / "controlOutput.json")
    ref = wio.load_control_output(os.path.join(d, "nominal" if nominal else "", "controlOutput.json"))
    assert ours["terminationReason"] == ref["terminationReason"]
    assert ours["iterations"] == ref["iterations"]
    assert rel_err(ours["u0"], ref["u0"]) <= 1e-8, (ours["u0"], ref["u0"])
    assert abs(ours["primalResidual"] - ref["primalResidual"]) <= 1e-8 * (1 + abs(ref["primalResidual"]))
    assert abs(ours["dualChange"] - ref["dualChange"]) <= 1e-6 * (1 + abs(ref["dualChange"]))
