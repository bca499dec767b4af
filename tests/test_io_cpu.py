"""JSON documents of the solve path (paper_1904_10548_b200/io.py, SURVEY §8f
item 4) against the reference's own documents and readers
(tests/golden/io, made by tests/golden/make_io_golden.py from
`watermpc generate-demo` / `watermpc solve`)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1904_10548_b200 import cli
from paper_1904_10548_b200 import io as wio

KINDS = ("tank1", "net3")
DOCS = ("network.json", "scenarioTree.json", "forecaster.json", "controllerconfig.json", "state.json")


def _dir(kind):
    return os.path.join(GOLDEN, "io", kind)


def _load_all(kind):
    d = _dir(kind)
    return (wio.load_network(os.path.join(d, "network.json")), wio.load_tree(os.path.join(d, "scenarioTree.json")),
            wio.load_forecast(os.path.join(d, "forecaster.json")),
            wio.load_controller_config(os.path.join(d, "controllerconfig.json")),
            wio.load_state(os.path.join(d, "state.json")))


@pytest.mark.parametrize("kind", KINDS)
def test_readers_match_reference_readers(kind):
    m, t, f, (h, w, s), (x, up, k) = _load_all(kind)
    ref = np.load(os.path.join(_dir(kind), "docs.npz"))
    ours = dict(A=m.A, B=m.B, Gd=m.Gd, E=m.E, Ed=m.Ed, xmin=m.x_min, xmax=m.x_max, xsafe=m.x_safe, umin=m.u_min,
                umax=m.u_max, alpha0=m.alpha0, dt=m.dt, stage=t.stage, anc=t.anc, prob=t.prob, d_hat=f.d_hat,
                alpha_hat=f.alpha_hat, horizon=h, w_alpha=w.w_alpha, w_u=np.asarray(w.w_u), w_s=w.w_s, w_x=w.w_x,
                max_iter=s.max_iter, tol=s.tol, x=x, u_prev=up, k=k)
    for key in ("eps", "demand", "price"):
        if getattr(t, key) is not None:
            ours["tree_" + key] = getattr(t, key)
    assert sorted(ours) == sorted(ref.files)
    for key in ref.files:
        np.testing.assert_array_equal(np.asarray(ours[key]), ref[key], err_msg=key)
    assert s.gamma is None


@pytest.mark.parametrize("kind", KINDS)
def test_writers_reproduce_reference_documents(kind, tmp_path):
    m, t, f, (h, w, s), (x, up, k) = _load_all(kind)
    wio.save_network(m, tmp_path / "network.json")
    wio.save_tree(t, tmp_path / "scenarioTree.json")
    wio.save_forecast(f, tmp_path / "forecaster.json")
    wio.save_controller_config(h, w, s, tmp_path / "controllerconfig.json")
    wio.save_state(x, up, k, tmp_path / "state.json")
    for name in DOCS:
        with open(os.path.join(_dir(kind), name)) as a, open(tmp_path / name) as b:
            assert json.load(a) == json.load(b), name  # same fields, same values
    # and what we write reads back value-identical
    m2 = wio.load_network(tmp_path / "network.json")
    np.testing.assert_array_equal(m2.B, m.B)
    t2 = wio.load_tree(tmp_path / "scenarioTree.json")
    np.testing.assert_array_equal(t2.anc, t.anc)


def test_control_output_round_trip(tmp_path):
    d = wio.load_control_output(os.path.join(_dir("net3"), "controlOutput.json"))
    assert d["terminationReason"] == "converged" and d["u0"].shape == (4,)

    class R:
        u0 = d["u0"]
        iterations = d["iterations"]
        termination = d["terminationReason"]
        primal_residual = d["primalResidual"]
        dual_change = d["dualChange"]
        solve_time_s = d["solveTimeMs"] / 1e3

    wio.save_control_output(R, tmp_path / "c.json")
    d2 = wio.load_control_output(tmp_path / "c.json")
    np.testing.assert_array_equal(d2["u0"], d["u0"])
    assert d2["iterations"] == d["iterations"] and d2["dualChange"] == d["dualChange"]


def _write(tmp_path, name, doc):
    p = tmp_path / name
    p.write_text(doc if isinstance(doc, str) else json.dumps(doc))
    return p


@pytest.mark.parametrize("mutate,pointer", [
    (lambda d: d.pop("B"), "/B: missing required field"),
    (lambda d: d.update(schemaVersion=2), "/schemaVersion: unsupported schema version 2"),
    (lambda d: d["B"].pop(), "/B: expected"),
    (lambda d: d["xmin"].append(1.0), "/xmin: expected"),
    (lambda d: d["A"][0].append(0.0), "/A: rows have inconsistent lengths"),
    (lambda d: d.update(dt="1"), "/dt: expected a number"),
    (lambda d: d["umax"].__setitem__(0, True), "/umax/0: expected a number"),
])
def test_schema_errors_carry_pointers(tmp_path, mutate, pointer):
    doc = json.load(open(os.path.join(_dir("net3"), "network.json")))
    mutate(doc)
    p = _write(tmp_path, "network.json", doc)
    with pytest.raises(wio.SchemaError, match=pointer.replace("/", "/").replace("[", r"\[")):
        wio.load_network(p)


def test_non_finite_and_parse_errors(tmp_path):
    p = _write(tmp_path, "state.json", '{"schemaVersion": 1, "x": [NaN], "uPrev": [0.0]}')
    with pytest.raises(wio.SchemaError, match="non-finite number 'NaN'"):
        wio.load_state(p)
    p = _write(tmp_path, "state.json", '{"schemaVersion": 1, "x": [1.0,]')
    with pytest.raises(wio.SchemaError, match="parse error at byte"):
        wio.load_state(p)
    p = _write(tmp_path, "state.json", "[1, 2]")
    with pytest.raises(wio.SchemaError, match="top-level value must be an object"):
        wio.load_state(p)
    with pytest.raises(ValueError):
        wio.save_document({"x": float("nan")}, tmp_path / "bad.json")


def test_cross_validate_reports_mismatches():
    m, t, f, (h, w, s), (x, up, k) = _load_all("net3")
    assert wio.cross_validate(model=m, tree=t, forecast=f, horizon=h, weights=w, state=(x, up, k)) == []
    msgs = wio.cross_validate(model=m, tree=t, horizon=h + 1, state=(x[:-1], up, k))
    assert any("controller horizon" in s for s in msgs)
    assert any("state x has" in s for s in msgs)


def test_cli_validate(tmp_path, capsys):
    d = _dir("net3")
    args = ["validate", "--network", os.path.join(d, "network.json"), "--tree", os.path.join(d, "scenarioTree.json"),
            "--forecast", os.path.join(d, "forecaster.json"), "--config", os.path.join(d, "controllerconfig.json"),
            "--state", os.path.join(d, "state.json")]
    assert cli.main(args) == 0
    assert capsys.readouterr().out.strip() == "ok"
    assert cli.main(["validate"]) == 2
    other = os.path.join(_dir("tank1"), "network.json")  # 1 tank vs net3's tree and state
    assert cli.main(["validate", "--network", other, "--tree", os.path.join(d, "scenarioTree.json"),
                     "--state", os.path.join(d, "state.json")]) == 1
    assert "problem(s) found" in capsys.readouterr().out


def test_cli_solve_schema_error_exit_code(tmp_path, capsys):
    d = _dir("net3")
    bad = _write(tmp_path, "network.json", {"schemaVersion": 1})
    rc = cli.main(["solve", "--network", str(bad), "--tree", os.path.join(d, "scenarioTree.json"),
                   "--forecast", os.path.join(d, "forecaster.json"), "--config", os.path.join(d, "controllerconfig.json"),
                   "--state", os.path.join(d, "state.json"), "--out", str(tmp_path)])
    assert rc == 1
    assert "error: /A: missing required field" in capsys.readouterr().err
