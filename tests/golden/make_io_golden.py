"""Golden documents for the JSON/CLI solve path (paper_1904_10548_b200/io.py, cli.py).

Run in the build container, where the Python reference is importable:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py
For each bundled demo kind it writes the reference's own document set
(`watermpc generate-demo`: network, scenarioTree, forecaster,
controllerconfig, state; the simulator-only documents are dropped) and the
reference's `watermpc solve` output (controlOutput.json) under
tests/golden/io/<kind>/. The GPU test runs our CLI on the same documents and
compares controlOutput.json; the CPU tests load every document with our
readers and compare with the reference readers' arrays (stored in docs.npz).
"""
import json
import os
import shutil
import sys
import tempfile

import numpy as np

from watermpc import io as rio
from watermpc.cli import main as ref_main

HERE = os.path.dirname(os.path.abspath(__file__))
KEEP = ("network.json", "scenarioTree.json", "forecaster.json", "controllerconfig.json", "state.json")

for kind in ("tank1", "net3"):
    out = os.path.join(HERE, "io", kind)
    os.makedirs(out, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        assert ref_main(["generate-demo", "--kind", kind, "--out", tmp]) == 0
        for name in KEEP:
            shutil.copy(os.path.join(tmp, name), os.path.join(out, name))
    args = ["--network", "network.json", "--tree", "scenarioTree.json", "--forecast", "forecaster.json",
            "--config", "controllerconfig.json", "--state", "state.json"]
    cwd = os.getcwd()
    os.chdir(out)
    try:
        assert ref_main(["solve", *args, "--out", "."]) == 0
        # certainty-equivalent prices (zero_price_errors before attaching the forecast)
        assert ref_main(["solve", *args, "--nominal-prices", "--out", "nominal"]) == 0
    finally:
        os.chdir(cwd)
    # the reference readers' view of every document (our readers must agree)
    m = rio.load_network(os.path.join(out, "network.json"))
    t = rio.load_tree(os.path.join(out, "scenarioTree.json"))
    f = rio.load_forecast(os.path.join(out, "forecaster.json"))
    h, w, s = rio.load_controller_config(os.path.join(out, "controllerconfig.json"))
    x, up, k = rio.load_state(os.path.join(out, "state.json"))
    arrays = dict(A=m.A, B=m.B, Gd=m.Gd, E=m.E, Ed=m.Ed, xmin=m.x_min, xmax=m.x_max, xsafe=m.x_safe,
                  umin=m.u_min, umax=m.u_max, alpha0=m.alpha0, dt=m.dt, stage=t.stage, anc=t.anc, prob=t.prob,
                  d_hat=f.d_hat, alpha_hat=f.alpha_hat, horizon=h, w_alpha=w.w_alpha, w_u=np.asarray(w.w_u),
                  w_s=w.w_s, w_x=w.w_x, max_iter=s.max_iter, tol=s.tol, x=x, u_prev=up, k=k)
    for key in ("eps", "demand", "price"):
        if getattr(t, key) is not None:
            arrays["tree_" + key] = getattr(t, key)
    np.savez(os.path.join(out, "docs.npz"), **arrays)
    print(kind, json.load(open(os.path.join(out, "controlOutput.json")))["iterations"], "iterations")
