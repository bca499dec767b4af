"""Command line for the solve path: ``python -m paper_1904_10548_b200.cli solve ...``.

Mirrors the reference's ``watermpc solve`` (``cli.py:129-160``) and
``validate`` (``cli.py:84-126``) on the GPU solver.
Arguments, documents, stdout and exit codes are the same:
* on success the command writes ``<out>/controlOutput.json``, prints
  ``iters=... residual=... time_ms=...`` and returns 0;
* schema errors, I/O errors, cross-document mismatches and solver failures
  print a message on stderr and return 1.

``--threads`` is accepted for parity and ignored, as in ``SolverConfig``. The
simulate, reduce and generate-demo commands prepare data around the path and
are out of scope.
"""

from __future__ import annotations

import argparse
import sys
from dataclasses import replace
from pathlib import Path

from . import io as wio
from .problem import assemble_problem
from .solver import solve as solve_instance
from .tree import attach_forecast, validate_tree, zero_price_errors


def _common(p: argparse.ArgumentParser) -> None:
    p.add_argument("--out", type=Path, default=Path("."), help="output directory")
    p.add_argument("--seed", type=int, default=0, help="random seed")
    p.add_argument("--threads", type=int, default=1, help="solver worker threads (ignored on the GPU)")
    p.add_argument("--nominal-prices", action="store_true",
                   help="ignore price uncertainty (certainty-equivalent prices)")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="watermpc",
                                     description="Scenario-based stochastic MPC for flow-based water networks (B200)")
    sub = parser.add_subparsers(dest="command", required=True)
    pv = sub.add_parser("validate", help="check documents and their cross-consistency")
    for name in ("network", "tree", "forecast", "config", "state"):
        pv.add_argument(f"--{name}", type=Path)
    _common(pv)
    ps = sub.add_parser("solve", help="compute one control action")
    for name in ("network", "tree", "forecast", "config", "state"):
        ps.add_argument(f"--{name}", type=Path, required=True)
    _common(ps)
    return parser


def _cmd_validate(args) -> int:
    """Load every given document, collecting (not raising) their errors, then the
    tree invariants and the cross-document checks; exit 0 clean, 1 with
    problems, 2 when no document is given."""
    problems: list[str] = []
    given = [p for p in (args.network, args.tree, args.forecast, args.config, args.state) if p is not None]
    if not given:
        print("error: no documents given", file=sys.stderr)
        return 2

    def load(path, loader):
        if path is None:
            return None
        try:
            return loader(path)
        except (wio.SchemaError, OSError) as exc:
            problems.append(f"{path}: {exc}")
            return None

    model = load(args.network, wio.load_network)
    tree = load(args.tree, wio.load_tree)
    forecast = load(args.forecast, wio.load_forecast)
    cfg = load(args.config, wio.load_controller_config)
    state = load(args.state, wio.load_state)
    horizon, weights = (cfg[0], cfg[1]) if cfg is not None else (None, None)
    if tree is not None:
        problems.extend(validate_tree(tree))
    problems.extend(wio.cross_validate(model=model, tree=tree, forecast=forecast, horizon=horizon,
                                       weights=weights, state=state))
    for line in problems:
        print(line, file=sys.stderr)
    print("ok" if not problems else f"{len(problems)} problem(s) found")
    return 1 if problems else 0


def _cmd_solve(args) -> int:
    model = wio.load_network(args.network)
    tree = wio.load_tree(args.tree)
    forecast = wio.load_forecast(args.forecast)
    horizon, weights, cfg = wio.load_controller_config(args.config)
    x, u_prev, k = wio.load_state(args.state)
    issues = wio.cross_validate(model=model, tree=tree, forecast=forecast, horizon=horizon, weights=weights,
                                state=(x, u_prev, k))
    if issues:
        for line in issues:
            print(line, file=sys.stderr)
        return 1
    if args.nominal_prices:
        tree = zero_price_errors(tree)
    if not tree.is_attached:
        tree = attach_forecast(tree, forecast.d_hat, forecast.alpha_hat)
    instance = assemble_problem(model, tree, weights, x, u_prev, k)
    cfg = replace(cfg, threads=args.threads)
    try:
        result = solve_instance(instance, cfg)
    except RuntimeError as exc:
        print(f"solver failed: {exc}", file=sys.stderr)
        return 1
    args.out.mkdir(parents=True, exist_ok=True)
    wio.save_control_output(result, args.out / "controlOutput.json")
    print(f"iters={result.iterations} residual={result.primal_residual:.6e} "
          f"time_ms={result.solve_time_s * 1e3:.3f}")
    return 0


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    handler = {"validate": _cmd_validate, "solve": _cmd_solve}[args.command]
    try:
        return handler(args)
    except wio.SchemaError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
