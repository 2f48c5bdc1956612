"""Command line of the solver (the reference's tools/main.cpp:8-65):

    python -m paper_2206_13164_b200 solve --config FILE [--solver euler|fs|nmg]
        [--order 1|2] [--levels auto|N] [--threads N] [--output DIR]

Loads the JSON scenario (scenario.load_config), applies the command-line
overrides, prints the configuration echo, runs the scenario on the GPU
(scenario.run_scenario) and prints the summary line.  Exit codes as the
reference's: 0 converged, 2 NonConvergence ("solver did not converge: ..."),
1 configuration / command-line / other errors.
"""
from __future__ import annotations

import argparse
import sys


class _ParseError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # command-line errors: exit code 1 (main.cpp:30-33)
        raise _ParseError(message)


def _order(text: str) -> int:
    v = int(text)
    if not 1 <= v <= 2:
        raise argparse.ArgumentTypeError(f"value {text} not in range [1 - 2]")
    return v


def _positive(text: str) -> int:
    v = int(text)
    if not v > 0:
        raise argparse.ArgumentTypeError(f"value {text} not a positive number")
    return v


def _parser() -> _Parser:
    app = _Parser(prog="momg", description="Steady-state moment-method solver for rarefied cavity flows")
    sub = app.add_subparsers(dest="command", parser_class=_Parser)
    sub.required = True
    solve = sub.add_parser("solve", help="Run a configured cavity scenario to steady state")
    solve.add_argument("--config", required=True, help="JSON scenario configuration file")
    solve.add_argument("--solver", choices=["euler", "fs", "nmg"], help="time iteration: euler, fs, or nmg")
    solve.add_argument("--order", type=_order, default=0, help="spatial reconstruction order")
    solve.add_argument("--levels", default="", help="grid levels: auto or a count")
    solve.add_argument("--threads", type=_positive, default=0, help="worker threads")
    solve.add_argument("--output", default="", help="output directory")
    return app


def main(argv=None) -> int:
    try:
        args = _parser().parse_args(argv)
    except _ParseError as e:
        print(f"momg: error: {e}", file=sys.stderr)
        return 1

    from . import scenario
    from .momg import ConfigError, NonConvergence
    try:
        config = scenario.load_config(args.config)
        if args.solver:
            config.solver = scenario.solver_kind_from_string(args.solver)
        if args.order != 0:
            config.space_order = args.order
        if args.levels:
            config.levels = scenario.levels_from_string(args.levels)
        if args.threads != 0:
            config.threads = args.threads
        if args.output:
            config.output_dir = args.output
        sys.stdout.write(scenario.config_echo(config))
        sys.stdout.flush()
        result = scenario.run_scenario(config)
        r = result.report
        print(f"converged in {r.iterations} iterations, final ratio {r.final_ratio:g}, {r.seconds:g} s, "
              f"{r.work} cell evaluations")
        print(f"wrote history.tsv, field.tsv, report.txt under {config.output_dir}")
        return 0
    except NonConvergence as e:
        print(f"solver did not converge: {e}", file=sys.stderr)
        return 2
    except ConfigError as e:
        print(f"configuration error: {e}", file=sys.stderr)
        return 1
    except Exception as e:  # noqa: BLE001 (main.cpp:60-62)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
