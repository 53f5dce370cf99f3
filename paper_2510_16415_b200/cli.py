"""`python -m paper_2510_16415_b200 train ...` — the reference's `faultsim train`
(reference pkg/src/faultsim/cli.py:36-165) on the B200 engine.

Only the step path's subcommand is provided: `train` writes metrics.csv,
events.jsonl and final_weights.bin/.json into --out, with the reference's exit
codes: 0 ok, 2 config error, 3 numerical failure, 4 unrecoverable cluster.
The cost-model, probe and plotting subcommands are out of scope.
"""

from __future__ import annotations

import argparse
import json
import sys

from . import harness
from .errors import ConfigError, NumericalFailure, UnrecoverableRankError

EXIT_OK, EXIT_CONFIG, EXIT_NUMERICAL, EXIT_UNRECOVERABLE = 0, 2, 3, 4


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="mecefo-b200", description="MeCeFO degraded-step training on B200")
    sub = p.add_subparsers(dest="command", required=True)
    t = sub.add_parser("train", help="run the fault-tolerant training loop")
    t.add_argument("--config", type=str, default=None, help="JSON config file (reference schema)")
    t.add_argument("--seed", type=int, default=None, help="override the run seed")
    t.add_argument("--out", type=str, default=None, help="output directory")
    t.add_argument("--quiet", action="store_true", help="suppress progress output")
    t.add_argument("--precision", choices=["fp32", "bf16"], default="fp32", help="engine compute precision")
    return p


def load_run_config(args) -> harness.RunConfig:
    """cli.py:22-31: --seed also reseeds the failure stream to seed*31+7."""
    cfg = harness.load_config(args.config) if args.config is not None else harness.config_from_dict({})
    if args.seed is not None:
        cfg.run.seed = args.seed
        cfg = harness.replace_scenario_seed(cfg, args.seed * 31 + 7)
    return cfg


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        cfg = load_run_config(args)
        result = harness.run_training(cfg, out_dir=args.out, quiet=args.quiet, precision=args.precision)
        if not args.quiet:
            print(json.dumps(result.summary, indent=2))
        return EXIT_OK
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except NumericalFailure as exc:
        print(f"numerical failure: {exc}", file=sys.stderr)
        return EXIT_NUMERICAL
    except UnrecoverableRankError as exc:
        print(f"unrecoverable cluster: {exc}", file=sys.stderr)
        return EXIT_UNRECOVERABLE


if __name__ == "__main__":
    sys.exit(main())
