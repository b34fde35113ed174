"""Command line (the reference's dasmc CLI surface over runner.hpp's config / trace):

  python -m paper_2601_21983_b200 run CONFIG.json [--precision fp32|tf32|3xtf32|f16] [--device N] [--output PATH]
  python -m paper_2601_21983_b200 strip-timing TRACE
"""
import argparse
import sys

from . import runner


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2601_21983_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="run a config (runner.hpp run_experiment) and write its trace")
    r.add_argument("config")
    r.add_argument("--precision", default="fp32", choices=["fp32", "tf32", "3xtf32", "f16"])
    r.add_argument("--device", type=int, default=0)
    r.add_argument("--output", default=None, help="trace path (default: the config's output, else stdout)")
    s = sub.add_parser("strip-timing", help="print a trace without its wall-time fields")
    s.add_argument("trace")
    a = ap.parse_args(argv)
    if a.cmd == "strip-timing":
        sys.stdout.write(runner.strip_timing(open(a.trace).read()))
        return 0
    try:
        cfg = runner.parse_config(open(a.config).read())
    except runner.ConfigError as err:
        print(f"config error: {err}", file=sys.stderr)
        return 2
    if a.output is not None:
        cfg.output = a.output
    _, summary, trace = runner.run(cfg, precision=a.precision, device=a.device)
    if not cfg.output:
        sys.stdout.write(trace)
    print(f"final_ess={summary['final_ess']:.6g} test_log_pred={summary['test_log_pred']:.6g} "
          f"test_acc={summary['test_acc']:.6g}", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
