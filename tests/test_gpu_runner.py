"""GPU: the run_experiment driver with the reference's config / trace surface
(paper_2601_21983_b200/runner.py, runner.hpp:453-617) against the oracle's hot loop."""
import json
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = {"dataset": {"kind": "two_moons", "n": 400, "noise": 0.1, "test_n": 100},
       "model": {"kind": "mlp", "layers": [2, 8, 2], "activation": "tanh"},
       "kernel": {"kind": "hmc", "step_size": 0.01, "leapfrog_steps": 2},
       "schedule": {"kind": "linear", "initial_batch": 100, "increment": 50},
       "particles": 16, "iterations": 5, "seed": 3, "eval_every": 2}


def test_runner_matches_oracle_loop(product, oracle):
    from paper_2601_21983_b200 import runner
    cfg = runner.parse_config(json.dumps(CFG))
    recs, summary, trace = runner.run(cfg)
    X, y = runner._synthetic("two_moons", 500, 0.1, 3)
    o = oracle.run([2, 8, 2], 1, X[:400].astype(np.float64), y[:400], kernel=(0.01, 2, 0), sched=(3, 100, 50, 1, -1),
                   particles=16, iterations=5, seed=3, resample_kind=0)
    assert [r["batch"] for r in recs] == [r["batch"] for r in o]
    for a, b in zip(recs, o):
        np.testing.assert_allclose(a["ess"], b["ess"], rtol=1e-3)
        np.testing.assert_allclose(a["mean_log_target"], b["mean_log_target"], rtol=1e-4)
    evals = [r for r in recs if not np.isnan(r["test_acc"])]
    assert [r["k"] for r in evals] == [1, 3, 4] and all(0 <= r["test_acc"] <= 100 for r in evals)
    assert trace.splitlines()[-1] == "# status complete"


def test_cli_run_and_strip_timing(product, tmp_path):
    cfgp, out = tmp_path / "cfg.json", tmp_path / "trace.txt"
    cfgp.write_text(json.dumps(dict(CFG, output=str(out))))
    r = subprocess.run([sys.executable, "-m", "paper_2601_21983_b200", "run", str(cfgp)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    tr = out.read_text()
    assert tr.startswith("# dasmc trace v1") and len([l for l in tr.splitlines() if not l.startswith("#")]) == 5
    s = subprocess.run([sys.executable, "-m", "paper_2601_21983_b200", "strip-timing", str(out)], capture_output=True,
                       text=True, timeout=60)
    assert s.returncode == 0 and "sampler_ms=" not in s.stdout and "final_ess=" in s.stdout
