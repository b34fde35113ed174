"""CPU: the run_experiment config / trace surface (runner.hpp:105-448) and the host
data generators the runner uses (dataset.hpp:208-267)."""
import json
import math

import numpy as np
import pytest

CFG = {"dataset": {"kind": "two_moons", "n": 400, "noise": 0.1, "test_n": 100},
       "model": {"kind": "mlp", "layers": [2, 8, 2], "activation": "tanh"},
       "kernel": {"kind": "hmc", "step_size": 0.01, "leapfrog_steps": 2},
       "schedule": {"kind": "linear", "initial_batch": 100, "increment": 50},
       "particles": 16, "iterations": 5, "seed": 3, "eval_every": 2}


def test_parse_config_and_canonical_json(product):
    from paper_2601_21983_b200 import runner
    cfg = runner.parse_config(json.dumps(CFG))
    canon = runner.config_to_json(cfg)
    # nlohmann::json dump: sorted keys, compact; defaults made explicit
    assert canon.startswith('{"dataset":{"kind":"two_moons","n":400,"noise":0.1,"test_n":100},"eval_every":2')
    again = runner.parse_config(canon)
    assert runner.config_to_json(again) == canon
    for bad, msg in ((dict(CFG, bogus=1), 'unknown key "bogus"'),
                     (dict(CFG, schedule={"kind": "ctr"}), "initial_batch"),
                     (dict(CFG, schedule={"kind": "ctr", "initial_batch": 5, "redraw_constant": True}),
                      "redraw_constant"),
                     (dict(CFG, kernel={"kind": "langevin", "step_size": 0.1, "leapfrog_steps": 2}), "langevin"),
                     (dict(CFG, particles=1), "particles"),
                     (dict(CFG, resample_fraction=1.5), "resample_fraction")):
        with pytest.raises(runner.ConfigError, match=msg):
            runner.parse_config(json.dumps(bad))
    with pytest.raises(runner.ConfigError, match="not valid JSON"):
        runner.parse_config("{")


def test_trace_format_and_strip_timing(product):
    from paper_2601_21983_b200 import runner
    cfg = runner.parse_config(json.dumps(CFG))
    recs = [{"k": 0, "batch": 100, "beta": 1.0, "ess": 12.5, "resampled": True, "mean_log_target": -3.25,
             "sampler_ms": 1.5, "test_log_pred": math.nan, "test_acc": math.nan}]
    summ = {"sampler_ms": 1.5, "total_ms": 9.0, "final_ess": 16.0, "test_log_pred": math.nan, "test_acc": math.nan}
    tr = runner.write_trace(cfg, recs, summ, "complete")
    lines = tr.splitlines()
    assert lines[0] == "# dasmc trace v1" and lines[1].startswith("# config {")
    assert lines[3] == "0\t100\t1\t12.5\t1\t-3.25\t1.5\tnan\tnan"
    st = runner.strip_timing(tr).splitlines()
    assert st[3] == "0\t100\t1\t12.5\t1\t-3.25\tnan\tnan"
    assert st[4] == "# summary iterations=1 final_ess=16 test_log_pred=nan test_acc=nan"


def test_host_synthetic_matches_oracle(product, oracle):
    from paper_2601_21983_b200 import runner
    for kind, k in (("gaussian_blobs", 0), ("two_moons", 1)):
        X, y = runner._synthetic(kind, 101, 0.2, 7)
        Xo, yo, _ = oracle.make_synthetic(k, 101, 0.2, 7)
        assert np.array_equal(y, yo) and np.array_equal(X, Xo.astype(np.float32))
