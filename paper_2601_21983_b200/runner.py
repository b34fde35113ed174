"""run_experiment driver with the reference's config and trace formats (runner.hpp:105-617).

``parse_config`` / ``config_to_json`` / ``write_trace`` / ``strip_timing`` restate the
reference's JSON config schema (runner.hpp:105-326), its canonical echo and the
``# dasmc trace v1`` text format (runner.hpp:374-448), so traces from this build can be
diffed against the reference's (numerically: fp32 values are not ``%.12g``-identical to
fp64).  ``run`` is the hot loop of runner.hpp:453-617 on one B200 through the C-ABI:
shuffle with fork(kPermutation), ``context_for`` (schedule / SDA / constant redraw),
``smc_step``, ``sda_advance`` on the post-step ensemble, ``evaluate_predictive`` every
``eval_every`` iterations, and the trace.  The ``linear_gaussian`` model stays in the CPU
oracle; it is rejected here with a ConfigError.

  python -m paper_2601_21983_b200 run config.json [--precision tf32] [--device 0]
  python -m paper_2601_21983_b200 strip-timing trace.txt
"""
from __future__ import annotations

import ctypes as C
import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .api import (GpuEnsembleTarget, KernelConfig, NetSpec, ScheduleConfig, batch_size, load_idx, sda_advance_with,
                  sda_init, shuffle_permutation, redraw_rows)


class ConfigError(ValueError):
    """runner.hpp:27-30."""


_CONFIG_KEYS = {"dataset", "model", "prior", "kernel", "schedule", "particles", "iterations", "seed", "eval_every",
                "output", "threads", "resample_fraction"}
_DATASET_KEYS = {"kind", "train_images", "train_labels", "test_images", "test_labels", "train_limit", "test_limit",
                 "n", "test_n", "noise", "dim"}


def _check_keys(obj, where, allowed):  # runner.hpp:82-93
    if not isinstance(obj, dict):
        raise ConfigError(f"{where}: must be an object")
    for k in obj:
        if k not in allowed:
            raise ConfigError(f'{where}: unknown key "{k}"')


def _require(obj, where, key):
    if key not in obj:
        raise ConfigError(f'{where}: missing required key "{key}"')
    return obj[key]


@dataclass
class RunConfig:  # runner.hpp:57-70
    dataset: dict = field(default_factory=dict)
    model: dict = field(default_factory=dict)
    prior_sigma: float = 1.0
    kernel: dict = field(default_factory=dict)
    schedule: dict = field(default_factory=dict)
    particles: int = 128
    iterations: int = 1
    seed: int = 0
    eval_every: int = 10
    output: str = ""
    threads: int = 1
    resample_fraction: float = 0.5


def parse_config(text: str) -> RunConfig:  # runner.hpp:105-247
    try:
        root = json.loads(text)
    except json.JSONDecodeError as err:
        raise ConfigError(f"config is not valid JSON: {err}") from None
    _check_keys(root, "config", _CONFIG_KEYS)
    cfg = RunConfig()
    ds = _require(root, "config", "dataset")
    _check_keys(ds, "dataset", _DATASET_KEYS)
    kind = _require(ds, "dataset", "kind")
    d = {"kind": kind}
    if kind == "idx":
        d["train_images"] = _require(ds, "dataset", "train_images")
        d["train_labels"] = _require(ds, "dataset", "train_labels")
        d["test_images"] = ds.get("test_images", "")
        d["test_labels"] = ds.get("test_labels", "")
        if (d["test_images"] == "") != (d["test_labels"] == ""):
            raise ConfigError("dataset: test_images and test_labels must be given together")
    elif kind in ("gaussian_blobs", "two_moons", "linear_gaussian"):
        d["n"] = int(_require(ds, "dataset", "n"))
        if d["n"] < 2:
            raise ConfigError("dataset.n: must be >= 2")
        d["noise"] = float(ds.get("noise", 0.1))
        d["dim"] = int(ds.get("dim", 2))
        d["test_n"] = int(ds.get("test_n", 0))
    else:
        raise ConfigError(f'dataset.kind: unknown kind "{kind}"')
    d["train_limit"] = int(ds.get("train_limit", 0))
    d["test_limit"] = int(ds.get("test_limit", 0))
    cfg.dataset = d

    model = _require(root, "config", "model")
    _check_keys(model, "model", {"kind", "layers", "activation", "noise_std", "dim"})
    mk = _require(model, "model", "kind")
    if mk == "mlp":
        layers = [int(v) for v in _require(model, "model", "layers")]
        act = model.get("activation", "relu")
        if act not in ("relu", "tanh"):
            raise ConfigError('model.activation: must be "relu" or "tanh"')
        if len(layers) < 2:
            raise ConfigError("model.layers: NetSpec: need at least input and output layers")
        if min(layers) < 1:
            raise ConfigError("model.layers: NetSpec: layer sizes must be >= 1")
        cfg.model = {"kind": "mlp", "layers": layers, "activation": act}
    elif mk == "linear_gaussian":
        dim = int(_require(model, "model", "dim"))
        ns = float(_require(model, "model", "noise_std"))
        if dim < 1:
            raise ConfigError("model.dim: must be >= 1")
        if not ns > 0.0:
            raise ConfigError("model.noise_std: must be > 0")
        cfg.model = {"kind": "linear_gaussian", "dim": dim, "noise_std": ns}
    else:
        raise ConfigError(f'model.kind: unknown kind "{mk}"')

    if "prior" in root:
        _check_keys(root["prior"], "prior", {"sigma"})
        cfg.prior_sigma = float(root["prior"].get("sigma", 1.0))
        if not cfg.prior_sigma > 0.0:
            raise ConfigError("prior.sigma: must be > 0")

    kern = _require(root, "config", "kernel")
    _check_keys(kern, "kernel", {"kind", "step_size", "leapfrog_steps"})
    kk = _require(kern, "kernel", "kind")
    h = float(_require(kern, "kernel", "step_size"))
    S = int(kern.get("leapfrog_steps", 1))
    if kk not in ("hmc", "langevin"):
        raise ConfigError(f'kernel.kind: unknown kind "{kk}"')
    if not h > 0.0:
        raise ConfigError("kernel: KernelConfig: step_size must be > 0")
    if S < 1:
        raise ConfigError("kernel: KernelConfig: leapfrog_steps must be >= 1")
    if kk == "langevin" and S != 1:
        raise ConfigError("kernel: KernelConfig: langevin requires leapfrog_steps == 1")
    cfg.kernel = {"kind": kk, "step_size": h, "leapfrog_steps": S}

    sch = _require(root, "config", "schedule")
    _check_keys(sch, "schedule", {"kind", "initial_batch", "increment", "redraw_constant", "beta0", "entropy_step"})
    sk = _require(sch, "schedule", "kind")
    if sk not in ("constant", "full_batch", "ctr", "linear", "automated", "sda"):
        raise ConfigError(f'schedule.kind: unknown kind "{sk}"')
    s = {"kind": sk}
    if sk != "full_batch":
        s["initial_batch"] = int(_require(sch, "schedule", "initial_batch"))
        if s["initial_batch"] < 1:
            raise ConfigError("schedule.initial_batch: must be >= 1")
    else:
        s["initial_batch"] = int(sch.get("initial_batch", 0))
    s["increment"] = int(sch.get("increment", 0))
    if s["increment"] < 0:
        raise ConfigError("schedule.increment: must be >= 1")
    s["redraw_constant"] = bool(sch.get("redraw_constant", False))
    if s["redraw_constant"] and sk != "constant":
        raise ConfigError("schedule.redraw_constant: only valid for the constant schedule")
    s["beta0"] = float(sch.get("beta0", 0.1))
    if not (0.0 < s["beta0"] <= 1.0):
        raise ConfigError("schedule.beta0: must be in (0, 1]")
    s["entropy_step"] = float(sch.get("entropy_step", 1.0))
    cfg.schedule = s

    cfg.particles = int(root.get("particles", 128))
    if cfg.particles < 2:
        raise ConfigError("particles: must be >= 2")
    cfg.iterations = int(_require(root, "config", "iterations"))
    if cfg.iterations < 1:
        raise ConfigError("iterations: must be >= 1")
    cfg.seed = int(_require(root, "config", "seed"))
    cfg.eval_every = int(root.get("eval_every", 10))
    if cfg.eval_every < 1:
        raise ConfigError("eval_every: must be >= 1")
    cfg.output = str(root.get("output", ""))
    cfg.threads = int(root.get("threads", 1))
    if cfg.threads < 1:
        raise ConfigError("threads: must be >= 1")
    cfg.resample_fraction = float(root.get("resample_fraction", 0.5))
    if not (0.0 <= cfg.resample_fraction <= 1.0):
        raise ConfigError("resample_fraction: must be in [0, 1]")
    return cfg


def config_to_json(cfg: RunConfig) -> str:  # runner.hpp:251-326 (nlohmann::json: sorted keys, compact)
    d = cfg.dataset
    ds = {"kind": d["kind"]}
    if d["kind"] == "idx":
        ds["train_images"] = d["train_images"]
        ds["train_labels"] = d["train_labels"]
        if d.get("test_images"):
            ds["test_images"] = d["test_images"]
            ds["test_labels"] = d["test_labels"]
    else:
        ds["n"] = d["n"]
        ds["noise"] = d["noise"]
        if d["kind"] == "linear_gaussian":
            ds["dim"] = d["dim"]
        if d["test_n"] > 0:
            ds["test_n"] = d["test_n"]
    if d["train_limit"] > 0:
        ds["train_limit"] = d["train_limit"]
    if d["test_limit"] > 0:
        ds["test_limit"] = d["test_limit"]
    m = cfg.model
    model = ({"kind": "mlp", "layers": m["layers"], "activation": m["activation"]} if m["kind"] == "mlp"
             else {"kind": "linear_gaussian", "dim": m["dim"], "noise_std": m["noise_std"]})
    s = cfg.schedule
    sched = {"kind": s["kind"]}
    if s["initial_batch"] > 0:
        sched["initial_batch"] = s["initial_batch"]
    if s["increment"] > 0:
        sched["increment"] = s["increment"]
    if s["redraw_constant"]:
        sched["redraw_constant"] = True
    if s["kind"] == "sda":
        sched["beta0"] = s["beta0"]
        sched["entropy_step"] = s["entropy_step"]
    root = {"dataset": ds, "model": model, "prior": {"sigma": cfg.prior_sigma},
            "kernel": {"kind": cfg.kernel["kind"], "step_size": cfg.kernel["step_size"],
                       "leapfrog_steps": cfg.kernel["leapfrog_steps"]},
            "schedule": sched, "particles": cfg.particles, "iterations": cfg.iterations, "seed": cfg.seed,
            "eval_every": cfg.eval_every, "resample_fraction": cfg.resample_fraction}
    return json.dumps(root, sort_keys=True, separators=(",", ":"))


def _fmt(v: float) -> str:  # format_double: %.12g
    return "%.12g" % v


def write_trace(cfg: RunConfig, records, summary, status: str) -> str:  # runner.hpp:386-413
    out = ["# dasmc trace v1", "# config " + config_to_json(cfg),
           "# columns k\tbatch\tbeta\tess\tresampled\tmean_log_target\tsampler_ms\ttest_log_pred\ttest_acc"]
    for r in records:
        out.append("\t".join([str(r["k"]), str(r["batch"]), _fmt(r["beta"]), _fmt(r["ess"]),
                              "1" if r["resampled"] else "0", _fmt(r["mean_log_target"]), _fmt(r["sampler_ms"]),
                              _fmt(r["test_log_pred"]), _fmt(r["test_acc"])]))
    out.append(f"# summary iterations={len(records)} sampler_ms={_fmt(summary['sampler_ms'])} "
               f"total_ms={_fmt(summary['total_ms'])} final_ess={_fmt(summary['final_ess'])} "
               f"test_log_pred={_fmt(summary['test_log_pred'])} test_acc={_fmt(summary['test_acc'])}")
    out.append("# status " + status)
    return "\n".join(out) + "\n"


def strip_timing(trace: str) -> str:  # runner.hpp:417-448
    out = []
    for line in trace.split("\n")[:-1] if trace.endswith("\n") else trace.split("\n"):
        if line.startswith("# summary"):
            toks = [t for t in line.split() if not (t.startswith("sampler_ms=") or t.startswith("total_ms="))]
            out.append(" ".join(toks))
        elif line and line[0] != "#":
            cols = line.split("\t")
            out.append("\t".join(c for i, c in enumerate(cols) if i != 6))
        else:
            out.append(line)
    return "\n".join(out) + "\n"


def _synthetic(kind: str, n: int, noise: float, seed: int):
    if kind == "linear_gaussian":
        raise ConfigError("model: linear_gaussian runs in the CPU oracle only (DESIGN.md §9)")
    X = np.empty((n, 2), dtype=np.float32)
    y = np.empty(n, dtype=np.int32)
    L.check(L.load().dasmc_make_synthetic(0 if kind == "gaussian_blobs" else 1, n, noise, seed,
                                          X.ctypes.data_as(L._F), y.ctypes.data_as(L._I32)))
    return X, y


def run(cfg: RunConfig, precision: str = "fp32", device: int = 0):
    """runner.hpp:453-617 on one B200; returns (records, summary, trace)."""
    t_run = time.perf_counter()
    if cfg.model["kind"] != "mlp":
        raise ConfigError("model: linear_gaussian runs in the CPU oracle only (DESIGN.md §9)")
    d = cfg.dataset
    test = None
    if d["kind"] == "idx":
        Xtr, ytr, _ = load_idx(d["train_images"], d["train_labels"])
        if d.get("test_images"):
            Xte, yte, _ = load_idx(d["test_images"], d["test_labels"])
            test = (Xte, yte)
    else:
        X, y = _synthetic(d["kind"], d["n"] + d["test_n"], d["noise"], cfg.seed)
        if d["test_n"] > 0:
            test = (X[d["n"]:], y[d["n"]:])
        Xtr, ytr = X[:d["n"]], y[:d["n"]]
    perm = shuffle_permutation(cfg.seed, Xtr.shape[0])  # runner.hpp:486-489
    Xtr, ytr = np.ascontiguousarray(Xtr[perm]), np.ascontiguousarray(ytr[perm])
    if 0 < d["train_limit"] < Xtr.shape[0]:
        Xtr, ytr = Xtr[:d["train_limit"]], ytr[:d["train_limit"]]
    if test is not None and 0 < d["test_limit"] < test[0].shape[0]:
        test = (test[0][:d["test_limit"]], test[1][:d["test_limit"]])
    layers = cfg.model["layers"]
    if Xtr.shape[1] != layers[0]:
        raise ConfigError("model.layers: input size does not match dataset dimension")
    if int(ytr.max()) + 1 > layers[-1]:
        raise ConfigError("model.layers: output size smaller than the number of classes")
    n = Xtr.shape[0]
    s = cfg.schedule
    init = min(s["initial_batch"], n) if s["initial_batch"] > 0 else n
    inc = min(s["increment"], n) if s["increment"] > 0 else init
    sched = ScheduleConfig(s["kind"], init, inc, cfg.iterations, n)
    is_sda = s["kind"] == "sda"
    st = sda_init(sched, s["beta0"], s["entropy_step"]) if is_sda else None
    spec = NetSpec(layers, cfg.model["activation"])
    t = GpuEnsembleTarget(spec, Xtr, ytr, cfg.particles, device=device, precision=precision)
    kc = KernelConfig(cfg.kernel["step_size"], cfg.kernel["leapfrog_steps"], cfg.kernel["kind"])

    def context_for(k):  # runner.hpp:544-564
        if is_sda:
            t.set_rows(None)
            t.set_target(st.prefix_end, st.block_end, n, "sda", st.beta, cfg.prior_sigma)
            return st.block_end, st.beta
        if s["redraw_constant"]:
            t.set_rows(redraw_rows(cfg.seed, k, n, init))
            t.set_target(0, init, n, "scaled", 1.0, cfg.prior_sigma)
            return init, 1.0
        M = batch_size(sched, k)
        t.set_target(0, M, n, "scaled", 1.0, cfg.prior_sigma)
        return M, 1.0

    records, status = [], "complete"
    sampler_total = 0.0
    context_for(0)
    t.init_ensemble(cfg.particles, cfg.seed)
    try:
        for k in range(cfg.iterations):
            t0 = time.perf_counter()
            M, beta = context_for(k)
            r = t.smc_step(kc, cfg.seed, "multinomial", cfg.resample_fraction, sync=True)
            rec = {"k": r["k"], "batch": M, "beta": beta if is_sda else 1.0, "ess": r["ess"],
                   "resampled": r["resampled"], "mean_log_target": r["mean_log_target"],
                   "test_log_pred": math.nan, "test_acc": math.nan}
            if is_sda and not st.terminal:  # sda_advance on the post-step ensemble (runner.hpp:592)
                m6 = t.sda_moments(st.prefix_end, st.block_end)
                st = sda_advance_with(sched, st, m6)
            rec["sampler_ms"] = 1e3 * (time.perf_counter() - t0)
            sampler_total += rec["sampler_ms"]
            if test is not None and ((k + 1) % cfg.eval_every == 0 or k + 1 == cfg.iterations):
                rec["test_log_pred"], rec["test_acc"] = t.evaluate_predictive(*test)
            records.append(rec)
    except L.SamplerError as err:
        status = f"incomplete: {err}"
    _, lw, _ = t.get_ensemble(cfg.particles)
    w = np.exp(lw - lw.max()) if np.isfinite(lw.max()) else np.zeros_like(lw)
    final_ess = float(1.0 / np.sum((w / w.sum()) ** 2)) if w.sum() > 0 else math.nan
    summary = {"sampler_ms": sampler_total, "total_ms": 1e3 * (time.perf_counter() - t_run), "final_ess": final_ess,
               "test_log_pred": records[-1]["test_log_pred"] if records else math.nan,
               "test_acc": records[-1]["test_acc"] if records else math.nan}
    t.close()
    trace = write_trace(cfg, records, summary, status)
    if cfg.output:
        with open(cfg.output, "w") as f:
            f.write(trace)
    if status != "complete":
        raise L.SamplerError(L.DASMC_EDEAD, status)
    return records, summary, trace
