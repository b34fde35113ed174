"""Isolated HBM throughput of the step's memory-bound kernels:
resample gather, momentum sum of squares, momentum generation and the weights /
resampling kernel, on the context's own buffers at a BASELINE config's shape.

  python tools/membench.py [--config c2|c5] [--J 1024] [--reps 20]

The gather is driven by systematic indices of a non-degenerate weight vector
(log-weights ~ N(0, 1)), so its sources are distinct rows spread over HBM, not
one L2-resident particle (the C2 bench collapses to ESS ~ 1).  Prints one JSON
line: ms per launch, algorithmic bytes, GB/s and the fraction of the measured
HBM copy bandwidth (MEASURED_PEAKS.json)."""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_21983_b200 as p  # noqa: E402
from paper_2601_21983_b200 import _lib as L  # noqa: E402

CONFIGS = {"c2": ([784, 200, 10], "relu"), "c5": ([3072, 512, 512, 10], "relu")}
NAMES = ["gather", "p_sumsq", "normals", "weights_resample"]


def systematic(w, u):
    cdf = np.cumsum(w)
    pts = (np.arange(len(w)) + u) / len(w)
    return np.minimum(np.searchsorted(cdf, pts, side="right"), len(w) - 1).astype(np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--J", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    layers, act = CONFIGS[a.config]
    spec = p.NetSpec(layers, act)
    X = np.zeros((1024, layers[0]), np.float32)
    y = np.zeros(1024, np.int32)
    t = p.GpuEnsembleTarget(spec, X, y, a.J, precision="fp32")
    t.init_ensemble(a.J, 1)
    rng = np.random.default_rng(0)
    lw = rng.standard_normal(a.J)
    w = np.exp(lw - lw.max())
    w /= w.sum()
    idx = systematic(w, rng.random())
    ms = np.zeros(4)
    by = np.zeros(4)
    L.check(t.lib.dasmc_gpu_bench_memory(t.h, a.J, idx.ctypes.data_as(C.POINTER(C.c_int32)), a.reps,
                                         ms.ctypes.data_as(C.POINTER(C.c_double)),
                                         by.ctypes.data_as(C.POINTER(C.c_double))))
    t.close()
    peak = None
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    out = {"config": a.config, "J": a.J, "D": p.param_count(spec), "distinct_gather_sources": int(len(set(idx))),
           "hbm_peak_gbs": peak, "kernels": {}}
    for i, nm in enumerate(NAMES):
        gbs = by[i] / (ms[i] * 1e-3) / 1e9
        out["kernels"][nm] = {"ms": round(float(ms[i]), 5), "bytes": float(by[i]), "GB/s": round(gbs, 1),
                              "frac_hbm": round(gbs / peak, 3) if peak else None}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
