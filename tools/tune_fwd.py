"""Interleaved A/B timing of tensor-core path settings on the C2 workload.

Profiling aid (not part of the product): each setting is a set of DASMC_* tuning
environment variables; settings are run round-robin `--rounds` times in one
process so that box-to-box clock differences cancel.  Prints, per setting, the
median fused-forward ms per launch, weight-gradient ms per launch and step ms.

  python tools/tune_fwd.py "DASMC_TC_CLUSTER=1" "DASMC_TC_CLUSTER=1 DASMC_TC_HINTA=1"
  python tools/tune_fwd.py "PREC=tf32h" "PREC=tf32h LIB=_exp/variant.so"   # code A/B
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("settings", nargs="+")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--precision", default="tf32")
    ap.add_argument("--config", default="c2", help="bench.py workload (MLP configs)")
    args = ap.parse_args()
    import torch
    import paper_2601_21983_b200 as p
    from paper_2601_21983_b200 import _lib as L

    w = bench.WORKLOADS[args.config]
    lib = p.load()
    spec, X, y = bench.make_data(w)
    J, S, N = w["J"], w["S"], w["n"]
    k0 = w["k0"]
    M = bench.window(w, k0)
    kc = p.KernelConfig.hmc(w["h"], S)
    res = {s: [] for s in args.settings}
    base_env = dict(os.environ)
    for _ in range(args.rounds):
        for s in args.settings:
            os.environ.clear()
            os.environ.update(base_env)
            prec, lib_path = args.precision, None
            for kv in s.split():
                k, v = kv.split("=", 1)
                if k == "PREC":  # precision mode of this setting
                    prec = v
                elif k == "LIB":  # a second build of the library (A/B of code variants)
                    lib_path = os.path.abspath(v)
                else:
                    os.environ[k] = v
            t = None
            try:
                t = p.GpuEnsembleTarget(spec, X, y, J, device=0, precision=prec, lib_path=lib_path)
                lib = t.lib
                L.check(lib.dasmc_gpu_reserve_rows(t.h, M))
                t.set_target(0, M, N, "scaled", 1.0, 1.0)
                L.check(lib.dasmc_gpu_init_ensemble_at(t.h, J, 0, 0))
                for _ in range(2):
                    t.smc_step(kc, 0, "systematic", 0.5)
                t.sync_records(0)
                stream = torch.cuda.ExternalStream(lib.dasmc_gpu_stream(t.h))
                torch.cuda.synchronize()
                L.check(lib.dasmc_gpu_set_timing(t.h, 1))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.steps):
                    t.smc_step(kc, 0, "systematic", 0.5)
                e1.record(stream)
                e1.synchronize()
                kms = np.zeros(3)
                kcnt = np.zeros(3, dtype=np.int64)
                L.check(lib.dasmc_gpu_kernel_times(t.h, kms.ctypes.data_as(L._D), kcnt.ctypes.data_as(L._I64)))
                L.check(lib.dasmc_gpu_set_timing(t.h, 0))
                t.sync_records(0)
                res[s].append((kms[0] / max(kcnt[0], 1), kms[1] / max(kcnt[1], 1), e0.elapsed_time(e1) / args.steps))
                t.close()
                del t
                torch.cuda.synchronize()
            except Exception as e:  # a variant that cannot run: report and go on
                print(f"{s}: FAILED {e}", flush=True)
                if t is not None:
                    t.close()
    os.environ.clear()
    os.environ.update(base_env)
    for s, v in res.items():
        if not v:
            continue
        f = statistics.median(x[0] for x in v)
        d = statistics.median(x[1] for x in v)
        st = statistics.median(x[2] for x in v)
        print(f"{s:60s} fwd {f:7.2f} ms  dW1 {d:7.2f} ms  step {st:8.2f} ms   all fwd: "
              + " ".join(f"{x[0]:.2f}" for x in v), flush=True)


if __name__ == "__main__":
    main()
