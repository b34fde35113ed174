"""bench.py -- SMC-with-data-annealing hot path on B200.

A "step" is one SMC iteration (smc_step: fresh momenta, S+1 gradient
evaluations of the annealed-window log target for every particle, leapfrog,
incremental weights, normalise/ESS, resampling, gather) of BASELINE.json
configs[1] (C2: MLP 784-200-10 ReLU, J = 1024, 60000 synthetic 28x28 k/255
images with teacher labels, mini-batch 1000, +1 MB every 5 iterations,
HMC S = 3, h = 0.002), run at the schedule's iterations k0 .. k0+W+K-1.

metric = particle-sample grad evals/sec = sum_k J (S+1) M_k / time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU (torchrun): one particle-sharded ensemble of J = 1024 x N (weak
scaling): NCCL all-gather of the log-weights, redundant resampling indices,
point-to-point particle migration (paper_2601_21983_b200/dist.py).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]
    "c2": dict(layers=[784, 200, 10], act="relu", n=60000, J=1024, feature_kind=1, mb=1000, period=5, K=300,
               S=3, h=0.002, k0=150, cfg_id=2,
               desc="C2: MLP 784-200-10 ReLU, J=1024 particles, n=60000 synthetic 28x28x1 k/255 teacher-labelled, "
                    "MB=1000 (+1 MB every 5 iterations, 300 iterations), HMC S=3 h=0.002, prior N(0,1)"),
    # BASELINE.json configs[2]: CNN, SDA annealing; measured at a constant window of MB rows
    "c3": dict(layers=[512, 10], conv=((1, 28, 28), [(5, 16, True), (5, 32, True)]), act="relu", n=60000, J=512,
               feature_kind=1, mb=500, sda=True, K=200, S=3, h=0.002, k0=0, cfg_id=3, cpu_rows=48,
               desc="C3: CNN conv5x5x16-ReLU-pool-conv5x5x32-ReLU-pool-FC512-10 on 28x28x1 k/255 teacher-labelled, "
                    "J=512, MB=500, adaptive (SDA) annealing from the first MB (beta0=0.1, entropy step 1), "
                    "HMC S=3 h=0.002"),
    # BASELINE.json configs[3]: CNN on 32x32x3, constant-to-refine phase window
    "c4": dict(layers=[1600, 256, 10], conv=((3, 32, 32), [(3, 32, False), (3, 32, True), (3, 64, False),
                                                           (3, 64, True)]),
               act="relu", n=50000, J=256, feature_kind=1, mb=500, const_window=True, K=200, S=3, h=0.002, k0=0,
               cfg_id=4, cpu_rows=6,
               desc="C4: CNN conv3x3x32-conv3x3x32-pool-conv3x3x64-conv3x3x64-pool-FC256-10 (valid, ReLU) on 32x32x3 "
                    "U{0..255}/255, J=256, window M=500 (the CTR phase), HMC S=3 h=0.002"),
    # BASELINE.json configs[3]: the full-batch run (window = all 50000 images)
    "c4fb": dict(layers=[1600, 256, 10], conv=((3, 32, 32), [(3, 32, False), (3, 32, True), (3, 64, False),
                                                             (3, 64, True)]),
                 act="relu", n=50000, J=256, feature_kind=1, mb=50000, const_window=True, K=200, S=3, h=0.002, k0=0,
                 cfg_id=4, cpu_rows=6,
                 desc="C4: CNN conv3x3x32-conv3x3x32-pool-conv3x3x64-conv3x3x64-pool-FC256-10 (valid, ReLU) on "
                      "32x32x3 U{0..255}/255, J=256, full-batch window M=50000, HMC S=3 h=0.002"),
    # BASELINE.json configs[4] at J=1024 per GPU (the scaling sweep's per-GPU unit)
    "c5": dict(layers=[3072, 512, 512, 10], act="relu", n=50000, J=1024, feature_kind=0, mb=1000, const_window=True,
               K=100, S=3, h=0.002, k0=0, cfg_id=5,
               desc="C5: MLP 3072-512-512-10 ReLU, J=1024 per GPU, 50000 U[0,1]^3072 teacher-labelled, window "
                    "M=1000, resample every iteration, HMC S=3 h=0.002"),
    # BASELINE.json configs[0] (CPU-runnable case)
    "c1": dict(layers=[64, 32, 10], act="tanh", n=2000, J=128, feature_kind=0, mb=100, period=1, K=50, S=3,
               h=0.002, k0=0, cfg_id=1, ctr=(200, 40), big=False,
               desc="C1: MLP 64-32-10 tanh, J=128, n=2000 U[0,1]^64 teacher-labelled, CTR 2 MB -> 20 MB at it 40"),
}

DATA_DESC = "synthetic (teacher-labelled, seeded; BASELINE.json config shapes)"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# arithmetic of the dense contractions per --precision
DTYPES = {"fp32": "f32", "tf32": "tf32", "3xtf32": "3xtf32", "f16": "f16",
          "tf32h": "tf32 (forward), f16-stored operands in the weight-gradient GEMMs",
          "f16x2": "f16 MMAs: X f16 x W1 split f16 hi+lo (forward), f16-stored operands (weight gradients)"}


def window(w, k):
    if w.get("const_window") or w.get("sda"):  # SDA: the initial window (the schedule is adaptive)
        return w["mb"]
    if "ctr" in w:
        c0, sw = w["ctr"]
        return c0 if k < sw else w["n"]
    return min(w["mb"] * (1 + k // w["period"]), w["n"])


def algorithmic_flops_per_row(layers, conv=None):
    """F_grad = 4 sum_l MAC_l + 2 sum_{l>=2} MAC_l per datapoint (forward + dW + dX,
    no dX for the first layer); MAC_l = n_{l-1} n_l for a dense layer, outputs x cin k^2 for a conv."""
    macs = []
    if conv is not None:
        (c, h, w), stages = conv
        for k, co, pool in stages:
            h, w = h - k + 1, w - k + 1
            macs.append(h * w * co * c * k * k)
            if pool:
                h, w = h // 2, w // 2
            c = co
    macs += [layers[i - 1] * layers[i] for i in range(1, len(layers))]
    return 4 * sum(macs) + 2 * sum(macs[1:])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[2:6]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    try:
        return json.load(open(PEAKS_FILE))
    except Exception:
        return {}


def make_data(w):
    import paper_2601_21983_b200 as p
    spec = p.NetSpec(w["layers"], w["act"], w.get("conv"))
    X, y = p.make_teacher_data(spec, w["n"], w["feature_kind"], 0, w["cfg_id"], threads=os.cpu_count() or 8)
    perm = p.shuffle_permutation(0, w["n"])  # runner.hpp:486-489 (seed 0)
    return spec, np.ascontiguousarray(X[perm]), np.ascontiguousarray(y[perm])


def oracle_data(w):
    """The same teacher data and shuffle from the CPU oracle alone (the reference arm never
    loads the product library)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    layers = w["layers"] if "conv" not in w else O.cnn_layers(w["conv"][0], w["conv"][1], w["layers"])
    a = 0 if w["act"] == "relu" else 1
    X, y = O.make_teacher(layers, a, w["n"], w["feature_kind"], 0, w["cfg_id"], threads=os.cpu_count() or 8)
    perm = O.shuffle_perm(0, w["n"])
    return np.ascontiguousarray(X[perm].astype(np.float32)), np.ascontiguousarray(y[perm])


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_of(args, w, ks, Ms, world):
    """The workload description both arms print (same dict: the driver compares them)."""
    J = w["J"] if not getattr(args, "J_total", None) else -(-args.J_total // world)
    return {"workload": w["desc"], "particles_per_gpu": J, "particles_total": J * world if not getattr(args, "J_total", None)
            else args.J_total, "iterations": [ks[0], ks[-1]],
            "window_rows": [Ms[0], Ms[-1]], "precision": args.precision, "resample": args.resample,
            "l2": "inputs larger than L2 (activations >= 24 GB per step)" if w.get("big", True)
            else "inputs smaller than L2 (launch-bound config)",
            "parallelism": (f"one particle-sharded ensemble of J={J * world} over {world} GPUs "
                            "(NCCL all-gather of log-weights, P2P particle migration)"
                            if world > 1 else "single GPU")}


def cpu_sample(w, X, y, ks, threads, warm=0):
    """The CPU oracle (fp64 restatement of the reference, OpenBLAS dgemm, parallel_for
    over particles) on a bounded sample: one smc_step of `threads` particles per k, after
    `warm` untimed steps."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    O.use_blas(True)
    layers = w["layers"] if "conv" not in w else O.cnn_layers(w["conv"][0], w["conv"][1], w["layers"])
    a = 0 if w["act"] == "relu" else 1
    Jc = max(2, threads)
    X64 = X.astype(np.float64)
    # the CNN oracle is plain loops: its sample takes fewer window rows (per-unit rate)
    rows = lambda k: min(window(w, k), w.get("cpu_rows", 1 << 62))  # noqa: E731
    th, lw = O.init_ensemble(layers, a, X64, y, (0, rows(ks[0]), w["n"]), 0, 1.0, 1.0, 0, Jc, threads=threads)
    units, secs = 0.0, 0.0
    for i, k in enumerate([ks[0]] * warm + list(ks)):
        M = rows(k)
        t0 = time.perf_counter()
        th, lw, _, _, _ = O.smc_step(layers, a, X64, y, (0, M, w["n"]), 0, 1.0, 1.0, (w["h"], w["S"], 0), 0, 0.5, 1,
                                     False, th, lw, k, threads=threads, dumps=False)
        if i >= warm:
            secs += time.perf_counter() - t0
            units += Jc * (w["S"] + 1) * M
    return units, secs, Jc


def cpu_sample_desc(w, Jc, threads, nsteps):
    rows = f"min(window, {w['cpu_rows']}) rows" if "cpu_rows" in w else "the step's window"
    return (f"{nsteps} warm smc_step(s) of {Jc} particles at {rows} (CPU oracle: fp64 restatement of the "
            f"reference, OpenBLAS dgemm 1 thread x {threads} particle threads, {cpu_model()}); the per-unit rate "
            "extrapolates linearly in J (per-particle work is independent, parallel.hpp static partition); "
            "the reference itself is not buildable here (Eigen3 absent)")


def run_reference(args, w):
    """--impl reference: the reference's CPU path (the oracle port; the reference does not
    build without Eigen3) on this box's host cores, same metric / config as our arm.  Only
    the oracle is loaded (no product library)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    X, y = oracle_data(w)
    threads = os.cpu_count() or 1
    k0 = w["k0"]
    ks = [k0 + args.warmup + i for i in range(args.steps)]
    Ms = [window(w, k) for k in ks]
    units, secs, Jc = cpu_sample(w, X, y, ks, threads, warm=min(args.warmup, 1))
    v = units / secs
    line = {"impl": "reference", "metric": "particle-sample grad evals/sec", "value": v,
            "unit": "particle-sample grad evals/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA_DESC,
            "config": config_of(args, w, ks, Ms, world),
            "cpu_baseline": {"value": v, "unit": "particle-sample grad evals/s", "cores": threads, "kind": "port",
                             "cpu": cpu_model(), "sample": cpu_sample_desc(w, Jc, threads, args.steps)},
            "e2e": {"value": v, "unit": "particle-sample grad evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, w):
    import torch
    import paper_2601_21983_b200 as p
    from paper_2601_21983_b200 import _lib as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = p.load()
    spec, X, y = make_data(w)
    J, S, N = w["J"], w["S"], w["n"]
    D = p.param_count(spec)
    if args.J_total:
        J = (args.J_total + world - 1) // world
    t = p.GpuEnsembleTarget(spec, X, y, J, device=local, precision=args.precision)
    k0 = w["k0"]
    ks_warm = [k0 + i for i in range(args.warmup)]
    ks = [k0 + args.warmup + i for i in range(args.steps)]
    sda = bool(w.get("sda"))
    if sda:  # adaptive annealing (annealing.hpp:84-208): the window grows when the trigger fires
        sched = p.ScheduleConfig("sda", w["mb"], w["mb"], w["K"], N)
        st = [p.sda_init(sched, 0.1, 1.0)]
        # CNN windows are chunked: reserving n rows sizes the log-likelihood slots only
        L.check(lib.dasmc_gpu_reserve_rows(t.h, N))
    else:
        L.check(lib.dasmc_gpu_reserve_rows(t.h, max(window(w, k) for k in ks_warm + ks + [k0])))

    def target_of(k):
        if sda:
            s_ = st[0]
            return s_.prefix_end, s_.block_end, "sda", s_.beta
        return 0, window(w, k), "scaled", 1.0

    def advance():  # sda_advance on the post-step ensemble (runner.hpp:589-592)
        if sda and not st[0].terminal:
            s_ = st[0]
            st[0] = p.sda_advance_with(sched, s_, t.sda_moments(s_.prefix_end, s_.block_end))

    P0, M0, mode0, beta0 = target_of(k0)
    t.set_target(P0, M0, N, mode0, beta0, 1.0)
    # world > 1: one particle-sharded ensemble (paper_2601_21983_b200/dist.py) of J_total = J * world
    # (weak scaling) or, with --J-total, a fixed J_total split over the ranks (strong scaling,
    # BASELINE configs[4]'s fixed-J sweep); this rank owns global slots [j0, j0 + J)
    if args.J_total:
        from paper_2601_21983_b200.dist import shard_range
        J_total = args.J_total
        j0, j1 = shard_range(J_total, world, rank)
        J = j1 - j0
    else:
        J_total = J * world
        j0 = J * rank
    L.check(lib.dasmc_gpu_init_ensemble_at(t.h, J, 0, j0))
    th0, lw0, _ = t.get_ensemble(J, dtype=np.float32)
    t.set_ensemble(th0, lw0, k0)
    kc = p.KernelConfig.hmc(w["h"], S)
    rk = args.resample
    if world == 1 and not w.get("big", True) and not args.no_graphs:
        # launch-bound config (C1): CUDA-graph replay of each smc_step (bit-identical,
        # tests/test_gpu_graphs.py).  Not for the big configs: their kernel-range timers (the
        # live roofline) run on eager launches, and launch overhead is < 1 % of their step
        t.set_graphs(True)
    sharded_recs = []
    Ms = []
    if world > 1:
        from paper_2601_21983_b200.dist import GpuShardEngine, TorchComm, sharded_step
        engine, comm = GpuShardEngine(t), TorchComm(torch.device("cuda", local))

        def step(k, sync=False):
            Pk, Mk, mode, beta = target_of(k)
            t.set_target(Pk, Mk, N, mode, beta, 1.0)
            Ms.append(Mk)
            sharded_recs.append(sharded_step(engine, comm, J_total, kc, 0, rk, 0.5, False, torch.device("cuda", local)))
    else:
        def step(k, sync=False):
            Pk, Mk, mode, beta = target_of(k)
            t.set_target(Pk, Mk, N, mode, beta, 1.0)
            Ms.append(Mk)
            t.smc_step(kc, 0, rk, 0.5, sync=sync)
            advance()
    for k in ks_warm:
        step(k)
    if world == 1:
        t.sync_records(0)
    stream = torch.cuda.ExternalStream(lib.dasmc_gpu_stream(t.h)) if world == 1 else torch.cuda.current_stream()
    L.check(lib.dasmc_gpu_set_timing(t.h, 1))
    n_launch0 = lib.dasmc_launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sharded_recs.clear()
    Ms.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for k in ks:
            step(k)
        if world > 1:
            # the shard engine's kernels run on the library's stream: drain it before the closing event,
            # so the last step's unpack is inside the timed region
            torch.cuda.synchronize()
        e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = lib.dasmc_launch_count() - n_launch0
    recs = t.sync_records(len(ks)) if world == 1 else sharded_recs
    kms = np.zeros(3)
    kcnt = np.zeros(3, dtype=np.int64)
    L.check(lib.dasmc_gpu_kernel_times(t.h, kms.ctypes.data_as(L._D), kcnt.ctypes.data_as(L._I64)))
    L.check(lib.dasmc_gpu_set_timing(t.h, 0))
    units = float(sum(J * (S + 1) * M for M in Ms))
    ms_max = ms
    if dist:
        tt = torch.tensor([ms, units], device="cuda", dtype=torch.float64)
        mx = tt.clone()
        dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        ms_max, units_all = float(mx[0]), float(tt[1])
    else:
        units_all = units
    value = units_all / (ms_max / 1e3)

    # ---- e2e through the C-ABI with host (pinned) buffers, copies inside the timed region
    Ms_timed = list(Ms)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    th_h = torch.empty((J, D), dtype=torch.float32, pin_memory=True).numpy()
    lw_h = torch.empty(J, dtype=torch.float64, pin_memory=True).numpy()
    th_h[:] = th0
    lw_h[:] = lw0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_units = 0.0
    for i in range(e2e_steps):
        k = ks[i]
        t.set_ensemble(th_h, lw_h, k)  # H2D: theta (fp32, reference layout) + log-weights
        step(k, sync=True)
        L.check(lib.dasmc_gpu_get_ensemble_f32(t.h, th_h.ctypes.data_as(L._F), lw_h.ctypes.data_as(L._D), None))
        e2e_units += J * (S + 1) * Ms[-1]
    e2e_s = time.perf_counter() - t0
    Ms[:] = Ms_timed
    if dist:
        tt = torch.tensor([e2e_s, e2e_units], device="cuda", dtype=torch.float64)
        mx = tt.clone()
        dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        e2e_s, e2e_units = float(mx[0]), float(tt[1])
    e2e_value = e2e_units / e2e_s
    step_bytes = J * D * 4 + J * 8

    # ---- roofline of the dominant kernel (live CUDA-event timing on the context stream)
    n0, n1 = w["layers"][0], w["layers"][1]
    fl_fwd = sum(2.0 * M * n0 * n1 * J * (S + 1) for M in Ms)
    fl_dw = sum(2.0 * M * n0 * n1 * J * (S + 1) for M in Ms)
    kinds = [("layer-1 forward GEMM Z1 = X W1^T (+bias, ReLU epilogue)", fl_fwd, kms[0], kcnt[0]),
             ("layer-1 weight-gradient GEMM dW1 = delta1^T X (+fused leapfrog epilogue)", fl_dw, kms[1], kcnt[1])]
    name, fl, kt_ms, kc_n = max(kinds, key=lambda x: x[2])
    if kt_ms <= 0 or "conv" in w:
        # no per-GEMM timers on this path (CNN stages): the whole gradient evaluation
        fl = sum(float(algorithmic_flops_per_row(w["layers"], w.get("conv"))) * M * J * (S + 1) for M in Ms)
        name, kt_ms, kc_n = ("whole gradient evaluation (CNN stages on tcgen05 tf32 implicit GEMMs + CUDA-core head)"
                             if args.precision != "fp32" else
                             "whole gradient evaluation (CNN stages + MLP head, SIMT fp32)"), kms[2], kcnt[2]
    peaks = load_peaks()
    if args.precision == "fp32":
        peak = 148 * 128 * 2 * 1.965e9 / 1e12
        peak_src = "nominal fp32 CUDA-core FMA peak (148 SMs x 128 lanes x 2 x 1965 MHz); not in MEASURED_PEAKS.json"
    else:
        # the kernel is timed inside a long step: the sustained bf16 figure applies
        bf16 = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops", 1590.0)
        kind = "sustained" if peaks.get("bf16_tflops_sustained") else "burst"
        # dense rate of the MMAs this kernel issues per algorithmic MAC: kind::tf32 runs at half
        # the f16/bf16 rate; split modes issue 2 (f16x2 forward) or 3 (3xtf32) MMAs per MAC
        fwd = name.startswith("layer-1 forward")
        div, what = {"tf32": (2.0, "tf32"), "3xtf32": (6.0, "3xtf32 (3 tf32 MMAs per MAC)"),
                     "f16": (1.0, "f16"),
                     "f16x2": (2.0 if fwd else 1.0, "f16x2 (2 f16 MMAs per MAC)" if fwd else "f16"),
                     "tf32h": (2.0 if fwd else 1.0, "tf32" if fwd else "f16")}[args.precision]
        peak = bf16 / div
        peak_src = f"dense {what} = measured bf16 {kind} {bf16} TFLOP/s / {div:g} (MEASURED_PEAKS.json)"
    achieved = fl / (kt_ms / 1e3) / 1e12 if kt_ms > 0 else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            # per workload and precision: ncu dram bytes (read + write) per launch of the dominant kernel
            traffic = json.load(open(tf)).get(args.config, {}).get(args.precision)
        except Exception:
            traffic = None
    roof = {"bound": "tensor" if args.precision != "fp32" else "compute", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic, "kernel": name,
            "launches": int(kc_n), "kernel_ms_total": float(kt_ms), "peak_source": peak_src,
            "share_of_step": float(kt_ms / ms) if ms > 0 else None,
            "eval_ms_total": float(kms[2])}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        ncpu = 2
        cu, cs, Jc = cpu_sample(w, X, y, ks[:ncpu], threads, warm=1)
        cpu = {"value": cu / cs, "unit": "particle-sample grad evals/s", "cores": threads, "kind": "port",
               "cpu": cpu_model(), "sample": cpu_sample_desc(w, Jc, threads, min(ncpu, len(ks)))}
    if rank == 0:
        line = {"metric": "particle-sample grad evals/sec", "value": value, "unit": "particle-sample grad evals/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong" if args.J_total else "weak", "vs_baseline": None,
                "dtype": DTYPES.get(args.precision, args.precision),
                "data": DATA_DESC,
                "config": config_of(args, w, ks, Ms, world),
                "iterations_per_sec": args.steps / (ms_max / 1e3),
                "particle_grad_evals_per_sec": world * J * (S + 1) * args.steps / (ms_max / 1e3),
                "clocks": clk.summary(), "gpu_launches": int(launches), "roofline": roof,
                "e2e": {"value": e2e_value, "unit": "particle-sample grad evals/s",
                        "h2d_bytes_per_step": step_bytes, "d2h_bytes_per_step": step_bytes + 64,
                        "steps": e2e_steps},
                "cpu_baseline": cpu,
                "records_tail": [{k: r[k] for k in ("k", "ess", "resampled", "n_divergent")} for r in recs[-2:]]}
        print(json.dumps(line), flush=True)
    t.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default=None, choices=["fp32", "tf32", "tf32h", "f16x2", "3xtf32", "f16"],
                    help="default: tf32 where the tensor-core path applies (one-hidden-layer MLPs), else fp32")
    ap.add_argument("--resample", default="systematic", choices=["systematic", "multinomial"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--J", type=int, default=None, help="particles per GPU (default: the config's)")
    ap.add_argument("--J-total", type=int, default=None,
                    help="fixed ensemble size split over the GPUs (strong scaling; C5's J sweep)")
    args = ap.parse_args()
    w = dict(WORKLOADS[args.config])
    if args.J:
        w["J"] = args.J
        w["desc"] = w["desc"].replace(f"J={WORKLOADS[args.config]['J']}", f"J={args.J}")
    if args.precision is None:
        # one hidden layer: tf32 forward + fp16-stored weight-gradient operands (tf32h, same
        # 11-bit significand, tolerance of the tf32 path); deep MLPs: tf32 chain; CNNs: fp32
        tc1 = "conv" not in w and len(w["layers"]) == 3 and w["layers"][1] <= 256 and w["layers"][2] <= 16
        deep = "conv" not in w and len(w["layers"]) > 3 and w["layers"][-1] <= 16
        # one hidden layer: f16x2 (fp16 X times [W1, b1] split into fp16 hi + lo; the most accurate
        # tensor-core mode within ~3 % of the fastest at the benched window:
        # tests/test_gpu_bench_window.py)
        args.precision = "f16x2" if tc1 else "tf32"  # deep MLPs: tf32 chain; CNNs: tf32 conv stages
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
