"""CUDA-graph replay of smc_step (dasmc_gpu_set_graphs; SURVEY.md §7 hard part 7): the step's
kernels read the iteration, record slot and resampling stream key from device memory, so one
instantiated graph per step signature replays every iteration.  Replayed steps must be
bit-identical to eager launches (smc.hpp:109-158), across window changes (new signatures),
the three-buffer rotation, resampling on / off, and set_ensemble."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(product, spec, X, y, prec, graphs, windows, mode="scaled", kind="systematic", always=False, J=64):
    t = product.GpuEnsembleTarget(spec, X, y, J, precision=prec)
    if graphs:
        t.set_graphs(True)
    n = X.shape[0]
    P0, M0 = windows[0]
    t.set_target(P0, M0, n, mode, 0.4 if mode == "sda" else 1.0, 1.0)
    t.init_ensemble(J, 21)
    cfg = product.KernelConfig.hmc(0.002, 3)
    recs = []
    for k, (P, M) in enumerate(windows):
        t.set_target(P, M, n, mode, 0.4 if mode == "sda" else 1.0, 1.0)
        if k % 4 == 3:  # asynchronous steps in between, as bench.py drives them
            t.smc_step(cfg, 21, kind, 0.5, always=always, sync=False)
            recs.append(t.sync_records(1)[0])
        else:
            recs.append(t.smc_step(cfg, 21, kind, 0.5, always=always))
        if k == 7:  # set_ensemble mid-run: the replay must pick up the new positions
            th, lw, it = t.get_ensemble(J, dtype=np.float32)
            t.set_ensemble(th, lw, it)
    th, lw, it = t.get_ensemble(J)
    t.close()
    return recs, th, lw, it


@pytest.mark.parametrize("prec,mode,kind,always", [("f16x2", "scaled", "systematic", False),
                                                   ("fp32", "sda", "multinomial", True),
                                                   ("tf32h", "scaled", "multinomial", False)])
def test_graph_replay_bit_identical(product, prec, mode, kind, always):
    spec = product.NetSpec([64, 32, 10], "tanh")
    X, y = product.make_teacher_data(spec, 2000, 0, 0, 1, threads=8)
    # the C1 constant-to-refine pattern: 200 rows, then the whole set (two signatures)
    windows = [(50, 200)] * 9 + [(50, 2000)] * 6 if mode == "sda" else [(0, 200)] * 9 + [(0, 2000)] * 6
    a = _run(product, spec, X, y, prec, False, windows, mode, kind, always)
    b = _run(product, spec, X, y, prec, True, windows, mode, kind, always)
    for ra, rb in zip(a[0], b[0]):
        assert {k: v for k, v in ra.items() if k != "sampler_ms"} == {k: v for k, v in rb.items() if k != "sampler_ms"}
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and a[3] == b[3] == len(windows)


def test_graph_replay_c2_shape(product):
    """The one-hidden-layer tensor-core path at the C2 shape (CTA-pair cluster launches of the
    fused forward, TMA descriptors as kernel parameters) replays bit-identically too."""
    spec = product.NetSpec([784, 200, 10], "relu")
    X, y = product.make_teacher_data(spec, 1200, 1, 0, 2, threads=8)
    windows = [(0, 512)] * 5 + [(0, 1024)] * 4
    a = _run(product, spec, X, y, "f16x2", False, windows, J=96)
    b = _run(product, spec, X, y, "f16x2", True, windows, J=96)
    for ra, rb in zip(a[0], b[0]):
        assert {k: v for k, v in ra.items() if k != "sampler_ms"} == {k: v for k, v in rb.items() if k != "sampler_ms"}
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
