"""Generates tests/golden/golden.npz from the CPU oracle (oracle/pyoracle.py).

The reference ships no golden files: its known answers are the
inline KATs ported in oracle/oracle_tests.cpp.  These vectors freeze the
oracle's outputs once it passes those KATs, so that (a) any later change to
the oracle is caught on CPU and (b) the GPU parity tests have fixed targets.
Run:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as O  # noqa: E402


def main():
    g = {}
    # RNG streams (rng.hpp): fork keys, raw draws, normals, uniforms
    g["fork_keys"] = np.array([O.fork_key(s, a, b, c) for s in (0, 1, 42) for a in (1, 2, 3) for b in (0, 7)
                               for c in (0, 5)], dtype=np.uint64)
    k = O.fork_key(0, 2, 0, 0)
    g["u64"] = O.rng_u64(k, 64)
    g["normals"] = O.rng_normals(O.fork_key(3, 2, 1, 4), 256)
    g["uniforms"] = O.rng_uniforms(O.fork_key(3, 3, 9, 0), 256)
    # teacher data + shuffle
    X, y = O.make_teacher([8, 4, 3], 0, 50, 0, 11, 1)
    g["teacher_X"], g["teacher_y"] = X, y
    X1, y1 = O.make_teacher([12, 6, 4], 1, 40, 1, 11, 2)
    g["teacher_px_X"], g["teacher_px_y"] = X1, y1
    g["perm"] = O.shuffle_perm(0, 100)
    # value_and_grad on a C1-shaped MLP (64-32-10 tanh) over a 100-row window
    layers = [64, 32, 10]
    Xc, yc = O.make_teacher(layers, 1, 300, 0, 0, 1)
    D = O.param_count(layers)
    th = np.random.default_rng(0).standard_normal((4, D))
    for mode, win, beta, tag in ((0, (0, 100, 300), 1.0, "scaled"), (1, (60, 100, 300), 0.37, "sda")):
        v, gr = O.value_and_grad(layers, 1, Xc, yc, win, mode, beta, 1.0, th)
        g[f"vg_{tag}_values"], g[f"vg_{tag}_grads"] = v, gr
    g["vg_theta"] = th
    # one smc_step on a small relu net
    layers2 = [6, 5, 3]
    X2, y2 = O.make_teacher(layers2, 0, 40, 0, 3, 1)
    th0, lw0 = O.init_ensemble(layers2, 0, X2, y2, (0, 20, 40), 0, 1.0, 1.0, 5, 8)
    g["init_theta"], g["init_logw"] = th0, lw0
    th1, lw1, it1, rec, d = O.smc_step(layers2, 0, X2, y2, (0, 20, 40), 0, 1.0, 1.0, (0.05, 3, 0), 5, 1.0, 0, False,
                                       th0, lw0, 0)
    g["step_theta"], g["step_logw"] = th1, lw1
    g["step_ess_mlt"] = np.array([rec["ess"], rec["mean_log_target"], float(rec["resampled"])])
    for key in ("p0", "pS", "lt_new", "lt_old", "weights", "indices"):
        g[f"step_{key}"] = d[key]
    # schedules at the paper's parameters (C = kappa = 500, N = 60000, K = 200)
    tab = []
    for kind in (0, 1, 2, 3, 4):
        tab.append([O.batch_size(kind, 500, 500, 200, 60000, 1, -1, kk) for kk in range(200)])
    g["schedules"] = np.array(tab, dtype=np.int64)
    g["schedule_c2"] = np.array([O.batch_size(3, 1000, 1000, 300, 60000, 5, 300, kk) for kk in range(300)])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
