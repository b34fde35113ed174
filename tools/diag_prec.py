"""Per-precision gradient / value error of the tensor-core modes against the fp64
oracle on the C2 shape (784-200-10 ReLU), printed as one JSON line per mode."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2601_21983_b200 as p  # noqa: E402
import pyoracle as O  # noqa: E402

layers, n, M, J = [784, 200, 10], 3000, 2500, 4
spec = p.NetSpec(layers, "relu")
X, y = p.make_teacher_data(spec, n, 1, 0, 2, threads=8)
D = p.param_count(spec)
th = np.random.default_rng(5).standard_normal((J, D)).astype(np.float32).astype(np.float64)
vo, go = O.value_and_grad(layers, 0, X.astype(np.float64), y, (0, M, n), 0, 1.0, 1.0, th)
for prec in sys.argv[1:] or ["fp32", "3xtf32", "tf32", "tf32h", "f16x2", "f16"]:
    t = p.GpuEnsembleTarget(spec, X, y, J, precision=prec)
    t.set_target(0, M, n, "scaled", 1.0, 1.0)
    v, g = t.log_target_with_grad(th)
    t.close()
    nr = [float(np.linalg.norm(g[j] - go[j]) / np.linalg.norm(go[j])) for j in range(J)]
    print(json.dumps({"prec": prec, "value_rel": float(np.max(np.abs(v - vo) / np.abs(vo))),
                      "grad_normwise_max": max(nr)}), flush=True)
