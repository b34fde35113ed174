"""One C4 (or C3) gradient evaluation at the bench shape on the tensor-core CNN path, twice
(profiling target: ncu -k regex:conv_tc_kernel --launch-skip 11 --launch-count 11)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_21983_b200 as p  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
if cfg == "c4":
    spec = p.NetSpec([1600, 256, 10], "relu", ((3, 32, 32), [(3, 32, False), (3, 32, True), (3, 64, False), (3, 64, True)]))
    J, M, n = 256, 500, 2000
else:
    spec = p.NetSpec([512, 10], "relu", ((1, 28, 28), [(5, 16, True), (5, 32, True)]))
    J, M, n = 512, 500, 2000
X, y = p.make_teacher_data(spec, n, 1, 0, 4, threads=8)
t = p.GpuEnsembleTarget(spec, X, y, J, precision=os.environ.get("PREC", "tf32"))
t.set_target(0, M, n, "scaled", 1.0, 1.0)
th = 0.05 * np.random.default_rng(0).standard_normal((J, p.param_count(spec)))
for i in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    t.log_target_with_grad(th)
    print(cfg, "eval", i, f"{1e3 * (time.perf_counter() - t0):.1f} ms")
