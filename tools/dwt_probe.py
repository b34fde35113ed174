"""Probe (debug aid): one value_and_grad of a two-stage CNN under DASMC_CONV_DWT=1; argv: k cin cout [pool1]"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2601_21983_b200 as p
k, c1, c2 = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
h1 = 28 - k + 1
hp = h1 // 2
h2 = hp - k + 1
h2p = h2 // 2
conv = ((1, 28, 28), [(k, c1, True), (k, c2, True)])
spec = p.NetSpec([c2 * h2p * h2p, 10], "relu", conv)
X, y = p.make_teacher_data(spec, 64, 1, 0, 3, threads=8)
D = p.param_count(spec)
th = (0.3 * np.random.default_rng(1).standard_normal((3, D))).astype(np.float32).astype(np.float64)
t = p.GpuEnsembleTarget(spec, X, y, 3, precision="tf32")
t.set_target(0, 40, 64, "scaled", 1.0, 1.0)
v, g = t.log_target_with_grad(th)
print("ok", sys.argv[1:], v[:2], float(np.abs(g).max()))
