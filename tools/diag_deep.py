"""Per-layer gradient error of the deep tensor-core path against the oracle (diagnostic)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2601_21983_b200 as p
import pyoracle as O
layers = [int(v) for v in sys.argv[1].split(",")]
M = int(sys.argv[2])
n = max(M, 400)
spec = p.NetSpec(layers, "relu")
X, y = p.make_teacher_data(spec, n, 0, 0, 9, threads=8)
D = p.param_count(spec)
J = 4
th = (0.5 * np.random.default_rng(8).standard_normal((J, D)) / np.sqrt(3)).astype(np.float32).astype(np.float64)
vo, go = O.value_and_grad(layers, 0, X.astype(np.float64), y, (0, M, n), 0, 1.0, 1.0, th)
for prec in ("fp32", "tf32"):
    t = p.GpuEnsembleTarget(spec, X, y, J, precision=prec)
    t.set_target(0, M, n, "scaled", 1.0, 1.0)
    v, g = t.log_target_with_grad(th)
    off = 0
    print(prec, "value rel", np.max(np.abs(v - vo) / np.abs(vo)))
    for l in range(1, len(layers)):
        nw = layers[l - 1] * layers[l]
        for name, sl in (("W", slice(off, off + nw)), ("b", slice(off + nw, off + nw + layers[l]))):
            e = [np.linalg.norm(g[j, sl] - go[j, sl]) / np.linalg.norm(go[j, sl]) for j in range(J)]
            print(f"  layer {l} {name}: normwise {max(e):.2e}")
        off += nw + layers[l]
    t.close()
