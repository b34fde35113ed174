"""CPU, world_size 2 over gloo: the particle-sharded SMC protocol of
paper_2601_21983_b200/dist.py (global-slot RNG streams, reference-order
all-gather, redundant resampling indices, the product's dasmc_shard_plan
migration) reproduces the single-process run exactly.  The per-rank compute
engine here is the CPU oracle (test infrastructure); on B200 the same protocol
drives GpuShardEngine (tests/test_gpu_dist.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

LAYERS, ACT = [6, 5, 3], 0
WIN = (0, 20, 40)
KERNEL = (0.05, 3, 0)
SEED = 5
J = 16
K = 4


def problem():
    import pyoracle as O
    X, y = O.make_teacher(LAYERS, ACT, 40, 0, 3, 1)
    th0, lw0 = O.init_ensemble(LAYERS, ACT, X, y, WIN, 0, 1.0, 1.0, SEED, J)
    return X, y, th0, lw0


class OracleShardEngine:
    """Per-rank engine over the fp64 oracle, mirroring GpuShardEngine's interface."""

    dtype = torch.float64

    def __init__(self, X, y, thetas, lw, j0, iteration):
        import pyoracle as O
        self.O, self.X, self.y = O, X, y
        self.th = np.array(thetas)
        self.lw = np.array(lw)
        self.j0 = j0
        self.k = iteration
        self.row = self.th.shape[1]

    def propose(self, cfg, seed, j0, Jr, device):
        gj = np.arange(j0, j0 + Jr)
        th, inc, lt = self.O.propose_particles(LAYERS, ACT, self.X, self.y, WIN, 0, 1.0, 1.0, KERNEL, seed, self.k, gj,
                                               self.th, threads=2)
        self.th = th
        return torch.from_numpy(self.lw + inc), torch.from_numpy(lt)

    def resample(self, lw_full, lt_full, j0, seed, kind, fraction, always):
        O = self.O
        lwf, ltf = lw_full.numpy(), lt_full.numpy()
        Jt = lwf.shape[0]
        w, ess = O.normalize(lwf)  # smc.hpp:142-143
        mlt = 0.0
        for j in range(Jt):  # smc.hpp:144-148, ascending j
            if w[j] > 0.0:
                mlt += w[j] * ltf[j]
        res = always or ess < fraction * Jt
        idx = np.arange(Jt, dtype=np.int32)
        if res:
            u = O.rng_uniforms(O.fork_key(seed, 3, self.k, 0), Jt if kind == "multinomial" else 1)
            idx = O.resample_indices(w, u, 0 if kind == "multinomial" else 1)
        Jr = self.th.shape[0]
        self.lw = np.full(Jr, -np.log(Jt)) if res else lwf[j0:j0 + Jr].copy()

        class Rec:
            pass
        r = Rec()
        r.k, r.ess, r.resampled, r.mean_log_target, r.n_divergent = self.k, ess, int(res), mlt, 0
        self.k += 1
        return torch.from_numpy(idx), r

    def pack(self, rows, device):
        return torch.from_numpy(self.th[np.asarray(rows, dtype=np.int64)].copy())

    def unpack(self, src, slots):
        new = np.empty_like(self.th)
        new[np.asarray(slots, dtype=np.int64)] = src.numpy()
        self.th = new


def _worker(rank, world, port, kind, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_21983_b200.dist import TorchComm, shard_range, sharded_step
    from paper_2601_21983_b200.api import KernelConfig
    X, y, th0, lw0 = problem()
    lo, hi = shard_range(J, world, rank)
    eng = OracleShardEngine(X, y, th0[lo:hi], lw0[lo:hi], lo, 0)
    comm = TorchComm("cpu")
    recs = []
    for _ in range(K):
        recs.append(sharded_step(eng, comm, J, KernelConfig.hmc(*KERNEL[:2]), SEED, kind, 1.0, True, "cpu"))
    ths = [torch.zeros((hi2 - lo2, eng.row), dtype=torch.float64) for lo2, hi2 in
           (shard_range(J, world, r) for r in range(world))]
    dist.all_gather(ths, torch.from_numpy(eng.th))
    lws = [torch.zeros(hi2 - lo2, dtype=torch.float64) for lo2, hi2 in (shard_range(J, world, r) for r in range(world))]
    dist.all_gather(lws, torch.from_numpy(eng.lw))
    if rank == 0:
        out_q.put((recs, torch.cat(ths).numpy(), torch.cat(lws).numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kind", ["systematic", "multinomial"])
def test_sharded_two_ranks_match_single_process(oracle, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    recs, th, lw = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: the oracle's own smc_step (smc.hpp:109-158)
    X, y, th_ref, lw_ref = problem()
    it = 0
    ref_recs = []
    for _ in range(K):
        th_ref, lw_ref, it, rec, _d = oracle.smc_step(LAYERS, ACT, X, y, WIN, 0, 1.0, 1.0, KERNEL, SEED, 1.0,
                                                      0 if kind == "multinomial" else 1, True, th_ref, lw_ref, it,
                                                      threads=2)
        ref_recs.append(rec)
    assert np.array_equal(th, th_ref)
    assert np.array_equal(lw, lw_ref)
    for a, b in zip(recs, ref_recs):
        assert a["ess"] == b["ess"] and a["mean_log_target"] == b["mean_log_target"] and a["resampled"]
    if kind == "multinomial":  # unsorted indices: particles actually crossed ranks
        assert sum(r["migrated_rows"] for r in recs) > 0


def test_shard_plan_roundtrip(product):
    """dasmc_shard_plan: every destination slot receives exactly the row idx[j] names."""
    from paper_2601_21983_b200.dist import shard_plan, shard_range
    rng = np.random.default_rng(0)
    for J, G in ((16, 2), (37, 3), (64, 8), (9, 9)):
        idx = rng.integers(0, J, size=J).astype(np.int32)
        plans = [shard_plan(idx, G, r) for r in range(G)]
        for d in range(G):
            lo_d, hi_d = shard_range(J, G, d)
            recv_src, recv_row = plans[d][0], plans[d][1]
            for s in range(G):
                # rows rank s sends to d, in d's slot order
                off = int(plans[s][2][:d].sum())
                sent = plans[s][3][off:off + int(plans[s][2][d])]
                lo_s, _ = shard_range(J, G, s)
                assert np.array_equal(sent, recv_row[recv_src == s])
                assert np.array_equal(sent + lo_s, idx[lo_d:hi_d][recv_src == s])


def _np_probs(th, X):
    """numpy forward of LAYERS (reference theta layout) -> softmax rows (test-side engine)."""
    a = X
    off = 0
    for l in range(1, len(LAYERS)):
        i, o = LAYERS[l - 1], LAYERS[l]
        W = th[off:off + i * o].reshape(i, o)
        off += i * o
        a = a @ W + th[off:off + o]
        off += o
        if l + 1 < len(LAYERS):
            a = np.maximum(a, 0.0)
    e = np.exp(a - a.max(1, keepdims=True))
    return e / e.sum(1, keepdims=True)


class _PredEngine:
    def __init__(self, th):
        self.th = th

    def classes(self):
        return LAYERS[-1]

    def predictive_mix(self, X, w_local, Jr, pred, y=None):
        for j in range(Jr):
            if w_local[j] > 0:
                pred += w_local[j] * _np_probs(self.th[j], X)
        return pred


def _pred_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_21983_b200.dist import TorchComm, shard_range, sharded_evaluate_predictive
    X, y, th0, lw0 = problem()
    lw0 = lw0.copy()
    lw0[2] = -np.inf
    lo, hi = shard_range(J, world, rank)
    res = sharded_evaluate_predictive(_PredEngine(th0[lo:hi]), TorchComm("cpu"), J, lw0[lo:hi], X, y)
    if rank == 0:
        out_q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_evaluate_predictive_two_ranks(oracle):
    """evaluate_predictive of a sharded ensemble (all-gathered weights, all-reduced mixture)
    equals the oracle's single-process runner.hpp:331-364."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pred_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    lp, acc = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X, y, th0, lw0 = problem()
    lw0 = lw0.copy()
    lw0[2] = -np.inf
    lpo, acco = oracle.evaluate_predictive(LAYERS, ACT, X, y, th0, lw0)
    assert abs(lp - lpo) < 1e-12 * abs(lpo) and acc == acco
