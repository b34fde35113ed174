"""GPU: the sharded-ensemble primitives (dasmc_gpu_shard_*, pack/unpack rows)
emulating G shards as G contexts on ONE GPU, stepped sequentially in one
process (no kernel waits on another), against a single-context run: results
must be bit-identical (RNG streams keyed by global slot, full-vector
normalisation in reference order)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _emulated_step(engines, J, cfg, seed, kind, fraction, always):
    from paper_2601_21983_b200.dist import shard_plan, shard_range
    G = len(engines)
    dev = torch.device("cuda", 0)
    bounds = [shard_range(J, G, r) for r in range(G)]
    parts = [e.propose(cfg, seed, lo, hi - lo, dev) for e, (lo, hi) in zip(engines, bounds)]
    lw_full = torch.cat([p[0] for p in parts])
    lt_full = torch.cat([p[1] for p in parts])
    outs = [e.resample(lw_full, lt_full, lo, seed, kind, fraction, always) for e, (lo, _) in zip(engines, bounds)]
    idx0, rec0 = outs[0]
    for idx, rec in outs[1:]:
        assert torch.equal(idx, idx0) and rec.ess == rec0.ess  # redundant decision identical on every shard
    if rec0.resampled:
        idx_h = idx0.cpu().numpy()
        plans = [shard_plan(idx_h, G, r) for r in range(G)]
        sends = []
        for r, e in enumerate(engines):
            cnt, rows = plans[r][2], plans[r][3]
            offs = np.concatenate([[0], np.cumsum(cnt)])
            sends.append([e.pack(rows[offs[d]:offs[d + 1]], dev) for d in range(G)])
        for d, e in enumerate(engines):
            recv_src = plans[d][0]
            src = torch.cat([sends[s][d] for s in range(G) if sends[s][d].shape[0]])
            slots = np.concatenate([np.nonzero(recv_src == s)[0] for s in range(G)]).astype(np.int32)
            e.unpack(src, slots)
    return rec0


@pytest.mark.parametrize("prec,kind", [("fp32", "multinomial"), ("tf32", "systematic")])
def test_sharded_matches_single_context(product, prec, kind):
    from paper_2601_21983_b200.dist import GpuShardEngine, shard_range
    layers = [64, 32, 10]
    spec = product.NetSpec(layers, "tanh")
    X, y = product.make_teacher_data(spec, 2000, 0, 0, 1, threads=8)
    J, G, K = 48, 3, 4
    cfg = product.KernelConfig.hmc(0.002, 3)
    single = product.GpuEnsembleTarget(spec, X, y, J, precision=prec)
    single.set_target(0, 200, 2000, "scaled", 1.0, 1.0)
    single.init_ensemble(J, 7)
    th0, lw0, _ = single.get_ensemble(J, dtype=np.float32)
    shards = []
    for r in range(G):
        lo, hi = shard_range(J, G, r)
        t = product.GpuEnsembleTarget(spec, X, y, hi - lo, precision=prec)
        t.set_target(0, 200, 2000, "scaled", 1.0, 1.0)
        t.set_ensemble(th0[lo:hi], lw0[lo:hi], 0)
        shards.append(t)
    engines = [GpuShardEngine(t) for t in shards]
    for _ in range(K):
        a = single.smc_step(cfg, 7, kind, 1.0, always=True)
        b = _emulated_step(engines, J, cfg, 7, kind, 1.0, True)
        assert a["ess"] == b.ess and a["mean_log_target"] == b.mean_log_target
    th_s, lw_s, it_s = single.get_ensemble(J, dtype=np.float32)
    got = [t.get_ensemble(t.max_particles, dtype=np.float32) for t in shards]
    assert np.array_equal(np.concatenate([g[0] for g in got]), th_s)
    assert np.array_equal(np.concatenate([g[1] for g in got]), lw_s)
    assert all(g[2] == it_s == K for g in got)
