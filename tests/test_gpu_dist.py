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


@pytest.mark.parametrize("prec,kind,always", [("fp32", "multinomial", True), ("tf32h", "systematic", False),
                                              ("f16x2", "systematic", True)])
def test_multi_gpu_group_matches_single_context(product, prec, kind, always):
    """The C++-owned multi-GPU group (dasmc_gpu_create_multi: peer all-gather of the log-weights,
    redundant resampling, P2P row migration by a gather kernel reading the owners' memory) with
    G = 3 shards placed on the one GPU of this box is bit-identical to one context, step after
    step (smc.hpp:109-158; the shard count must not change results, parallel.hpp:13-15)."""
    layers = [64, 32, 10]
    spec = product.NetSpec(layers, "tanh")
    X, y = product.make_teacher_data(spec, 2000, 0, 0, 1, threads=8)
    J, K = 50, 5
    cfg = product.KernelConfig.hmc(0.002, 3)
    single = product.GpuEnsembleTarget(spec, X, y, J, precision=prec)
    group = product.GpuEnsembleTarget(spec, X, y, J, precision=prec, devices=[0, 0, 0])
    assert product.load().dasmc_gpu_multi_shards(group.h) == 3
    for t in (single, group):
        t.set_target(0, 300, 2000, "scaled", 1.0, 1.0)
        t.init_ensemble(J, 11)
    a0, b0 = single.get_ensemble(J, dtype=np.float32), group.get_ensemble(J, dtype=np.float32)
    assert np.array_equal(a0[0], b0[0]) and np.array_equal(a0[1], b0[1])
    for k in range(K):
        a = single.smc_step(cfg, 11, kind, 0.5, always=always)
        b = group.smc_step(cfg, 11, kind, 0.5, always=always)
        assert a == {**b, "sampler_ms": a["sampler_ms"]}, (k, a, b)
    # asynchronous steps + sync_records, as bench.py drives them
    for k in range(3):
        single.smc_step(cfg, 11, kind, 0.5, always=always, sync=False)
        group.smc_step(cfg, 11, kind, 0.5, always=always, sync=False)
    ra, rb = single.sync_records(3), group.sync_records(3)
    assert [(r["ess"], r["resampled"], r["mean_log_target"]) for r in ra] == \
        [(r["ess"], r["resampled"], r["mean_log_target"]) for r in rb]
    th_a, lw_a, it_a = single.get_ensemble(J)
    th_b, lw_b, it_b = group.get_ensemble(J)
    assert np.array_equal(th_a, th_b) and np.array_equal(lw_a, lw_b) and it_a == it_b == K + 3
    single.close()
    group.close()


def test_multi_gpu_group_sda_moments(product):
    """Sharded SDA (annealing.hpp:153-174): the moments of the group's post-step ensemble -- from
    the all-gathered per-particle (prefix, block) log-likelihood pairs of the step's own
    evaluations -- equal the single context's, and an explicit pass after set_ensemble agrees."""
    layers = [36, 20, 3]
    spec = product.NetSpec(layers, "relu")
    X, y = product.make_teacher_data(spec, 900, 0, 0, 4, threads=8)
    J = 40
    cfg = product.KernelConfig.hmc(0.003, 2)
    single = product.GpuEnsembleTarget(spec, X, y, J, precision="fp32")
    group = product.GpuEnsembleTarget(spec, X, y, J, precision="fp32", devices=[0, 0])
    for t in (single, group):
        t.set_target(100, 300, 900, "sda", 0.3, 1.0)
        t.init_ensemble(J, 3)
    for _ in range(3):
        ra = single.smc_step(cfg, 3, "systematic", 0.5)
        rb = group.smc_step(cfg, 3, "systematic", 0.5)
        assert ra["ess"] == rb["ess"]
        ma, mb = single.sda_moments(100, 300), group.sda_moments(100, 300)
        assert np.array_equal(ma, mb), (ma, mb)
    # a different window forces the explicit forward pass on every shard
    assert np.array_equal(single.sda_moments(100, 400), group.sda_moments(100, 400))
    single.close()
    group.close()
