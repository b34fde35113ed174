"""Particle-sharded SMC across GPUs: one process per GPU.

Rank r owns global particle slots [J*r/G, J*(r+1)/G) (parallel.hpp:30-31
partition).  Every RNG stream is keyed by the GLOBAL slot (fork(kProposal, k,
j), smc.hpp:119-120), so a sharded run reproduces the single-GPU run.  One
iteration:

  1. engine.propose      local move + incremental weights (no communication)
  2. all-gather          J log-weights and log_target_new, in slot order
  3. engine.resample     normalise / ESS / decision / indices on the full
                         vectors -- computed redundantly, identically, on every rank
  4. migration           dasmc_shard_plan (identical on all ranks, so no extra
                         exchange) -> pack rows -> point-to-point send/recv ->
                         unpack into the next ensemble

The engine is the C-ABI (GpuShardEngine); the communicator is torch.distributed
(NCCL over NVLink on B200, gloo in the CPU tests) -- plumbing only.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import GpuEnsembleTarget, KernelConfig, _RESAMPLE


def shard_range(J: int, world: int, rank: int):
    lo, hi = C.c_int64(), C.c_int64()
    L.load().dasmc_shard_range(J, world, rank, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def shard_plan(idx: np.ndarray, world: int, rank: int):
    """dasmc_shard_plan: (recv_src[Jr], recv_row[Jr], send_cnt[G], send_rows[sum send_cnt])."""
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    J = idx.shape[0]
    lo, hi = shard_range(J, world, rank)
    recv_src = np.empty(hi - lo, dtype=np.int32)
    recv_row = np.empty(hi - lo, dtype=np.int32)
    send_cnt = np.empty(world, dtype=np.int64)
    send_rows = np.empty(J, dtype=np.int32)
    L.check(L.load().dasmc_shard_plan(idx.ctypes.data_as(L._I32), J, world, rank, recv_src.ctypes.data_as(L._I32),
                                      recv_row.ctypes.data_as(L._I32), send_cnt.ctypes.data_as(L._I64),
                                      send_rows.ctypes.data_as(L._I32)))
    return recv_src, recv_row, send_cnt, send_rows[: int(send_cnt.sum())]


class TorchComm:
    """all-gather + point-to-point row exchange over torch.distributed."""

    def __init__(self, device):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device

    def all_gather(self, x, counts):
        """Concatenate every rank's 1-D x (rank r contributes counts[r] entries)."""
        torch = self.torch
        mx = max(counts)
        pad = torch.zeros(mx, dtype=x.dtype, device=x.device)
        pad[: x.numel()] = x
        outs = [torch.empty(mx, dtype=x.dtype, device=x.device) for _ in range(self.world)]
        self.dist.all_gather(outs, pad)
        return torch.cat([o[:c] for o, c in zip(outs, counts)])

    def exchange(self, sends, recv_counts, row, dtype=None):
        """sends[d]: tensor [n_d, row] for rank d (self included); returns recvs[s]."""
        torch, dist = self.torch, self.dist
        dtype = dtype or torch.float32
        recvs = [torch.empty((int(n), row), dtype=dtype, device=self.device) for n in recv_counts]
        ops = []
        for p in range(self.world):
            if p == self.rank:
                if recv_counts[p]:
                    recvs[p].copy_(sends[p])
                continue
            if sends[p] is not None and sends[p].shape[0]:
                ops.append(dist.P2POp(dist.isend, sends[p].contiguous(), p))
            if recv_counts[p]:
                ops.append(dist.P2POp(dist.irecv, recvs[p], p))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return recvs


class GpuShardEngine:
    """The C-ABI shard primitives of one GPU context (include/dasmc_gpu.h)."""

    def __init__(self, target: GpuEnsembleTarget):
        import torch
        self.torch = torch
        self.t = target
        self.lib = target.lib
        self.row = int(self.lib.dasmc_gpu_row_floats(target.h))

    def propose(self, cfg: KernelConfig, seed: int, j0: int, Jr: int, device):
        torch = self.torch
        lw = torch.empty(Jr, dtype=torch.float64, device=device)
        lt = torch.empty(Jr, dtype=torch.float64, device=device)
        kc = cfg.c()
        torch.cuda.synchronize()
        L.check(self.lib.dasmc_gpu_shard_propose(self.t.h, C.byref(kc), seed, j0, lw.data_ptr(), lt.data_ptr()))
        return lw, lt

    def resample(self, lw_full, lt_full, j0, seed, kind, fraction, always):
        torch = self.torch
        J = lw_full.numel()
        idx = torch.empty(J, dtype=torch.int32, device=lw_full.device)
        rec = L.IterRecord()
        torch.cuda.synchronize()
        L.check(self.lib.dasmc_gpu_shard_resample(self.t.h, lw_full.data_ptr(), lt_full.data_ptr(), J, j0, seed,
                                                  _RESAMPLE[kind], fraction, 1 if always else 0, idx.data_ptr(),
                                                  C.byref(rec)))
        return idx, rec

    def pack(self, rows: np.ndarray, device):
        torch = self.torch
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        buf = torch.empty((rows.shape[0], self.row), dtype=torch.float32, device=device)
        if rows.shape[0]:
            torch.cuda.synchronize()
            L.check(self.lib.dasmc_gpu_pack_rows(self.t.h, rows.ctypes.data_as(L._I32), rows.shape[0], buf.data_ptr()))
        return buf

    def classes(self) -> int:
        return int(self.t.spec.layer_sizes[-1])

    def predictive_mix(self, X_test, w_local, J, pred, y_test=None):
        self.torch.cuda.synchronize()
        return self.t.predictive_mix(X_test, w_local, J, pred, y_test)

    def unpack(self, src, slots: np.ndarray):
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        self.torch.cuda.synchronize()
        L.check(self.lib.dasmc_gpu_unpack_rows(self.t.h, src.data_ptr(), slots.ctypes.data_as(L._I32), slots.shape[0]))


def sharded_step(engine, comm, J: int, cfg: KernelConfig, seed: int, kind: str = "systematic",
                 fraction: float = 0.5, always: bool = False, device=None):
    """One SMC iteration of a particle-sharded ensemble (smc.hpp:109-158)."""
    torch = comm.torch
    world, rank = comm.world, comm.rank
    bounds = [shard_range(J, world, r) for r in range(world)]
    counts = [hi - lo for lo, hi in bounds]
    j0, j1 = bounds[rank]
    lw, lt = engine.propose(cfg, seed, j0, j1 - j0, device)
    lw_full = comm.all_gather(lw, counts)
    lt_full = comm.all_gather(lt, counts)
    idx, rec = engine.resample(lw_full, lt_full, j0, seed, kind, fraction, always)
    out = {"k": rec.k, "ess": rec.ess, "resampled": bool(rec.resampled), "mean_log_target": rec.mean_log_target,
           "n_divergent": rec.n_divergent, "migrated_rows": 0}
    if rec.resampled:
        idx_h = idx.cpu().numpy() if hasattr(idx, "cpu") else np.asarray(idx)
        recv_src, recv_row, send_cnt, send_rows = shard_plan(idx_h, world, rank)
        # each distinct source row crosses the fabric once per destination rank: both
        # sides derive the same sorted unique row list from the (identical) plan, and
        # the receiver fans the rows out to its slots on the device.  Resampling
        # duplicates survivors, so after a weight collapse this is 1 row, not J/G
        sends, off = [], 0
        for d in range(world):
            n = int(send_cnt[d])
            sends.append(engine.pack(np.unique(send_rows[off:off + n]).astype(np.int32), device))
            off += n
        uniq, inv = [], np.empty(len(recv_src), dtype=np.int64)
        base = 0
        for s in range(world):
            sl = np.nonzero(recv_src == s)[0]
            u, iv = np.unique(recv_row[sl], return_inverse=True)
            uniq.append(u)
            inv[sl] = base + iv
            base += len(u)
        recv_counts = [len(u) for u in uniq]
        recvs = comm.exchange(sends, recv_counts, engine.row, getattr(engine, "dtype", None))
        src = torch.cat([r for r in recvs if r.shape[0]], dim=0)
        src = src.index_select(0, torch.as_tensor(inv, device=src.device))
        engine.unpack(src, np.arange(len(recv_src), dtype=np.int32))
        out["migrated_rows"] = int(sum(recv_counts) - recv_counts[rank])
    return out


def sharded_evaluate_predictive(engine, comm, J: int, local_log_w, X_test, y_test):
    """evaluate_predictive (runner.hpp:331-364) of a particle-sharded ensemble (SURVEY.md §8e
    item 5): all-gather the log-weights, normalise them identically on every rank, mix this
    rank's particles into pred[n x C], all-reduce pred (sum), then the metrics."""
    torch = comm.torch
    world, rank = comm.world, comm.rank
    bounds = [shard_range(J, world, r) for r in range(world)]
    counts = [hi - lo for lo, hi in bounds]
    j0, j1 = bounds[rank]
    lw = torch.as_tensor(np.ascontiguousarray(local_log_w, dtype=np.float64), device=comm.device)
    full = comm.all_gather(lw, counts).cpu().numpy()
    m = full.max()
    if m == -np.inf:
        raise L.SamplerError(L.DASMC_EDEAD, "normalize: all particles dead")
    w = np.exp(full - m)  # normalize (smc.hpp:57-64), same order on every rank
    w /= w.sum()
    pred = np.zeros((np.asarray(X_test).shape[0], engine.classes()), dtype=np.float64)
    engine.predictive_mix(X_test, w[j0:j1], j1 - j0, pred, y_test)
    pt = torch.as_tensor(pred, device=comm.device)
    comm.dist.all_reduce(pt)
    from .api import predictive_metrics
    return predictive_metrics(pt.cpu().numpy(), y_test)
