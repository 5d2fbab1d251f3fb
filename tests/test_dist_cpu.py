"""CPU: host logic of the sharded (N > 1) solve, SURVEY.md §8(e).

* the partition plan the C-ABI hands every rank (aapdhg_cuda_partition,
  host-only: no GPU needed) — contiguous, covering, non-empty, nnz-balanced;
* a world_size-2 `gloo` run of the exact exchange schedule the sm_100a path
  uses (shard.cu): relabelled K row block and K' row block per rank, all-gather
  of y, K'y on the column block, all-gather of xhat, K xhat on the row block,
  all-gather of the scalar partials summed in rank order — checked against the
  oracle's PDHG trajectory. This pins the decomposition and the relabelling;
  the kernels themselves are covered on the GPU (test_gpu_dist.py);
* a threaded model of the P2P transport's exchange protocol (remote stores,
  per-slot arrival sequences, waits) under random interleavings, with
  negative controls showing it catches a misplaced wait or arrival."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2508_08062_b200 import (Method, SolverConfig, UnsupportedError, partition,
                                   problems)


@pytest.mark.parametrize("cfg,scale", [(0, 1.0), (1, 0.02), (2, 0.05), (3, 0.001)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_plan(cfg, scale, world):
    p = problems.make_config(cfg, scale=scale)
    rows, cols = partition(p.k, world)
    m, n = p.k.nrows, p.n()
    for b, total in ((rows, m), (cols, n)):
        assert b[0] == 0 and b[-1] == total
        assert np.all(np.diff(b) >= 1)
    # nnz balance of the row blocks: weights nnz + 4 per row, greedy prefix
    # split, so every block is within one row of the ideal share
    rl = np.diff(p.k.row_ptr).astype(np.int64) + 4
    share = rl.sum() / world
    blocks = np.array([rl[rows[r]:rows[r + 1]].sum() for r in range(world)])
    assert np.all(np.abs(blocks - share) <= rl.max() + 1)
    cl = np.bincount(p.k.col_idx, minlength=n).astype(np.int64) + 4
    cshare = cl.sum() / world
    cblocks = np.array([cl[cols[r]:cols[r + 1]].sum() for r in range(world)])
    assert np.all(np.abs(cblocks - cshare) <= cl.max() + 1)


def test_partition_rejects_too_many_shards():
    p = problems.toy()
    with pytest.raises(UnsupportedError):
        partition(p.k, 2)


# ---- the exchange schedule over gloo ---------------------------------------
def _shard(p, rows, cols, r):
    """Shard r exactly as shard.cu builds it (relabelled padded indices)."""
    world = len(rows) - 1
    maxr, maxc = int(np.diff(rows).max()), int(np.diff(cols).max())
    xmap = np.empty(p.n(), dtype=np.int64)
    ymap = np.empty(p.k.nrows, dtype=np.int64)
    for o in range(world):
        xmap[cols[o]:cols[o + 1]] = o * maxc + np.arange(cols[o + 1] - cols[o])
        ymap[rows[o]:rows[o + 1]] = o * maxr + np.arange(rows[o + 1] - rows[o])
    k = p.k
    r0, r1, c0, c1 = rows[r], rows[r + 1], cols[r], cols[r + 1]
    e0, e1 = k.row_ptr[r0], k.row_ptr[r1]
    kr = sp.csr_matrix((k.vals[e0:e1], xmap[k.col_idx[e0:e1]], k.row_ptr[r0:r1 + 1] - e0),
                       shape=(r1 - r0, world * maxc))
    kt = sp.csr_matrix((k.vals, k.col_idx, k.row_ptr), shape=(k.nrows, p.n())).tocsc()
    # column j of K in ascending row order = row j of K' (matvec_transpose order)
    t0, t1 = kt.indptr[c0], kt.indptr[c1]
    ktr = sp.csr_matrix((kt.data[t0:t1], ymap[kt.indices[t0:t1]], kt.indptr[c0:c1 + 1] - t0),
                        shape=(c1 - c0, world * maxr))
    return dict(kr=kr, ktr=ktr, r0=r0, r1=r1, c0=c0, c1=c1, maxr=maxr, maxc=maxc,
                c=p.c[c0:c1], l=p.l[c0:c1], u=p.u[c0:c1], q=p.q[r0:r1],
                m1=max(0, min(p.m1 - r0, r1 - r0)))


def _worker(rank, world, port, iters, tau, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = problems.make_config(0, scale=0.3)
        rows, cols = partition(p.k, world)
        # every rank must hold the same plan
        plan = torch.tensor(np.concatenate([rows, cols]), dtype=torch.int64)
        plans = [torch.zeros_like(plan) for _ in range(world)]
        dist.all_gather(plans, plan)
        assert all(torch.equal(plans[0], q) for q in plans)
        s = _shard(p, rows, cols, rank)

        def allgather(local, chunk):
            buf = torch.zeros(chunk, dtype=torch.float64)
            buf[:len(local)] = torch.from_numpy(local)
            parts = [torch.zeros(chunk, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, buf)
            return torch.cat(parts).numpy()

        x = np.zeros(s["c1"] - s["c0"])
        y = np.zeros(s["r1"] - s["r0"])
        kx = np.zeros_like(y)
        g = []
        for _ in range(iters):
            yg = allgather(y, s["maxr"])                                   # AG y
            t = s["ktr"] @ yg                                              # K'y (C_r)
            xh = np.minimum(np.maximum(x - tau * (s["c"] - t), s["l"]), s["u"])
            xg = allgather(xh, s["maxc"])                                  # AG xhat
            kxh = s["kr"] @ xg                                             # K xhat (R_r)
            yh = y + tau * (s["q"] - (2.0 * kxh - kx))
            yh[:s["m1"]] = np.maximum(yh[:s["m1"]], 0.0)
            part = np.array([np.sum((xh - x) ** 2) + np.sum((yh - y) ** 2)])
            tot = allgather(part, 1)                                       # AG scalars
            acc = 0.0
            for v in tot:                                                  # rank order
                acc += v
            g.append(np.sqrt(acc))
            x, y, kx = xh, yh, kxh
        if rank == 0:
            np.save(out_path, np.array(g))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_gloo_world2_exchange_schedule_matches_oracle(tmp_path):
    import torch.multiprocessing as mp

    from oracle.pyoracle import Oracle
    p = problems.make_config(0, scale=0.3)
    tau, iters = 0.05, 25
    out = tmp_path / "g.npy"
    mp.start_processes(_worker, args=(2, _free_port(), iters, tau, str(out)), nprocs=2,
                       join=True, start_method="spawn")
    got = np.load(out)
    ref = Oracle("port").solve(p, SolverConfig(method=Method.PDHG, toll=1e-30,
                                               max_iters=iters, tau=tau, sigma=tau))
    want = ref.trajectory["g_norm"][:iters]
    np.testing.assert_allclose(got, want, rtol=1e-12)


# ---- the P2P exchange protocol (shard.cu / pipeline.cuh p2p_arrive, p2p_wait) ----
class _P2pModel:
    """Ranks as threads running the exact order of the P2P sharded iteration:
    producers store their chunk into every rank's buffer as soon as they run,
    arrivals bump a per-slot sequence number into every rank's flag array, a
    wait spins until every rank's flag has reached this rank's own count.
    Every read checks the version tag of each chunk it consumes: a producer
    that overwrote a buffer before its reader was done (a misplaced arrival
    or wait) shows up as a newer tag."""

    XG, YG, SCAL, DOTS, XG2 = 0, 1, 3, 4, 5

    def __init__(self, world, iters, aa_every, seed):
        import random
        import threading
        self.world, self.iters, self.aa_every = world, iters, aa_every
        self.xg = [[None] * world for _ in range(world)]
        self.yg = [[("y", 0)] * world for _ in range(world)]  # start iterate, all-gathered
        self.scal = [[None] * world for _ in range(world)]
        self.dots = [[None] * world for _ in range(world)]
        self.flags = [[[0] * world for _ in range(8)] for _ in range(world)]
        self.seq = [[0] * 8 for _ in range(world)]
        self.rng = [random.Random(seed * 131 + r) for r in range(world)]
        self.errors = []
        self.lock = threading.Lock()

    def jitter(self, r):
        import time
        if self.rng[r].random() < 0.5:
            time.sleep(self.rng[r].random() * 2e-4)

    def arrive(self, r, slot):
        self.seq[r][slot] += 1
        for q in range(self.world):
            self.jitter(r)
            self.flags[q][slot][r] = self.seq[r][slot]

    def wait(self, r, slot):
        import time
        t0 = time.monotonic()
        while any(self.flags[r][slot][p] < self.seq[r][slot] for p in range(self.world)):
            time.sleep(1e-5)
            if time.monotonic() - t0 > 20:
                raise RuntimeError(f"rank {r} deadlocked at slot {slot}")

    def store(self, r, buf, tag):
        for q in range(self.world):
            self.jitter(r)
            buf[q][r] = tag

    def read(self, r, buf, tag, what):
        for p in range(self.world):
            self.jitter(r)
            if buf[r][p] != tag:
                with self.lock:
                    self.errors.append((r, what, p, buf[r][p], tag))

    def rank(self, r):
        try:
            self.arrive(r, self.YG)  # the start iterate's exchange(YG)
            self.wait(r, self.YG)
            for k in range(self.iters):
                self.wait(r, self.YG)                     # K1: y of u_k
                self.read(r, self.yg, ("y", k), "K1 y")
                self.store(r, self.xg, ("x", k))          # xhat_k
                self.arrive(r, self.XG)                   # K1's last CTA
                self.wait(r, self.XG)                     # K2
                self.read(r, self.xg, ("x", k), "K2 xhat")
                self.store(r, self.yg, ("y", k + 1))      # yhat (y of u_{k+1} if plain)
                self.store(r, self.scal, k)
                self.arrive(r, self.YG)                   # K2's last CTA
                self.wait(r, self.YG)                     # control
                self.read(r, self.scal, k, "control totals")
                if k % self.aa_every == self.aa_every - 1:  # replicated decision: AA branch
                    self.store(r, self.dots, k)
                    self.arrive(r, self.DOTS)
                    self.wait(r, self.DOTS)
                    self.read(r, self.dots, k, "aa_solve dots")
                    self.store(r, self.xg, ("c", k))      # candidate x
                    self.store(r, self.yg, ("y", k + 1))  # candidate y
                    self.arrive(r, self.XG2)
                    self.wait(r, self.XG2)
                    self.read(r, self.xg, ("c", k), "recache candidate")
                    self.arrive(r, self.YG)               # end of the AA branch
        except Exception as e:  # noqa: BLE001
            with self.lock:
                self.errors.append((r, repr(e)))

    def run(self):
        import threading
        ts = [threading.Thread(target=self.rank, args=(r,)) for r in range(self.world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return self.errors


@pytest.mark.parametrize("world,seed", [(2, 1), (3, 2), (4, 3), (8, 4)])
def test_p2p_exchange_protocol_model(world, seed):
    """The P2P transport's arrival / wait placement never lets
    a rank overwrite a buffer another rank still reads, and never deadlocks,
    under random interleavings of world ranks over plain and AA iterations."""
    errors = _P2pModel(world, iters=24, aa_every=4, seed=seed).run()
    assert not errors, errors[:5]


def test_p2p_protocol_model_catches_a_missing_wait():
    """The model is sharp: dropping K2's wait for the XG arrivals lets a rank
    read xhat chunks its peers have not stored yet."""
    class NoXgWait(_P2pModel):
        def wait(self, r, slot):
            if slot == self.XG:
                return
            super().wait(r, slot)
    found = any(NoXgWait(4, iters=24, aa_every=4, seed=s).run() for s in range(6))
    assert found


def test_p2p_protocol_model_catches_a_missing_aa_arrival():
    """... and dropping the AA branch's closing YG arrival lets a fast rank's
    next K1 store xhat into a peer's xg while that peer's recache still reads
    the candidate there."""
    class NoAaArrival(_P2pModel):
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            self.in_aa = [False] * self.world

        def read(self, r, buf, tag, what):
            super().read(r, buf, tag, what)
            if what == "recache candidate":
                self.in_aa[r] = True

        def arrive(self, r, slot):
            if slot == self.YG and self.in_aa[r]:
                self.in_aa[r] = False
                return
            super().arrive(r, slot)
    found = any(NoAaArrival(4, iters=24, aa_every=4, seed=s).run() for s in range(6))
    assert found
