"""CPU: host logic of the sharded (N > 1) solve, SURVEY.md §8(e).

* the partition plan the C-ABI hands every rank (aapdhg_cuda_partition,
  host-only: no GPU needed) — contiguous, covering, non-empty, nnz-balanced;
* a world_size-2 `gloo` run of the exact exchange schedule the sm_100a path
  uses (shard.cu): relabelled K row block and K' row block per rank, all-gather
  of y, K'y on the column block, all-gather of xhat, K xhat on the row block,
  all-gather of the scalar partials summed in rank order — checked against the
  oracle's PDHG trajectory. This pins the decomposition and the relabelling;
  the kernels themselves are covered on the GPU (test_gpu_dist.py)."""
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
