"""Host-side logic of the row-sharded path on CPU with torch.distributed
(gloo, world_size 2, 127.0.0.1): nnz-balanced row partition, local problems,
broadcast of the communicator id, and the decomposition the sharded kernels
rely on -- the allreduce(sum) of per-rank partial products K_g' y_g equals
K' y, and each rank's K_g x equals its rows of K x."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import lpgen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_09734_b200 as mp  # binding + partition helpers (no GPU work)
        lp = lpgen.g_rand(301, 517, 9, seed=12)
        prob = mp.Problem.from_lp(lp)
        cuts = mp.row_partition(lp.row_ptr, world)
        r0, r1 = cuts[rank], cuts[rank + 1]
        loc = mp.local_rows(prob, r0, r1)
        # the communicator id: rank 0 creates (any 128 bytes stand in for ncclGetUniqueId on CPU), all receive
        obj = [bytes(np.random.default_rng(0).integers(0, 256, 128, dtype=np.uint8)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        rng = np.random.default_rng(3)
        x, y = rng.normal(size=lp.n), rng.normal(size=lp.m)
        Kl = lpgen.LP(loc.n, loc.m1, loc.m2, np.asarray(loc.row_ptr), np.asarray(loc.col_idx),
                      np.asarray(loc.values), lp.c, np.asarray(loc.q), lp.l, lp.u).dense_K()
        part = torch.from_numpy(Kl.T @ y[r0:r1])          # this rank's K_g' y_g
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        K = lp.dense_K()
        ok = bool(np.allclose(part.numpy(), K.T @ y, rtol=1e-12, atol=1e-12))
        ok &= bool(np.allclose(Kl @ x, (K @ x)[r0:r1], rtol=1e-13, atol=1e-13))
        ok &= loc.m1 == max(0, min(lp.m1 - r0, r1 - r0)) and loc.m1 + loc.m2 == r1 - r0
        nnz = torch.tensor([int(np.asarray(loc.row_ptr)[-1])])
        dist.all_reduce(nnz)
        ok &= int(nnz) == lp.nnz
        out[rank] = (ok, len(obj[0]), r1 - r0)
    finally:
        dist.destroy_process_group()


def test_two_rank_row_sharding_gloo():
    port = _free_port()
    with tmp.Manager() as mgr:
        out = mgr.dict()
        tmp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0][0] and res[1][0], res
    assert res[0][1] == res[1][1] == 128
    assert res[0][2] + res[1][2] == 301


def _worker_cols(rank, world, port, out):
    """Column sharding (m < n, reading 33): each rank's K_{:,g} x_g partial, summed over the ranks,
    is K x; with y replicated, each rank's K_g' y is its columns of K' y; the exchanged vector
    is the m-long one."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_09734_b200 as mp
        lp = lpgen.g_rand(211, 640, 9, seed=13)
        prob = mp.Problem.from_lp(lp)
        ok = mp.shard_axis(lp.m, lp.n) == mp.SHARD_COLS and mp.shard_axis(lp.n, lp.m) == mp.SHARD_ROWS
        ok &= mp.shard_axis(lp.n, lp.n) == mp.SHARD_ROWS
        cuts = mp.col_partition(prob, world)
        c0, c1 = cuts[rank], cuts[rank + 1]
        loc = mp.local_cols(prob, c0, c1)
        rng = np.random.default_rng(4)
        x, y = rng.normal(size=lp.n), rng.normal(size=lp.m)
        Kl = lpgen.LP(loc.n, loc.m1, loc.m2, np.asarray(loc.row_ptr), np.asarray(loc.col_idx),
                      np.asarray(loc.values), np.asarray(loc.c), lp.q, np.asarray(loc.l), np.asarray(loc.u)).dense_K()
        K = lp.dense_K()
        part = torch.from_numpy(Kl @ x[c0:c1])            # this rank's K_{:,g} x_g (m-long)
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        ok &= bool(np.allclose(part.numpy(), K @ x, rtol=1e-12, atol=1e-12))
        ok &= bool(np.allclose(Kl.T @ y, (K.T @ y)[c0:c1], rtol=1e-13, atol=1e-13))
        ok &= bool(np.array_equal(Kl, K[:, c0:c1])) and loc.m1 == lp.m1 and loc.m2 == lp.m2
        ok &= bool(np.array_equal(np.asarray(loc.c), lp.c[c0:c1])) and bool(np.array_equal(np.asarray(loc.q), lp.q))
        nnz = torch.tensor([int(np.asarray(loc.row_ptr)[-1])])
        dist.all_reduce(nnz)
        ok &= int(nnz) == lp.nnz
        out[rank] = (ok, c1 - c0, int(np.asarray(loc.row_ptr)[-1]), part.numel())
    finally:
        dist.destroy_process_group()


def test_two_rank_column_sharding_gloo():
    port = _free_port()
    with tmp.Manager() as mgr:
        out = mgr.dict()
        tmp.spawn(_worker_cols, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0][0] and res[1][0], res
    assert res[0][1] + res[1][1] == 640
    assert abs(res[0][2] - res[1][2]) <= 0.1 * (res[0][2] + res[1][2])   # nnz-balanced
    assert res[0][3] == 211                                             # the exchange is m-long
