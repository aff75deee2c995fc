"""Row-sharded (multi-GPU) host logic on CPU with torch.distributed/gloo, world 2.

The engine shards A by rows and follows every reduction over the row index
with an allreduce (comm.cu). These tests run the same decomposition with
the oracle as the per-rank compute and gloo as the collective, and check it
reproduces the unsharded reference: Gram, column means, total variance,
A^T Y, the whole randomized range finder (CholeskyQR on an allreduced Gram)
and truncated PCA's K. They also exercise the NCCL-id bootstrap that
bench.py uses (rank 0 creates the id, torch.distributed broadcasts it).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard_rows(m, world, rank):
    """Row range of `rank` (contiguous, first m % world ranks get one more)."""
    base, extra = divmod(m, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _worker(rank, port, out_q):
    import torch
    import torch.distributed as dist

    from oracle.pyoracle import Oracle
    from tests.datagen import make_matrix
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        port_o = Oracle("port")

        def allreduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            return t.numpy().reshape(x.shape, order="C")

        a = make_matrix(1203, 40, "c1", seed=5)  # every rank regenerates the same global A
        m, n = a.shape
        r0, r1 = shard_rows(m, WORLD, rank)
        ap = np.asfortranarray(a[r0:r1])
        res = {}
        # NCCL unique-id bootstrap (bench.py): rank 0 creates, all receive the same bytes
        from paper_1906_12085_b200 import _lib
        obj = [_lib.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        res["uid_len"] = len(obj[0])
        # column means over all rows (pca.cpp:37-53 sharded)
        sums = allreduce(ap.sum(axis=0))
        mean = sums / m
        c = np.asfortranarray(ap - mean)
        # total variance and Gram: allreduce of the local parts
        res["total"] = float(allreduce(np.array([(c * c).sum()]))[0])
        g = allreduce(np.ascontiguousarray(port_o.gram(c)))
        res["gram"] = g
        # randomized range finder, sharded: Y_p = A_p Omega; Z = sum A_p^T Y_p; Y_p = A_p Z;
        # CholeskyQR2 on the allreduced Gram; T = sum A_p^T Q_p
        l, q = 40, 2
        om = port_o.gaussian_matrix(n, l, 11)
        y = c @ om
        for _ in range(q):
            z = allreduce(np.ascontiguousarray(c.T @ y))
            y = c @ z
        for _ in range(2):  # CholeskyQR2
            gy = allreduce(np.ascontiguousarray(y.T @ y))
            r = np.linalg.cholesky(gy).T
            y = np.linalg.solve(r.T, y.T).T
        t = allreduce(np.ascontiguousarray(c.T @ y))
        res["sigma_rand"] = np.linalg.svd(t, compute_uv=False)
        res["orth"] = float(np.abs(allreduce(np.ascontiguousarray(y.T @ y)) - np.eye(l)).max())
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def test_shard_rows_partition():
    for m in (1, 7, 1203, 8388608):
        for world in (1, 2, 4, 8):
            spans = [shard_rows(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_sharded_matches_unsharded(sharded, ref):
    from tests.datagen import make_matrix
    a = make_matrix(1203, 40, "c1", seed=5)
    c, _ = ref.center(a, 1)
    for rank in range(WORLD):
        r = sharded[rank]
        assert r["uid_len"] == 128
        assert abs(r["total"] - ref.frobenius_norm_sq(c)) <= 1e-13 * r["total"]
        g_ref = ref.gram(c)
        nrm = np.sqrt(np.diag(g_ref))
        assert np.max(np.abs(r["gram"] - g_ref) / np.outer(nrm, nrm)) <= 1e-14
        s_ref = ref.randomized_pca(c, 40, 2, 11).sigma
        assert np.max(np.abs(r["sigma_rand"] - s_ref) / s_ref) <= 1e-10
        assert r["orth"] <= 1e-13
    # every rank holds the same replicated results
    assert np.array_equal(sharded[0]["gram"], sharded[1]["gram"])
