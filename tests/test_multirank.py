"""Multi-rank host logic on CPU (world size 2, gloo): lane sharding and the one
exchange step of the method — every rank combines its own lanes with its shard of the
weights (rows a5), the partial sums are summed across ranks (row a6).  The shard of the
weights is libpsp's own host logic (psp_shard_weights, the code psp_set_weights_dense runs
on every rank); the NCCL id that psp_comm_init needs is drawn by libpsp on rank 0 and
broadcast (psp_comm_init itself needs a GPU per rank).  The lanes are the oracle's (this
checks the sharding plan and the reduce semantics, not a kernel); a ladder deliberately
straddles the rank boundary."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2311_11833_b200 import psp
from psp_inputs import config, integer_ladder

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")
import multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _ladders():
    # three 4-lane ladders and one 8-lane ladder: K = 20, so the 2-rank split [0,10), [10,20)
    # cuts the second ladder in half
    return [integer_ladder(2e-3, 2), integer_ladder(1e-3, 2), integer_ladder(3e-3, 2),
            integer_ladder(5e-4, 4)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = config(0).system()
        lad = _ladders()
        eps = np.concatenate([np.ravel([[m, -m] for m in l]) for l in lad])
        K = len(eps)
        kb, ke = psp.shard_range(K, rank, world)
        perm = np.arange(s.n, dtype=np.int32)
        tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
        X, st = oracle.dense_batch(s, perm, eps[kb:ke], tol)
        wp, wl, wv = psp.psp_shard_weights(oracle.ladder_weight_matrix(lad), kb, ke - kb)
        wp2, wl2, wv2 = psp.ladder_weights_csr(lad, k_begin=kb, k_end=ke)   # the binding's own
        assert np.array_equal(wp, wp2) and np.array_equal(wl, wl2)
        assert np.max(np.abs(wv - wv2)) <= 4 * np.finfo(float).eps * np.max(np.abs(wv))
        W = len(wp) - 1
        uid = [psp.psp_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        assert isinstance(uid[0], bytes) and len(uid[0]) == 128
        part = np.zeros((W, 1, s.n))
        for w in range(W):                       # ascending local lane, one fma per term
            for e in range(wp[w], wp[w + 1]):
                part[w] += wv[e] * X[wl[e]]
        t = torch.tensor(part)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        q.put((rank, t.numpy(), (kb, ke), uid[0]))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for K in (1, 7, 20, 65536):
        for world in (1, 2, 3, 8):
            got = [psp.shard_range(K, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == K
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(e - b for b, e in got) - min(e - b for b, e in got) <= 1


def test_two_rank_partial_sums_equal_full_combination():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    assert res[0][2] == (0, 10) and res[1][2] == (10, 20)
    # both ranks hold the same reduced result (and the same communicator id)
    assert np.array_equal(res[0][1], res[1][1])
    assert res[0][3] == res[1][3]
    s = config(0).system()
    lad = _ladders()
    eps = np.concatenate([np.ravel([[m, -m] for m in l]) for l in lad])
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    X, _ = oracle.dense_batch(s, np.arange(s.n, dtype=np.int32), eps, tol)
    full = oracle.combine(oracle.ladder_weight_matrix(lad), X)
    scale = np.abs(full).max()
    # only the summation order differs (reading R16): a few ulp of sum |w_k x_k|
    assert np.max(np.abs(res[0][1] - full)) <= 64 * np.finfo(float).eps * scale
