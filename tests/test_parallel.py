"""Multi-process (gloo, world_size 2, CPU) test of the sparse gradient
exchange used for view-sharded training: the union of touched nodes is
identical on every rank and the reduced gradient of each node equals the
sum of the per-rank (per-view) gradients."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01110_b200.parallel import sparse_grad_allreduce
    rng = np.random.default_rng(100 + rank)
    R = 50 + 17 * rank
    nodes = rng.choice(200, size=R, replace=False).astype(np.int32)   # unique per view
    grads = rng.normal(size=23 * R)
    U, GU = sparse_grad_allreduce(torch.from_numpy(nodes), torch.from_numpy(grads), R)
    results[rank] = (nodes, grads, U.numpy(), GU.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sparse_grad_allreduce_gloo():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    (n0, g0, U0, G0), (n1, g1, U1, G1) = results[0], results[1]
    np.testing.assert_array_equal(U0, U1)
    np.testing.assert_array_equal(U0, np.union1d(n0, n1))
    np.testing.assert_array_equal(G0, G1)
    # expected: per-section sums over ranks at each union node
    cols = [3, 3, 4, 1, 3, 9]
    nU = U0.size
    want = np.zeros(23 * nU)
    for nodes, grads in ((n0, g0), (n1, g1)):
        R = nodes.size
        pos = np.searchsorted(U0, nodes)
        off = 0
        for c in cols:
            src = grads[off * R:(off + c) * R].reshape(R, c)
            dst = want[off * nU:(off + c) * nU].reshape(nU, c)
            np.add.at(dst, pos, src)
            off += c
    np.testing.assert_allclose(G0, want, rtol=1e-6, atol=1e-6)   # f32 wire format
