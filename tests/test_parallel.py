"""Multi-process (gloo, world_size 2, CPU) test of the view-sharded gradient
exchange's collective sequence (parallel.exchange_with_group /
params_with_group): ids all-gather, union, owner buckets shipped point to
point, owner-side sums, owner broadcast of the updated rows.  The device
phases (csrc/exchange.cu) are replaced by `CpuPhases`, a numpy statement of
the same layout (owner(id) = (id >> 5) mod N, U owner-major and sorted
within each owner chunk); tests/test_dist_gpu.py checks the kernels against
the same statement."""
from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

F, ROW = 23, 24
COLS = [3, 3, 4, 1, 3, 9]


def union_layout(ids_all, nranks):
    """Owner-major union: [(owner chunk of sorted ids) for each owner]."""
    ids = np.unique(np.asarray(ids_all, np.int64))
    ids = ids[ids >= 0]
    own = (ids >> 5) % nranks
    chunks = [ids[own == o] for o in range(nranks)]
    off = np.concatenate([[0], np.cumsum([c.size for c in chunks])]).astype(np.int64)
    return np.concatenate(chunks) if chunks else ids, off


def row_major(grads, R):
    """Section-major packed grads (23·R) -> [R, 23]."""
    out, off = [], 0
    for c in COLS:
        out.append(grads[off * R:(off + c) * R].reshape(R, c))
        off += c
    return np.concatenate(out, axis=1)


def section_major(rows):
    n = rows.shape[0]
    parts, off = [], 0
    for c in COLS:
        parts.append(rows[:, off:off + c].reshape(-1))
        off += c
    return np.concatenate(parts) if n else np.zeros(0)


class CpuPhases:
    """numpy statement of the glod_xchg phases on torch CPU tensors."""

    def __init__(self, nranks, rank):
        self.nranks, self.rank = nranks, rank

    def union(self, ids_all):
        self.U, off = union_layout(ids_all.numpy(), self.nranks)
        self.offsets = [int(x) for x in off]
        self.index = {int(i): j for j, i in enumerate(self.U)}
        return self.offsets

    def pack(self, row_node, grads, R):
        ids = row_node.numpy()[:R].astype(np.int64)
        g = row_major(grads.numpy(), R)
        own = (ids >> 5) % self.nranks
        rows, counts = [], []
        for o in range(self.nranks):
            sel = np.nonzero(own == o)[0]
            pos = np.array([self.index[int(i)] - self.offsets[o] for i in ids[sel]], dtype=np.float64)
            rows.append(np.concatenate([pos[:, None], g[sel]], axis=1) if sel.size else np.zeros((0, ROW)))
            counts.append(int(sel.size))
        return torch.from_numpy(np.concatenate(rows)), counts

    def begin_accumulate(self):
        self.n = self.offsets[self.rank + 1] - self.offsets[self.rank]
        self.acc = np.zeros((self.n, F))
        return self.n

    def accumulate(self, rows):
        r = rows.numpy()
        self.acc[r[:, 0].astype(np.int64)] += r[:, 1:]

    def owned(self):
        lo, hi = self.offsets[self.rank], self.offsets[self.rank + 1]
        return self.U[lo:hi], section_major(self.acc), self.n

    def pack_params(self, records, stride):
        self.params = torch.zeros((self.offsets[-1], F), dtype=torch.float64)
        lo, hi = self.offsets[self.rank], self.offsets[self.rank + 1]
        self.params[lo:hi] = records[torch.from_numpy(self.U[lo:hi]), :F]
        return self.params

    def scatter_params(self, records, stride):
        records[torch.from_numpy(self.U), :F] = self.params


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
    from paper_2507_01110_b200.parallel import exchange_with_group, params_with_group
    rng = np.random.default_rng(100 + rank)
    R = 300 + 17 * rank
    cap = 2000
    nodes = rng.choice(cap, size=R, replace=False).astype(np.int32)     # unique per view
    grads = rng.normal(size=23 * R)
    ph = CpuPhases(world, rank)
    n = exchange_with_group(ph, torch.from_numpy(nodes), torch.from_numpy(grads), R)
    ids, G, n2 = ph.owned()
    # owner "ADAM": a rank-specific update of its owned rows; then replicate
    records = torch.from_numpy(np.tile(np.arange(cap, dtype=np.float64)[:, None], (1, 72)))
    records[torch.from_numpy(ids.astype(np.int64)), :F] += 1000.0 * (rank + 1)
    params_with_group(ph, records, 72)
    results[rank] = (nodes, grads, ids, G, n, n2, ph.offsets, records.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_exchange_with_group_gloo():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    r0, r1 = results[0], results[1]
    U, off = union_layout(np.concatenate([r0[0], r1[0]]), world)
    assert r0[6] == r1[6] == [int(x) for x in off]
    want = np.zeros((U.size, F))
    index = {int(i): j for j, i in enumerate(U)}
    for nodes, grads in ((r0[0], r0[1]), (r1[0], r1[1])):
        g = row_major(grads, nodes.size)
        for k, i in enumerate(nodes):
            want[index[int(i)]] += g[k]
    for rank, r in enumerate((r0, r1)):
        ids, G, n, n2 = r[2], r[3], r[4], r[5]
        assert n == n2 == off[rank + 1] - off[rank]
        np.testing.assert_array_equal(ids, U[off[rank]:off[rank + 1]])
        assert np.all(((ids >> 5) % world) == rank)
        np.testing.assert_allclose(row_major(G, n), want[off[rank]:off[rank + 1]], rtol=1e-12, atol=1e-12)
    # replication: both ranks hold every owner's update of U, nothing else moved
    a, b = r0[7], r1[7]
    np.testing.assert_array_equal(a[:, :F], b[:, :F])
    own = (U >> 5) % world
    np.testing.assert_array_equal(a[U, 0], U + 1000.0 * (own + 1))
    rest = np.setdiff1d(np.arange(a.shape[0]), U)
    np.testing.assert_array_equal(a[rest, 0], rest)
