"""View-sharded training on the GPU (csrc/exchange.cu).

* The exchange kernels against the numpy statement of tests/test_parallel.py:
  three ranks emulated in one process (one glod_xchg context each, rows
  routed by hand): owner-major union, owner buckets, owner sums =
  Σ of the ranks' gradients, parameter replication.
* NCCL inside the library (glod_grad_exchange / glod_param_allgather) on a
  1-rank communicator, driven by the Trainer: the same counters, losses
  and state as the local path with the same render-row source.
* Two ranks as two processes on this one GPU (NCCL refuses a duplicate
  device, so the group runs gloo around the same device phases): different
  views per rank; every rank ends with identical attribute values, and the
  first step's owner sums equal the sum of both ranks' gradients."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

from paper_2507_01110_b200.core import SECTIONS, AttributeArrays  # noqa: E402
from paper_2507_01110_b200.parallel import DevicePhases, make_exchange  # noqa: E402

from .test_parallel import F, row_major, union_layout  # noqa: E402
from .test_train_gpu import make_case  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_exchange_kernels_match_layout():
    N, cap = 3, 5000
    rng = np.random.default_rng(7)
    nodes = [rng.choice(cap, size=n, replace=False).astype(np.int32) for n in (700, 1, 1300)]
    grads = [rng.normal(size=23 * x.size) for x in nodes]
    Rmax = max(x.size for x in nodes)
    ids_all = np.full(N * Rmax, -1, np.int32)
    for r, x in enumerate(nodes):
        ids_all[r * Rmax:r * Rmax + x.size] = x
    U, off = union_layout(ids_all, N)
    ctx = [DevicePhases(N, r, cap) for r in range(N)]
    for r in range(N):
        got_off = ctx[r].union(torch.from_numpy(ids_all).cuda())
        assert got_off == [int(v) for v in off]
        np.testing.assert_array_equal(ctx[r].union_ids().cpu().numpy(), U)
    sends = []
    for r in range(N):
        rows, counts = ctx[r].pack(torch.from_numpy(nodes[r]).cuda(), torch.from_numpy(grads[r]).cuda(),
                                   nodes[r].size)
        st = np.concatenate([[0], np.cumsum(counts)])
        sends.append([rows[st[o]:st[o + 1]].clone() for o in range(N)])
    want = np.zeros((U.size, F))
    index = {int(i): j for j, i in enumerate(U)}
    for x, g in zip(nodes, grads):
        gm = row_major(g, x.size)
        for k, i in enumerate(x):
            want[index[int(i)]] += gm[k]
    records = torch.arange(cap, dtype=torch.float64, device="cuda")[:, None].repeat(1, 72).contiguous()
    recs = [records.clone() for _ in range(N)]
    for o in range(N):
        n = ctx[o].begin_accumulate()
        assert n == off[o + 1] - off[o]
        for s in range(N):                       # source by source
            ctx[o].accumulate(sends[s][o])
        ids, G, n2 = ctx[o].owned()
        np.testing.assert_array_equal(ids.cpu().numpy(), U[off[o]:off[o + 1]])
        np.testing.assert_allclose(row_major(G.cpu().numpy(), n), want[off[o]:off[o + 1]], rtol=1e-12,
                                   atol=1e-12)
        recs[o][ids.long(), :F] += 1000.0 * (o + 1)            # the owner's "ADAM"
    # replication: every rank gets every owner's chunk
    packed = [ctx[o].pack_params(recs[o], 72).clone() for o in range(N)]
    full = packed[0].clone()
    for o in range(N):
        full[off[o]:off[o + 1]] = packed[o][off[o]:off[o + 1]]
    for r in range(N):
        ctx[r].pack_params(recs[r], 72).copy_(full)
        ctx[r].scatter_params(recs[r], 72)
    for r in range(1, N):
        assert torch.equal(recs[r][:, :F], recs[0][:, :F])
    own = (U >> 5) % N
    np.testing.assert_array_equal(recs[0][:, 0].cpu().numpy()[U], U + 1000.0 * (own + 1))


def test_nccl_exchange_path_matches_local():
    """glod_grad_exchange / glod_param_allgather over a 1-rank NCCL
    communicator inside the Trainer, against the local path with the same
    render-row source (SPT rows from the master records, as in sharded
    mode): identical counters and losses, and the same parameters, moments
    and step counts (one source: the owner sum is an exact copy; ADAM is
    elementwise)."""
    from .test_train_gpu import same_state
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        a, _, lrs = make_case()
        a.spt_from_master = True
        b, _, _ = make_case()
        b.distributed = b.spt_from_master = True
        b.xchg = make_exchange(b.scene.cap)
        assert type(b.xchg).__name__ == "NcclExchange"
        for it in range(1, 7):
            ra, rb = a.train_step(it), b.train_step(it)
            for k in ("view", "gaussians_rendered", "gaussians_loaded_from_store", "cache_hits",
                      "bytes_streamed"):
                assert ra[k] == rb[k], (it, k)
            assert abs(ra["loss"] - rb["loss"]) <= 1e-9 * abs(ra["loss"]), it
            st = b.xchg.stats()
            assert st["union"] == st["owned"] == ra["gaussians_rendered"]
        torch.cuda.synchronize()
        assert same_state(a.scene.params, b.scene.params)
        assert same_state(a.scene.mv, b.scene.mv)
        assert torch.equal(a.scene.step, b.scene.step)
    finally:
        dist.destroy_process_group()


def _two_rank_worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        tr, _, _ = make_case()
        tr.rng = np.random.default_rng(100 + rank)      # each rank walks its own views
        assert tr.distributed and type(tr.xchg).__name__ == "GroupExchange"
        unions = []
        for it in range(1, 6):
            rec = tr.train_step(it)
            assert np.isfinite(rec["loss"])
            if it == 1:
                R = rec["gaussians_rendered"]
                np.save(os.path.join(out_dir, f"rows{rank}.npy"), tr._last_rows.cpu().numpy())
                np.save(os.path.join(out_dir, f"grads{rank}.npy"), tr._last_grads[:23 * R].cpu().numpy())
                ids, G, n = tr.xchg.owned()
                np.save(os.path.join(out_dir, f"owned{rank}.npy"), ids.cpu().numpy())
                np.save(os.path.join(out_dir, f"ownedg{rank}.npy"), G.cpu().numpy())
            unions.append(tr.xchg.stats()["union"])
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"params{rank}.npy"), tr.scene.records[:, :F].cpu().numpy())
        np.save(os.path.join(out_dir, f"unions{rank}.npy"), np.array(unions))
    finally:
        dist.destroy_process_group()


def test_two_rank_view_sharded_training(tmp_path):
    import torch.multiprocessing as mp
    port = _port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_two_rank_worker, args=(r, port, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    a, b = np.load(tmp_path / "params0.npy"), np.load(tmp_path / "params1.npy")
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    ua, ub = np.load(tmp_path / "unions0.npy"), np.load(tmp_path / "unions1.npy")
    assert np.array_equal(ua, ub) and ua.min() > 0
    # step 1: owner sums = Σ of both ranks' per-view gradients
    rows = [np.load(tmp_path / f"rows{r}.npy") for r in range(2)]
    grads = [np.load(tmp_path / f"grads{r}.npy") for r in range(2)]
    U, off = union_layout(np.concatenate(rows), 2)
    want = np.zeros((U.size, F))
    index = {int(i): j for j, i in enumerate(U)}
    for x, g in zip(rows, grads):
        gm = row_major(g, x.size)
        for k, i in enumerate(x):
            want[index[int(i)]] += gm[k]
    for r in range(2):
        ids = np.load(tmp_path / f"owned{r}.npy")
        np.testing.assert_array_equal(ids, U[off[r]:off[r + 1]])
        G = np.load(tmp_path / f"ownedg{r}.npy")
        np.testing.assert_allclose(row_major(G, ids.size), want[off[r]:off[r + 1]], rtol=1e-12, atol=1e-300)
