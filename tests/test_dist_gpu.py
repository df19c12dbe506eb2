"""The view-sharded training path on one GPU: a 1-rank NCCL group with the
union gradient exchange forced on must train like the local path (same
counters; parameters equal up to the f32 wire rounding of the gradients)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

from paper_2507_01110_b200.core import SECTIONS, AttributeArrays  # noqa: E402

from .test_train_gpu import make_case  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_union_allreduce_path_matches_local():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        a, _, lrs = make_case()
        b, _, _ = make_case()
        b.distributed = True
        for it in range(1, 6):
            ra, rb = a.train_step(it), b.train_step(it)
            for k in ("view", "gaussians_rendered", "gaussians_loaded_from_store", "cache_hits",
                      "bytes_streamed"):
                assert ra[k] == rb[k], (it, k)
            assert abs(ra["loss"] - rb["loss"]) <= 1e-4 * abs(ra["loss"])
        assert b._last_union[0].numel() == ra["gaussians_rendered"]
        pa = AttributeArrays.from_packed(a.scene.params.cpu().numpy(), a.scene.cap)
        pb = AttributeArrays.from_packed(b.scene.params.cpu().numpy(), b.scene.cap)
        for name, _ in SECTIONS:
            x, y = getattr(pa, name), getattr(pb, name)
            lr = lrs[name] if name not in ("scales", "opacities") else 1.0
            assert np.all(np.abs(x - y) <= 5 * 2.5 * lr * np.maximum(1.0, np.abs(x)) + 1e-12), name
            assert np.mean(np.abs(x - y) <= 1e-5 * np.maximum(1.0, np.abs(x))) > 0.98, name
        assert torch.equal(a.scene.step, b.scene.step)
    finally:
        dist.destroy_process_group()


def test_union_refresh_updates_resident_blocks():
    """View sharding: rows another rank updated reach this rank's resident
    cache blocks (and mark those entries dirty for write-back)."""
    from paper_2507_01110_b200 import _lib
    tr, _, _ = make_case()
    for it in range(1, 4):
        tr.train_step(it)
    torch.cuda.synchronize()
    sc = tr.scene
    flat = sc.hspt.flat_records()
    entries = tr.cache.entries()
    assert entries
    sid, _, P, addr, _ = entries[0]
    o = int(flat["offset"][sid])
    nodes = flat["nodes"][o:o + P]
    pick = nodes[::max(1, P // 7)].astype(np.int64)
    rng = np.random.default_rng(5)
    view = sc.params.view(-1)
    off = 0
    for name, cols in SECTIONS:      # new master values for the picked rows
        sec = view[off * sc.cap:(off + cols) * sc.cap].view(sc.cap, cols)
        sec[torch.from_numpy(pick).cuda()] = torch.from_numpy(rng.normal(size=(pick.size, cols))).cuda()
        off += cols
    ids = torch.from_numpy(pick.astype(np.int32)).cuda()
    tr._refresh_union(ids)
    torch.cuda.synchronize()
    blk = AttributeArrays.from_packed(tr.cache.read_block(addr, P), P)
    master = AttributeArrays.from_packed(sc.params.cpu().numpy(), sc.cap)
    pos = np.array([np.nonzero(nodes == n)[0][0] for n in pick])
    for name, _ in SECTIONS:
        np.testing.assert_array_equal(getattr(blk, name)[pos], getattr(master, name)[pick])
    assert tr._h_touched.numpy()[sid] == 1
    tr.cache.mark_dirty(tr._h_touched.numpy())
    assert [e for e in tr.cache.entries() if e[0] == sid][0][4]


def _two_rank_worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2507_01110_b200.parallel import union_of_rows
        tr, _, _ = make_case()
        tr.rng = np.random.default_rng(100 + rank)      # each rank walks its own views
        assert tr.distributed
        unions = []
        for it in range(1, 6):
            rec = tr.train_step(it)
            assert np.isfinite(rec["loss"])
            ids, GU = tr._last_union
            unions.append(int(ids.numel()))
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"params{rank}.npy"), tr.scene.records.cpu().numpy())
        np.save(os.path.join(out_dir, f"unions{rank}.npy"), np.array(unions))
    finally:
        dist.destroy_process_group()


def test_two_rank_view_sharded_training(tmp_path):
    """Two ranks (two processes sharing this GPU, gloo transport) train
    different views with the union gradient exchange: after every step the
    replicated ADAM leaves both ranks with bit-identical node records
    (params, moments, steps)."""
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
