"""The native cache (csrc/cache_table.cu) against the Python mirror of
cache.DeviceCache, which itself is pinned to the reference's traces
(tests/test_host_golden.py).  Random per-view step sequences; after every
step the LRU order, cached distances, prefixes, dirty flags, counters and
the per-item outputs must agree exactly, and every freshly loaded block
must hold the store's rows."""
from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2507_01110_b200.cache import CacheConfig, CacheEntry, DeviceCache, NativeCache, OverBudgetError  # noqa: E402
from paper_2507_01110_b200.core import SECTIONS, AttributeArrays  # noqa: E402
from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene  # noqa: E402
from paper_2507_01110_b200.store import HostStore  # noqa: E402


def _py_step(c: DeviceCache, ids, d, P):
    out = []
    loaded = 0
    for sid, dd, pp in zip(ids, d, P):
        e = c.lookup(int(sid), float(dd))
        if e is None:
            e = CacheEntry(int(sid), float(dd), int(pp), None, int(pp) * 92)
            c.insert(e)
            loaded += int(pp)
        out.append((e.cached_distance, e.prefix_len))
    return out, loaded


@pytest.mark.parametrize("seed,budget_frac,flush", [(0, 0.2, 5), (1, 0.6, 3), (2, 1.5, 100)])
def test_native_cache_matches_mirror(seed, budget_frac, flush):
    h, hs, _ = designed_scene(SceneSpec(n_leaves=4000, spt_leaves=128, seed=seed, relabel=False))
    st = HostStore(h, hs)
    S = len(hs.spts)
    counts = hs.flat_records()["count"]
    budget = int(budget_frac * counts.sum() * 92 / 4)
    cfg = CacheConfig(budget_bytes=max(budget, int(counts.max()) * 92), flush_interval=flush)
    nat, py = NativeCache(cfg, st), DeviceCache(config=cfg)
    rng = np.random.default_rng(seed)
    base = rng.uniform(5, 50, S)
    for it in range(1, 40):
        k = int(rng.integers(1, S + 1))
        ids = np.sort(rng.choice(S, k, replace=False)).astype(np.int32)
        d = base[ids] * rng.choice([1.0, 1.1, 1.3, 1.6, 0.7], k)
        if it % 9 == 0:
            d[0] = 0.0
        P = np.maximum(1, (counts[ids] * rng.uniform(0.2, 1.0, k)).astype(np.int32))
        dist = np.zeros(k, np.float64)
        blk = np.zeros(k, np.uint64)
        rows = np.zeros(k, np.int64)
        loaded, hits = nat.step(ids, d, P, dist, blk, rows)
        want, want_loaded = _py_step(py, ids, d, P)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(dist, [w[0] for w in want])
        np.testing.assert_array_equal(rows, [w[1] for w in want])
        assert loaded == want_loaded
        # a block handed out this step holds the store's rows (nothing written yet)
        j = int(rng.integers(k))
        got = nat.read_block(int(blk[j]), int(rows[j]))
        ga = AttributeArrays.from_packed(got, int(rows[j]))
        ref = st.load_spt_prefix(int(ids[j]), int(rows[j])).attrs
        for name, _ in SECTIONS:
            np.testing.assert_array_equal(getattr(ga, name), np.asarray(getattr(ref, name), np.float64))
        nat.end_step(it, mark_dirty=True)
        for sid in ids:
            e = py.entries.get(int(sid))
            if e is not None:
                e.dirty = True
        py.tick_and_maybe_flush(it)
        ents = nat.entries()
        assert [e[0] for e in ents] == py.resident_ids()
        assert [(e[1], e[2], e[4]) for e in ents] == \
            [(e.cached_distance, e.prefix_len, e.dirty) for e in py.entries.values()]
        s = nat.stats()
        assert (s["hits"], s["misses"], s["resident_bytes"]) == (py.hits, py.misses, py.resident_bytes)
    torch.cuda.synchronize()


def test_native_cache_over_budget():
    h, hs, _ = designed_scene(SceneSpec(n_leaves=2000, spt_leaves=128, seed=5, relabel=False))
    st = HostStore(h, hs)
    nat = NativeCache(CacheConfig(budget_bytes=92 * 3), st)
    z = np.zeros(1)
    with pytest.raises(OverBudgetError):
        nat.step(np.array([0], np.int32), np.array([1.0]), np.array([4], np.int32), z,
                 np.zeros(1, np.uint64), np.zeros(1, np.int64))
    # the error leaves no partial state: an over-budget SPT after ones that
    # fit raises before anything is inserted, evicted or counted
    nat.step(np.array([1], np.int32), np.array([1.0]), np.array([2], np.int32), z,
             np.zeros(1, np.uint64), np.zeros(1, np.int64))
    before, stats = nat.entries(), nat.stats()
    with pytest.raises(OverBudgetError):
        nat.step(np.array([2, 3, 0], np.int32), np.array([1.0, 1.0, 1.0]), np.array([1, 1, 4], np.int32),
                 np.zeros(3), np.zeros(3, np.uint64), np.zeros(3, np.int64))
    assert nat.entries() == before
    after = nat.stats()
    assert (after["hits"], after["misses"], after["loaded_rows"]) == (stats["hits"], stats["misses"],
                                                                     stats["loaded_rows"])


def _write_block(address: int, values: np.ndarray):
    from cuda.bindings import runtime as rt
    v = np.ascontiguousarray(values, dtype=np.float64)
    err, = rt.cudaMemcpy(address, v.ctypes.data, v.nbytes, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
    assert int(err) == 0


def _write_block_async(address: int, values: np.ndarray):
    """cudaMemcpyAsync on torch's current stream (the one the cache uses)."""
    from cuda.bindings import runtime as rt
    err, = rt.cudaMemcpyAsync(address, values.ctypes.data, values.nbytes,
                              rt.cudaMemcpyKind.cudaMemcpyHostToDevice,
                              torch.cuda.current_stream().cuda_stream)
    assert int(err) == 0


@pytest.mark.parametrize("interleaved", [True, False])
@pytest.mark.parametrize("seed,budget_frac", [(3, 0.15), (4, 0.4)])
def test_native_cache_block_contents(seed, budget_frac, interleaved):
    """Block and store *contents* through evictions, write-backs, reloads of
    blocks evicted earlier in the same step (overlay path) and flushes,
    against a numpy mirror of the reference's load → insert → write_back
    order (trainer.py:329-345, store.py:314-333).  Blocks rendered in a step
    are modified between steps (the ADAM refresh) so every write-back
    carries new values.  Both store layouts: interleaved rows (one copy per
    prefix) and section-major (six per prefix)."""
    h, hs, _ = designed_scene(SceneSpec(n_leaves=4000, spt_leaves=128, seed=seed, relabel=False))
    st = HostStore(h, hs, interleaved=interleaved)
    S = len(hs.spts)
    counts = hs.flat_records()["count"]
    cfg = CacheConfig(budget_bytes=max(int(budget_frac * counts.sum() * 92 / 3), int(counts.max()) * 92),
                      flush_interval=11)
    nat, py = NativeCache(cfg, st), DeviceCache(config=cfg)
    store = [s.numpy().copy() for s in st.sections]
    cols = [c for _, c in SECTIONS]

    def load(sid, P):
        sl = st.spt_slot_start(sid)
        return np.concatenate([sec[sl:sl + P].reshape(-1).astype(np.float64) for sec in store])

    def write_back(sid, blk):
        sl = st.spt_slot_start(sid)
        P = blk.size // 23
        off = 0
        for k, c in enumerate(cols):
            store[k][sl:sl + P] = blk[off:off + c * P].reshape(store[k][sl:sl + P].shape).astype(np.float32)
            off += c * P

    rng = np.random.default_rng(seed)
    base = rng.uniform(5, 50, S)
    for it in range(1, 30):
        k = int(rng.integers(S // 2, S + 1))
        ids = np.sort(rng.choice(S, k, replace=False)).astype(np.int32)
        d = base[ids] * rng.choice([1.0, 1.2, 1.6, 0.6], k)
        P = np.maximum(1, (counts[ids] * rng.uniform(0.3, 1.0, k)).astype(np.int32))
        dist = np.zeros(k, np.float64)
        blk = np.zeros(k, np.uint64)
        rows = np.zeros(k, np.int64)
        nat.step(ids, d, P, dist, blk, rows)
        for sid, dd, pp in zip(ids, d, P):
            e = py.lookup(int(sid), float(dd))
            if e is None:
                e = CacheEntry(int(sid), float(dd), int(pp), load(int(sid), int(pp)), int(pp) * 92)
                for esid, eblk in py.insert(e):
                    write_back(esid, eblk)
        # blocks rendered this step but evicted later in it are still
        # refreshed by this step's ADAM (main stream, no host sync): their
        # write-back must have read them first (the mirror keeps the old values)
        keep = []
        for j, sid in enumerate(ids):
            if py.entries.get(int(sid)) is None:
                junk = np.full(23 * int(rows[j]), 7.0)
                keep.append(junk)
                _write_block_async(int(blk[j]), junk)
        torch.cuda.synchronize()
        for j, sid in enumerate(ids):
            e = py.entries.get(int(sid))
            if e is None:
                continue
            np.testing.assert_array_equal(nat.read_block(int(blk[j]), int(rows[j])), e.block,
                                          err_msg=f"step {it} spt {sid}")
            # the step's ADAM refresh: new values in every rendered block
            e.block = e.block + rng.normal(0, 1e-3, e.block.size)
            _write_block(int(blk[j]), e.block)
        nat.end_step(it, mark_dirty=True)
        for sid in ids:
            e = py.entries.get(int(sid))
            if e is not None:
                e.dirty = True
        for esid, eblk in py.tick_and_maybe_flush(it):
            write_back(esid, eblk)
        torch.cuda.synchronize()
        for k_, sec in enumerate(st.sections):
            np.testing.assert_array_equal(sec.numpy(), store[k_], err_msg=f"store after step {it}")


@pytest.mark.parametrize("interleaved", [True, False])
def test_store_transfer_capi(interleaved):
    """glod_store_load_prefixes / glod_store_write_back (the zero-copy
    public transfers, store.py:314-333) on both store layouts: loaded blocks
    hold f64(store rows) section-major; written-back blocks land as f32 in
    the right slots and nothing else changes."""
    import ctypes as C
    from paper_2507_01110_b200 import _lib
    h, hs, _ = designed_scene(SceneSpec(n_leaves=3000, spt_leaves=128, seed=7, relabel=False))
    st = HostStore(h, hs, interleaved=interleaved)
    counts = hs.flat_records()["count"]
    rng = np.random.default_rng(0)
    sids = rng.choice(len(counts), 6, replace=False)
    P = [int(max(1, counts[s] * f)) for s, f in zip(sids, rng.uniform(0.2, 1.0, 6))]
    blocks = [torch.zeros(23 * p + (p + 63) // 64, dtype=torch.float64, device="cuda") for p in P]
    items = (_lib.PrefixItem * 6)()
    acc = 0
    for j, (s, p) in enumerate(zip(sids, P)):
        items[j].slot_start = st.spt_slot_start(int(s))
        items[j].rows = p
        items[j].elem_start = acc
        items[j].block = blocks[j].data_ptr()
        acc += 23 * p
    ditems = torch.frombuffer(bytearray(bytes(items)), dtype=torch.uint8).cuda()
    view = st.device_view()
    L = _lib.lib()
    _lib.check(L.glod_store_load_prefixes(C.byref(view), _lib.ptr(ditems), 6, acc, _lib.stream_ptr()))
    torch.cuda.synchronize()
    host = [s.numpy().copy() for s in st.sections]
    for j, (s, p) in enumerate(zip(sids, P)):
        sl = st.spt_slot_start(int(s))
        want = np.concatenate([sec[sl:sl + p].reshape(-1).astype(np.float64) for sec in host])
        np.testing.assert_array_equal(blocks[j][:23 * p].cpu().numpy(), want)
    for j, p in enumerate(P):
        blocks[j][:23 * p] = torch.from_numpy(rng.normal(size=23 * p)).cuda()
    _lib.check(L.glod_store_write_back(C.byref(view), _lib.ptr(ditems), 6, acc, _lib.stream_ptr()))
    torch.cuda.synchronize()
    for j, (s, p) in enumerate(zip(sids, P)):
        sl = st.spt_slot_start(int(s))
        b = blocks[j][:23 * p].cpu().numpy().astype(np.float32)
        off = 0
        for k, (_, c) in enumerate(SECTIONS):
            host[k][sl:sl + p] = b[off:off + c * p].reshape(host[k][sl:sl + p].shape)
            off += c * p
    for k, sec in enumerate(st.sections):
        np.testing.assert_array_equal(sec.numpy(), host[k])


@pytest.mark.gpu
def test_kernel_upload_and_readbacks():
    """glod_upload / glod_readback / glod_readback_multi (kernel copies
    through mapped pinned memory): exact bytes, stream-ordered, odd sizes,
    unaligned pinned sources fall back to cudaMemcpyAsync."""
    from paper_2507_01110_b200 import _lib
    rng = np.random.default_rng(0)
    for n in (1, 7, 1000, 123457):
        h = torch.from_numpy(rng.integers(0, 2 ** 31, n, dtype=np.int64)).pin_memory()
        d = torch.empty(n, dtype=torch.int64, device="cuda")
        _lib.upload(d, h)
        back = torch.empty(n, dtype=torch.int64).pin_memory()
        _lib.readback(back, d)
        torch.cuda.synchronize()
        assert torch.equal(back, h)
    srcs = [torch.arange(k, dtype=torch.int32, device="cuda") * (k + 1) for k in (4, 33, 1024, 70000)]
    dsts = [torch.empty(s.numel(), dtype=torch.int32).pin_memory() for s in srcs]
    _lib.readback_multi(list(zip(dsts, srcs)))
    torch.cuda.synchronize()
    for s, dd in zip(srcs, dsts):
        assert torch.equal(dd, s.cpu())
