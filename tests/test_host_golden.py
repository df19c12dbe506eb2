"""Host-kept pieces against the reference's own outputs (golden vectors):
the view scheduler's exact sequence and the device-cache decision logic,
plus the pinned store's slot layout and byte counters.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_01110_b200.cache import CacheConfig, CacheEntry, DeviceCache, OverBudgetError
from paper_2507_01110_b200.core import AttributeArrays
from paper_2507_01110_b200.scheduler import build_view_graph, next_view
from paper_2507_01110_b200.store import AttributeBlock, HostStore, InvalidBlockError, NotFoundError

from .conftest import golden


def test_scheduler_sequence_matches_reference():
    d = golden("scheduler_cases.npz")
    for c in range(int(d["n_cases"])):
        g = build_view_graph(d[f"s{c}_pos"], k=int(d[f"s{c}_k"]),
                             random_every=int(d[f"s{c}_random_every"]))
        np.testing.assert_array_equal(g.neighbors, d[f"s{c}_neighbors"])
        np.testing.assert_array_equal(g.weights, d[f"s{c}_weights"])
        r = np.random.default_rng(100 + c)
        cur, seq = 0, []
        for it in range(1, 200):
            cur = next_view(g, cur, it, r)
            seq.append(cur)
        np.testing.assert_array_equal(seq, d[f"s{c}_seq"])


def test_device_cache_matches_reference_traces():
    d = golden("cache_cases.npz")
    for c in range(int(d["n_cases"])):
        cache = DeviceCache(config=CacheConfig(budget_bytes=int(d[f"c{c}_budget"]),
                                               flush_interval=int(d[f"c{c}_flush"])))
        ops = d[f"c{c}_ops"]
        lens = d[f"c{c}_reslen"]
        res = np.split(d[f"c{c}_res"], np.cumsum(lens)[:-1])
        for (kind, a, dd, nb, dirty), want in zip(ops, res):
            kind, a = int(kind), int(a)
            if kind == 0:
                got = [int(cache.lookup(a, float(dd)) is not None)]
            elif kind == 1:
                ev = cache.insert(CacheEntry(spt_id=a, cached_distance=float(dd), prefix_len=0,
                                             block=None, nbytes=int(nb), dirty=bool(dirty)))
                got = [e[0] for e in ev]
            else:
                got = [e[0] for e in cache.tick_and_maybe_flush(a)]
            got = got + [-7] + cache.resident_ids() + [-8, cache.resident_bytes, cache.hits,
                                                        cache.misses]
            assert got == list(want)


def test_cache_known_answers():
    """cache ratio examples (test_cache.py:40-60) and the over-budget error."""
    c = DeviceCache(config=CacheConfig(budget_bytes=10_000, d_min=0.9, d_max=1.5))
    c.insert(CacheEntry(7, 100.0, 1, None, 92))
    assert c.lookup(7, 120.0) is not None and c.lookup(7, 80.0) is None
    assert c.lookup(7, 90.0) is not None and c.lookup(7, 150.0) is not None
    z = DeviceCache(config=CacheConfig(budget_bytes=100))
    z.insert(CacheEntry(1, 0.0, 1, None, 92))
    assert z.lookup(1, 0.0) is not None and z.lookup(1, 1e-9) is None
    with pytest.raises(OverBudgetError):
        z.insert(CacheEntry(2, 1.0, 2, None, 184))
    with pytest.raises(ValueError):
        CacheConfig(budget_bytes=1, d_min=1.1, d_max=1.4)


def _small_scene():
    from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene
    return designed_scene(SceneSpec(n_leaves=3000, spt_leaves=128, seed=4, relabel=False))


def test_host_store_layout_and_counters():
    h, hs, _ = _small_scene()
    st = HostStore(h, hs, pin=False)
    flat = hs.flat_records()
    # slot order: non-SPT nodes ascending, then each SPT's records (store.py:143-154)
    nonspt = np.setdiff1d(np.arange(h.capacity), flat["nodes"])
    np.testing.assert_array_equal(st.slot_to_node[:nonspt.size], nonspt)
    np.testing.assert_array_equal(st.slot_to_node[nonspt.size:], flat["nodes"])
    assert st.bytes_per_gaussian == 92
    sid = len(hs.spts) // 2
    P = int(flat["count"][sid]) // 2
    blk = st.load_spt_prefix(sid, P)
    assert st.attribute_bytes_read == 92 * P
    nodes = hs.spts[sid].nodes[:P]
    np.testing.assert_array_equal(blk.attrs.means, h.attrs.means[nodes].astype(np.float32))
    np.testing.assert_array_equal(blk.attrs.opacities, h.attrs.opacities[nodes].astype(np.float32))
    # write-back round trip
    blk.attrs.means = blk.attrs.means + 1.0
    st.write_back(blk)
    again = st.load_spt_prefix(sid, P)
    np.testing.assert_array_equal(again.attrs.means, blk.attrs.means.astype(np.float32))
    with pytest.raises(InvalidBlockError):
        st.load_spt_prefix(sid, int(flat["count"][sid]) + 1)
    with pytest.raises(NotFoundError):
        st.load_spt_prefix(len(hs.spts), 1)
    rep = st.memory_report(60_000_000)
    assert rep["attribute_bytes_per_gaussian"] == 92 and rep["optimizer_bytes_per_gaussian"] == 184
    assert rep["spt_metadata_bytes_per_gaussian"] == 12 and rep["training_bytes_per_gaussian"] < 800
