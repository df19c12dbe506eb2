"""GPU parity of the LoD cut (K1/K2) through the C-ABI: bit-exact against
the reference's own outputs (golden vectors) and against the C oracle on
larger generated scenes."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import glod_oracle as O  # noqa: E402
from paper_2507_01110_b200 import hspt as H  # noqa: E402
from paper_2507_01110_b200.core import Frustum, LodConfig  # noqa: E402
from paper_2507_01110_b200.spt import Spt, cut_spt  # noqa: E402

from .conftest import golden, lod_files  # noqa: E402
from .helpers import (assert_rs_equal, camera_of, golden_rs, hierarchy_of, hspt_of,  # noqa: E402
                      rs_dict, view_cfg)


@pytest.mark.parametrize("path", lod_files(), ids=lambda p: p.stem)
def test_cut_hspt_bitexact_vs_reference(path):
    d = np.load(path)
    h, hs = hierarchy_of(d), hspt_of(d)
    for v in range(int(d["n_views"])):
        cam = camera_of(d, f"v{v}_")
        rs = H.cut_hspt(hs, h, cam, view_cfg(d, v), cull=bool(d[f"v{v}_cull"]))
        assert_rs_equal(rs_dict(rs), golden_rs(d, v), where=f"{path.stem} v{v}")


@pytest.mark.parametrize("path", lod_files()[:12], ids=lambda p: p.stem)
def test_bfs_cut_bitexact_vs_reference(path):
    d = np.load(path)
    h = hierarchy_of(d)
    for v in range(int(d["n_views"])):
        cam = camera_of(d, f"v{v}_")
        fr = Frustum(planes=d[f"v{v}_planes"]) if d[f"v{v}_cull"] else None
        got = H.bfs_cut(h, cam, view_cfg(d, v), frustum=fr)
        np.testing.assert_array_equal(got.node_ids, d[f"v{v}_bfs"])


def test_cut_spt_bitexact_vs_reference():
    d = golden("spt_cases.npz")
    for k in range(int(d["n_cases"])):
        p = f"c{k}_"
        spt = Spt(root=int(d[p + "root"]), root_center=np.zeros(3), nodes=d[p + "nodes"],
                  key_self=d[p + "key_self"], key_parent=d[p + "key_parent"])
        pl, sel = cut_spt(spt, float(d[p + "d"]))
        assert pl == int(d[p + "prefix"]), k
        np.testing.assert_array_equal(sel, d[p + "sel"])


@pytest.mark.parametrize("n_leaves,spt_leaves", [(20_000, 512), (300_000, 2048)])
def test_cut_hspt_vs_oracle_generated(n_leaves, spt_leaves):
    from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene, orbit_views, scene_extent
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=n_leaves, spt_leaves=spt_leaves, seed=5))
    E = scene_extent(n_leaves)
    cams = orbit_views(6, 1.6 * E, 0.7 * E, resolution=(1920, 1080), seed=3, jitter=0.3,
                       target_jitter=0.2 * E)
    flat = hs.flat_records()
    kind = np.full(h.capacity, -1, np.int32)
    kind[flat["roots"]] = np.arange(flat["roots"].size)
    kind[hs.passthrough_roots] = -2
    for i, cam in enumerate(cams):
        for cull in (True, False):
            rs = H.cut_hspt(hs, h, cam, cfg, cull=cull)
            want = O.cut_hspt(h.root, h.children, kind, h.attrs.means, h.attrs.scales,
                              flat["offset"], flat["count"], flat["roots"], flat["centers"],
                              flat["key_self"], flat["key_parent"], flat["nodes"], cam.position,
                              cfg.threshold, cfg.metric_code,
                              Frustum.from_camera(cam).planes if cull else None)
            assert_rs_equal(rs_dict(rs), want, where=f"view {i} cull={cull}")
            assert len(rs) > 100


def test_cut_spt_large_f32_keys():
    """C3 shape: one SPT of 1M records with f32 keys, sweep of distances."""
    rng = np.random.default_rng(11)
    n = 1_000_000
    ks = (25.0 / rng.uniform(0.03, 0.3, n) + rng.uniform(0, 5, n)).astype(np.float32).astype(np.float64)
    kp = np.sort(ks)[::-1].copy()
    kp[0] = np.inf
    nodes = rng.permutation(n).astype(np.int64)
    spt = Spt(root=int(nodes[0]), root_center=np.zeros(3), nodes=nodes, key_self=ks, key_parent=kp)
    for q in np.linspace(0.05, 0.95, 7):
        dd = float(np.quantile(ks, q))
        pl, sel = cut_spt(spt, dd)
        pl2, sel2 = O.cut_spt(ks, kp, nodes, spt.root, dd)
        assert pl == pl2
        np.testing.assert_array_equal(sel, sel2)


@pytest.mark.parametrize("f64", [False, True], ids=["f32_keys", "f64_keys"])
def test_compact_span_boundaries(f64):
    """K1 over many SPTs at once, with prefix lengths on and around the
    span (512 / 256 records), sub-tile (2048 / 1024) and tile boundaries, a
    share of SPTs taking the root rule, and per-SPT distances: the selected
    node ids, their (segment, position) and the prefix lengths are
    bit-exact against the C oracle (spt.py:67-75) — the span fast path and
    the general path must agree wherever a warp's span starts."""
    import torch
    from paper_2507_01110_b200.device import DeviceLodScene
    from paper_2507_01110_b200.hierarchy import Hierarchy
    from paper_2507_01110_b200.hspt import Hspt
    rng = np.random.default_rng(5)
    lens = [1, 2, 3, 4, 5, 255, 256, 257, 511, 512, 513, 1023, 1024, 1025, 2047, 2048, 2049,
            4095, 4096, 4097, 16383, 16384, 16385, 70001] + [int(x) for x in rng.integers(1, 40_000, 40)]
    spts, base = [], 0
    for n in lens:
        ks = 25.0 / rng.uniform(0.03, 0.3, n) + rng.uniform(0, 5, n)
        if not f64:
            ks = ks.astype(np.float32).astype(np.float64)
        kp = np.sort(ks)[::-1].copy()
        kp[0] = np.inf
        nodes = (base + rng.permutation(n)).astype(np.int64)
        base += n
        ks[0] = ks.max()
        spts.append(Spt(root=int(nodes[0]), root_center=np.zeros(3), nodes=nodes, key_self=ks, key_parent=kp))
    stub = Hierarchy(attrs=None, parent=np.full(base, -1, np.int32), children=np.full((base, 2), -1, np.int32),
                     root=0)
    hs = Hspt(upper_nodes=np.zeros(0, np.int64), spts=spts, passthrough_roots=np.zeros(0, np.int64),
              size_threshold=1.0, min_subtree=1, lod=LodConfig(1.0))
    dev = DeviceLodScene(stub, hs)
    assert dev.key_f64 == f64
    S = len(spts)
    order = [spts[int(dev.spt_perm[j])] for j in range(S)]
    for trial in range(3):
        d = np.array([s.key_self.max() + 1.0 if rng.uniform() < 0.1 else
                      float(np.quantile(s.key_self, rng.uniform(0.02, 0.98))) for s in order])
        res = dev.compact(torch.tensor([S], dtype=torch.int32, device="cuda"),
                          torch.arange(S, dtype=torch.int32, device="cuda"),
                          torch.tensor(d, dtype=torch.float64, device="cuda"))
        total = int(res.total[0].item())
        want_pl, want_nodes, counts = [], [], []
        for s, dd in zip(order, d):
            pl, sel = O.cut_spt(s.key_self, s.key_parent, s.nodes, s.root, dd)
            want_pl.append(pl)
            want_nodes.append(np.asarray(sel, np.int64))
            counts.append(len(sel))
        want = np.concatenate(want_nodes)
        assert total == want.size, trial
        np.testing.assert_array_equal(res.prefix_len[:S].cpu().numpy(), np.asarray(want_pl))
        got_nodes = res.sel_node[:total].cpu().numpy().astype(np.int64)
        np.testing.assert_array_equal(got_nodes, want)
        seg = res.sel_seg[:total].cpu().numpy()
        np.testing.assert_array_equal(seg, np.repeat(np.arange(S), counts))
        pos = res.sel_pos[:total].cpu().numpy()
        flat_nodes = np.concatenate([s.nodes for s in order])
        offs = np.concatenate([[0], np.cumsum([len(s.nodes) for s in order])[:-1]])
        np.testing.assert_array_equal(flat_nodes[offs[seg] + pos], want)
