"""HSPT / SPT build: the device build K12 (through the
C-ABI) and the host restatement, bit-exact against the reference's own
build_hspt outputs stored in the golden LoD cases (tests/golden/
make_golden.py: 24 merged / rescaled / designed hierarchies, both metrics,
min_subtree 1-32)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_01110_b200 import hspt as H
from paper_2507_01110_b200.core import LodConfig

from .conftest import lod_files
from .helpers import hierarchy_of


def build_args(d):
    cfg = LodConfig(float(d["lod_threshold"]), ("max_scale", "surface_area")[int(d["lod_metric"])])
    return float(d["size_threshold"]), int(d["min_subtree"]), cfg


def assert_hspt_equal(got, d, where=""):
    np.testing.assert_array_equal(got.upper_nodes, d["upper_nodes"], err_msg=f"{where} upper")
    np.testing.assert_array_equal(got.passthrough_roots, d["pass_roots"], err_msg=f"{where} pass")
    roots = np.array([s.root for s in got.spts], dtype=np.int64)
    np.testing.assert_array_equal(roots, d["spt_root"], err_msg=f"{where} spt roots")
    cnt = np.array([s.subtree_size for s in got.spts], dtype=np.int64)
    np.testing.assert_array_equal(cnt, d["spt_count"], err_msg=f"{where} counts")
    cat = (lambda k: np.concatenate([getattr(s, k) for s in got.spts]) if got.spts else np.zeros(0))
    np.testing.assert_array_equal(cat("nodes").astype(np.int64), d["rec_node"], err_msg=f"{where} records")
    for k in ("key_self", "key_parent"):
        assert np.array_equal(cat(k).view(np.uint64), np.asarray(d[k]).view(np.uint64)), f"{where} {k} bits"
    if got.spts:
        centers = np.stack([s.root_center for s in got.spts])
        assert np.array_equal(centers, d["spt_center"]), f"{where} centres"
    assert got.spt_id_of == {int(r): i for i, r in enumerate(d["spt_root"])}


@pytest.mark.parametrize("path", lod_files(), ids=lambda p: p.stem)
def test_host_build_matches_reference(path):
    d = np.load(path)
    thr, ms, cfg = build_args(d)
    assert_hspt_equal(H.build_hspt_host(hierarchy_of(d), thr, ms, cfg), d, path.stem)


@pytest.mark.gpu
@pytest.mark.parametrize("path", lod_files(), ids=lambda p: p.stem)
def test_device_build_bitexact_vs_reference(path):
    d = np.load(path)
    thr, ms, cfg = build_args(d)
    assert_hspt_equal(H.build_hspt(hierarchy_of(d), thr, ms, cfg), d, path.stem)


@pytest.mark.gpu
def test_device_build_validates_like_reference():
    d = np.load(lod_files()[0])
    h = hierarchy_of(d)
    _, _, cfg = build_args(d)
    with pytest.raises(ValueError):
        H.build_hspt(h, 0.0, 8, cfg)
    with pytest.raises(ValueError):
        H.build_hspt(h, 1.0, 0, cfg)


@pytest.mark.gpu
def test_device_build_skips_free_slots():
    """A detached slot (Hierarchy.free, as left by densification) belongs
    to no list — the reference's BFS never reaches it."""
    d = np.load(lod_files()[3])
    h = hierarchy_of(d)
    thr, ms, cfg = build_args(d)
    want = H.build_hspt_host(h, thr, ms, cfg)
    cap = h.capacity
    # append two detached slots whose parent pointers are stale
    from paper_2507_01110_b200.core import AttributeArrays
    from paper_2507_01110_b200.hierarchy import Hierarchy
    A = h.attrs
    grow = lambda a: np.concatenate([a, a[:2]])
    h2 = Hierarchy(attrs=AttributeArrays(grow(A.means), np.concatenate([A.scales, A.scales[:2] * 1e-6]), grow(A.rotations),
                                         grow(A.opacities), grow(A.base_colors), grow(A.sh_rest)),
                   parent=np.concatenate([h.parent, [h.root, cap]]).astype(np.int32),
                   children=np.concatenate([h.children, [[-1, -1], [-1, -1]]]).astype(np.int32),
                   root=h.root)
    got = H.build_hspt(h2, thr, ms, cfg)
    np.testing.assert_array_equal(got.upper_nodes, want.upper_nodes)
    np.testing.assert_array_equal(got.passthrough_roots, want.passthrough_roots)
    assert len(got.spts) == len(want.spts)
    for a, b in zip(got.spts, want.spts):
        np.testing.assert_array_equal(a.nodes, b.nodes)
        assert np.array_equal(a.key_parent.view(np.uint64), b.key_parent.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("metric", ["max_scale", "surface_area"])
def test_device_build_large_vs_host(metric):
    """300k-leaf designed scene (600k nodes, ~150 SPTs, passthrough
    branches): device build == host restatement, record for record."""
    from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=300_000, spt_leaves=2048, seed=9, metric=metric))
    want = H.build_hspt_host(h, hs.size_threshold, hs.min_subtree, cfg)
    got = H.build_hspt(h, hs.size_threshold, hs.min_subtree, cfg)
    np.testing.assert_array_equal(got.upper_nodes, want.upper_nodes)
    np.testing.assert_array_equal(got.passthrough_roots, want.passthrough_roots)
    assert len(got.spts) == len(want.spts) > 50
    for k in ("nodes", "key_self", "key_parent", "offset", "count", "roots"):
        a, b = np.asarray(got.flat[k]), np.asarray(want.flat[k])
        assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.astype(a.dtype).view(np.uint8)), k
