"""Scene files: `.glod` write/read bit-exact against the
reference's own write_scene / open_scene (tests/golden/scenefile_cases.npz,
made by tests/golden/make_golden.py), and a trainer whose pinned store is
read straight from the file."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_01110_b200 import scenefile as SF

from .conftest import golden
from .helpers import hierarchy_of, hspt_of


def case(d, c):
    p = f"c{c}_"
    return {k[len(p):]: d[k] for k in d.files if k.startswith(p)}


def sub(cd, prefix):
    return {k[len(prefix):]: v for k, v in cd.items() if k.startswith(prefix)}


def test_write_scene_is_byte_identical(tmp_path):
    d = golden("scenefile_cases.npz")
    for c in range(int(d["n_cases"])):
        cd = case(d, c)
        path = tmp_path / f"s{c}.glod"
        SF.write_scene(hierarchy_of(cd), hspt_of(cd), path)
        assert path.read_bytes() == cd["file"].tobytes(), f"case {c}"


def test_open_scene_reads_like_reference(tmp_path):
    d = golden("scenefile_cases.npz")
    for c in range(int(d["n_cases"])):
        cd = case(d, c)
        path = tmp_path / f"s{c}.glod"
        path.write_bytes(cd["file"].tobytes())
        sc = SF.open_scene(path)
        h, hs = sc.read_hierarchy(), sc.read_hspt()
        rd = sub(cd, "rd_")
        for k in ("children", "parent", "means", "scales", "rotations", "opacities", "base_colors", "sh_rest"):
            got = {"children": h.children, "parent": h.parent}.get(k, getattr(h.attrs, k, None))
            np.testing.assert_array_equal(got, rd[k], err_msg=f"case {c} {k}")
        assert h.root == int(rd["root"])
        np.testing.assert_array_equal(hs.upper_nodes, rd["upper_nodes"])
        np.testing.assert_array_equal(hs.passthrough_roots, rd["pass_roots"])
        cat = lambda k: np.concatenate([getattr(s, k) for s in hs.spts])
        np.testing.assert_array_equal(cat("nodes"), rd["rec_node"])
        assert np.array_equal(cat("key_self").view(np.uint64), rd["key_self"].view(np.uint64))
        assert np.array_equal(cat("key_parent").view(np.uint64), rd["key_parent"].view(np.uint64))
        assert np.array_equal(np.stack([s.root_center for s in hs.spts]), rd["spt_center"])
        assert hs.size_threshold == float(rd["size_threshold"]) and hs.min_subtree == int(rd["min_subtree"])
        sid = int(cd["pf_spt"])
        blk = sc.load_spt_prefix(sid, int(cd["pf_len"]))
        np.testing.assert_array_equal(blk.attrs.means, cd["pf_means"])
        np.testing.assert_array_equal(blk.attrs.sh_rest, cd["pf_sh"])
        assert sc.spt_slot_start(sid) == int(cd["pf_slot"])
        assert sc.attribute_bytes_read == int(cd["bytes_read"])
        sc.close()


def test_corrupt_files_raise(tmp_path):
    d = golden("scenefile_cases.npz")
    raw = bytearray(case(d, 0)["file"].tobytes())
    bad = tmp_path / "bad.glod"
    bad.write_bytes(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(SF.CorruptFileError):
        SF.open_scene(bad)
    raw[4] = 9
    bad.write_bytes(bytes(raw))
    with pytest.raises(SF.CorruptFileError):
        SF.open_scene(bad)


def test_write_back_roundtrip(tmp_path):
    d = golden("scenefile_cases.npz")
    cd = case(d, 1)
    path = tmp_path / "w.glod"
    path.write_bytes(cd["file"].tobytes())
    sc = SF.open_scene(path)
    blk = sc.load_spt_prefix(0, 3)
    blk.attrs.means = blk.attrs.means + 1.0
    sc.write_back(blk)
    again = sc.load_spt_prefix(0, 3)
    np.testing.assert_array_equal(again.attrs.means, (blk.attrs.means).astype(np.float32))
    with pytest.raises(SF.InvalidBlockError):
        sc.load_spt_prefix(0, 10 ** 7)
    with pytest.raises(SF.NotFoundError):
        sc.load_spt_prefix(10 ** 6, 1)


@pytest.mark.gpu
def test_trainer_on_file_store_matches_in_memory_store(tmp_path):
    """A .glod scene trained from a pinned store read straight from the
    file gives the same steps as the store built from its hierarchy."""
    import torch

    from paper_2507_01110_b200.cache import CacheConfig
    from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene, orbit_views, scene_extent
    from paper_2507_01110_b200.trainer import TrainConfig, Trainer
    h0, hs0, cfg = designed_scene(SceneSpec(n_leaves=6000, spt_leaves=256, seed=8))
    path = tmp_path / "scene.glod"
    SF.write_scene(h0, hs0, path)
    sc = SF.open_scene(path)
    h, hs = sc.read_hierarchy(), sc.read_hspt()
    E = scene_extent(6000)
    cams = orbit_views(6, 1.5 * E, 0.6 * E, resolution=(96, 64), focal=(70.0, 70.0), seed=1)
    rng = np.random.default_rng(0)
    targets = [np.clip(rng.normal(0.5, 0.2, (64, 96, 3)), 0, 1) for _ in cams]
    budget = int(0.35 * hs.flat_records()["nodes"].size * 92)
    mk = lambda: TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=budget, flush_interval=5), scheduler_k=3)
    a = Trainer(h, hs, list(zip(cams, targets)), mk(), extent=2 * E)
    b = Trainer(h, hs, list(zip(cams, targets)), mk(), extent=2 * E, store=sc.host_store())
    for sa, sb in zip(a.scene.store.sections, b.scene.store.sections):
        assert torch.equal(sa, sb)
    assert b.scene.lod.key_f64 is False          # file keys are f32: the f32-key cut path
    for it in range(1, 11):
        assert a.train_step(it) == b.train_step(it), it
    torch.cuda.synchronize()
    from .test_train_gpu import same_state
    assert same_state(a.scene.records, b.scene.records)
    sc.save_store(b.scene.store)
    sc2 = SF.open_scene(path)
    st2 = sc2.host_store()
    for sa, sb in zip(st2.sections, b.scene.store.sections):
        assert torch.equal(sa, sb)
