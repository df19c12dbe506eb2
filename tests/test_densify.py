"""Densification against the reference's own
trainer.densify outputs (tests/golden/densify_cases.npz, made by
tests/golden/make_golden.py): tree surgery, RNG consumption, moment
reset/growth, and the HSPT rebuilt with the surface-area metric.

CPU: the host tree surgery (densify.py) + the host HSPT restatement.
GPU: Trainer.densify on device-resident state (node records read back,
surgery, device HSPT build K12, store/record re-layout)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_01110_b200 import hspt as H
from paper_2507_01110_b200.core import SECTIONS, AttributeArrays, LodConfig
from paper_2507_01110_b200.densify import Moments, densify_tree

from .conftest import golden
from .helpers import hierarchy_of, hspt_of


def case(d, c):
    p = f"c{c}_"
    return {k[len(p):]: d[k] for k in d.files if k.startswith(p)}


def moments_of(cd, prefix=""):
    blk = lambda t: AttributeArrays(*[cd[f"{prefix}{t}_{n}"].copy() for n, _ in SECTIONS])
    return Moments(blk("m"), blk("v"), cd[prefix + "step"].copy())


def check_tree(h, cd, where):
    np.testing.assert_array_equal(h.parent, cd["out_parent"], err_msg=f"{where} parent")
    np.testing.assert_array_equal(h.children, cd["out_children"], err_msg=f"{where} children")
    assert h.root == int(cd["out_root"])
    assert list(h.free) == list(cd["out_free"])
    for n, _ in SECTIONS:
        np.testing.assert_array_equal(getattr(h.attrs, n), cd["out_" + n], err_msg=f"{where} {n}")


def check_moments(opt, cd, where):
    for n, _ in SECTIONS:
        np.testing.assert_array_equal(getattr(opt.m, n), cd["out_m_" + n], err_msg=f"{where} m {n}")
        np.testing.assert_array_equal(getattr(opt.v, n), cd["out_v_" + n], err_msg=f"{where} v {n}")
    np.testing.assert_array_equal(opt.step, cd["out_step"], err_msg=f"{where} step")


def check_hspt(hs, cd, where):
    np.testing.assert_array_equal(hs.upper_nodes, cd["out_upper_nodes"], err_msg=f"{where} upper")
    np.testing.assert_array_equal(hs.passthrough_roots, cd["out_pass_roots"], err_msg=f"{where} pass")
    cat = lambda k: np.concatenate([getattr(s, k) for s in hs.spts]) if hs.spts else np.zeros(0)
    np.testing.assert_array_equal(cat("nodes").astype(np.int64), cd["out_rec_node"], err_msg=f"{where} records")
    for k in ("key_self", "key_parent"):
        assert np.array_equal(cat(k).view(np.uint64), cd["out_" + k].view(np.uint64)), f"{where} {k}"
    assert hs.lod.metric == "surface_area"


def spawns(cd):
    s = int(cd["spawns"])
    return None if s < 0 else s


def test_host_densify_matches_reference():
    d = golden("densify_cases.npz")
    for c in range(int(d["n_cases"])):
        cd = case(d, c)
        h, hs0 = hierarchy_of(cd), hspt_of(cd)
        opt = moments_of(cd)
        rng = np.random.default_rng(int(cd["seed"]))
        out = densify_tree(h, opt, rng, 0.005, spawns(cd))
        assert out == {"spawned": int(cd["out_spawned"]), "respawned": int(cd["out_respawned"])}
        check_tree(h, cd, f"case {c}")
        check_moments(opt, cd, f"case {c}")
        assert rng.random() == float(cd["out_next_draw"])          # same RNG consumption
        hs = H.build_hspt_host(h, hs0.size_threshold, hs0.min_subtree,
                               LodConfig(hs0.lod.threshold, "surface_area"))
        check_hspt(hs, cd, f"case {c}")


@pytest.mark.gpu
def test_trainer_densify_matches_reference():
    import torch

    from paper_2507_01110_b200.cache import CacheConfig
    from paper_2507_01110_b200.core import Camera
    from paper_2507_01110_b200.trainer import NODE_RECORD, REC_MV, REC_STEP, TrainConfig, Trainer
    d = golden("densify_cases.npz")
    for c in range(int(d["n_cases"])):
        cd = case(d, c)
        h, hs0 = hierarchy_of(cd), hspt_of(cd)
        cams = [Camera(position=np.array([x, 0.0, -30.0]), orientation=np.array([1.0, 0, 0, 0]),
                       focal=(30.0, 30.0), principal_point=(16.0, 16.0), resolution=(32, 32))
                for x in (0.0, 2.0)]
        targets = [np.zeros((32, 32, 3))] * 2
        tr = Trainer(h, hs0, list(zip(cams, targets)), TrainConfig(lod=hs0.lod, scheduler_k=1,
                                                                   cache=CacheConfig(budget_bytes=1 << 20)),
                     extent=1.0)
        opt = moments_of(cd)
        recs = tr.scene.records
        for k, blk in enumerate((opt.m, opt.v)):
            cols = np.concatenate([np.asarray(a).reshape(h.capacity, -1) for _, a in blk.arrays()], axis=1)
            recs[:, REC_MV + k:REC_MV + 46:2] = torch.from_numpy(cols).cuda()
        recs.view(torch.int64)[:, REC_STEP] = torch.from_numpy(opt.step).cuda()
        tr.rng = np.random.default_rng(int(cd["seed"]))
        out = tr.densify(0.005, spawns(cd))
        assert out == {"spawned": int(cd["out_spawned"]), "respawned": int(cd["out_respawned"])}
        sc = tr.scene
        hh = tr.hierarchy
        hh.attrs = sc.attrs_host()
        check_tree(hh, cd, f"case {c}")
        m, v = sc.moments_packed()
        got = Moments(AttributeArrays.from_packed(m.cpu().numpy(), sc.cap),
                      AttributeArrays.from_packed(v.cpu().numpy(), sc.cap), sc.step.cpu().numpy())
        check_moments(got, cd, f"case {c}")
        check_hspt(sc.hspt, cd, f"case {c}")
        assert sc.records.shape == (len(cd["out_parent"]), NODE_RECORD)
        assert tr.rng.random() == float(cd["out_next_draw"])
        # the re-laid-out scene keeps training
        tr.train_step(1)


def test_choice1_matches_numpy_choice():
    """densify's single weighted draw equals rng.choice(a, 1, replace=False,
    p=p) — same element and the same generator state afterwards."""
    from paper_2507_01110_b200.densify import _choice1
    for trial in range(300):
        r = np.random.default_rng(trial)
        n = int(r.integers(1, 3000))
        a = np.sort(r.choice(10 ** 6, n, replace=False))
        w = np.maximum(r.random(n) ** 3, 1e-12)
        p = w / w.sum()
        r1, r2 = np.random.default_rng(trial + 7), np.random.default_rng(trial + 7)
        for _ in range(3):
            assert r1.choice(a, size=1, replace=False, p=p)[0] == _choice1(r2, a, p)
        assert r1.bit_generator.state == r2.bit_generator.state
