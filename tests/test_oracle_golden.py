"""Pin the oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import glod_oracle as O

from .conftest import golden, lod_files
from .helpers import assert_rs_equal, camera_of, golden_rs, oracle_cut_hspt


@pytest.mark.parametrize("path", lod_files(), ids=lambda p: p.stem)
def test_oracle_cut_hspt_matches_reference(path):
    d = np.load(path)
    for v in range(int(d["n_views"])):
        got = oracle_cut_hspt(d, v)
        assert_rs_equal(got, golden_rs(d, v), where=f"{path.stem} view {v}")


@pytest.mark.parametrize("path", lod_files(), ids=lambda p: p.stem)
def test_oracle_bfs_cut_matches_reference(path):
    d = np.load(path)
    for v in range(int(d["n_views"])):
        planes = d[f"v{v}_planes"] if d[f"v{v}_cull"] else None
        got = O.bfs_cut(d["children"], d["means"], d["scales"], d[f"v{v}_position"],
                        float(d[f"v{v}_T"]), int(d[f"v{v}_metric"]), planes, root=int(d["root"]))
        np.testing.assert_array_equal(got, d[f"v{v}_bfs"])


def test_oracle_frustum_planes_bitexact():
    for path in lod_files()[:6]:
        d = np.load(path)
        for v in range(int(d["n_views"])):
            p = f"v{v}_"
            pl = O.frustum_planes(d[p + "orientation"], d[p + "position"], tuple(d[p + "focal"]),
                                  tuple(d[p + "pp"]), tuple(d[p + "res"]), float(d[p + "far"]))
            assert np.array_equal(pl.view(np.uint64), d[p + "planes"].view(np.uint64))


def test_oracle_cut_spt_matches_reference():
    d = golden("spt_cases.npz")
    for k in range(int(d["n_cases"])):
        p = f"c{k}_"
        pl, sel = O.cut_spt(d[p + "key_self"], d[p + "key_parent"], d[p + "nodes"],
                            int(d[p + "root"]), float(d[p + "d"]))
        assert pl == int(d[p + "prefix"]), k
        np.testing.assert_array_equal(sel, d[p + "sel"])


def _attrs(d, p):
    return {k: d[p + k] for k in ("means", "scales", "rotations", "opacities", "base_colors",
                                  "sh_rest")}


def test_oracle_render_forward_backward_loss():
    d = golden("render_cases.npz")
    for k in range(int(d["n_cases"])):
        cam = O.Cam.of(camera_of(d, f"r{k}_"))
        A = _attrs(d, f"r{k}_a_")
        img, ctx = O.render_forward(A, cam)
        assert np.array_equal(img, d[f"r{k}_image"]), k
        G = O.backward(ctx, d[f"r{k}_upstream"])
        for name in A:
            np.testing.assert_allclose(G[name], d[f"r{k}_g_{name}"], rtol=1e-12, atol=1e-13)
        lv, lg = O.ssim_l1_loss(img, d[f"r{k}_target"], 0.2)
        assert abs(lv - float(d[f"r{k}_loss"])) <= 1e-14
        np.testing.assert_allclose(lg, d[f"r{k}_loss_grad"], rtol=1e-10, atol=1e-16)


def test_oracle_adam():
    d = golden("adam_cases.npz")
    names = ("means", "scales", "rotations", "opacities", "base_colors", "sh_rest")
    P = {k: d["p0_" + k].copy() for k in names}
    M = {k: np.zeros_like(P[k]) for k in names}
    V = {k: np.zeros_like(P[k]) for k in names}
    step = np.zeros(P["means"].shape[0], dtype=np.int64)
    lrs = {k: float(d["lr_" + k]) for k in names}
    for it in range(3):
        G = {k: d[f"it{it}_g_{k}"] for k in names}
        ids = d[f"it{it}_ids"]
        O.adam_update(P, M, V, step, ids, G, np.arange(ids.size), lrs)
        for k in names:
            assert np.array_equal(P[k], d[f"it{it}_p_{k}"]), (it, k)
            assert np.array_equal(M[k], d[f"it{it}_m_{k}"]), (it, k)
            assert np.array_equal(V[k], d[f"it{it}_v_{k}"]), (it, k)
        np.testing.assert_array_equal(step, d[f"it{it}_step"])
