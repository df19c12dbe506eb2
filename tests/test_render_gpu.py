"""GPU rasteriser / loss / ADAM parity through the C-ABI.

Tolerances (BASELINE north star): images ≤ 1e-4 max-abs per channel;
gradients ≤ 1e-3 relative, evaluated per attribute array as
|g − g_ref| ≤ 1e-3 · (|g_ref| + 1e-2 · max|g_ref|)  (the second term keeps
entries that are ~0 from demanding infinite relative precision).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import glod_oracle as O  # noqa: E402
from paper_2507_01110_b200 import renderer as Rn  # noqa: E402
from paper_2507_01110_b200.core import AttributeArrays, SECTIONS  # noqa: E402

from .conftest import golden  # noqa: E402
from .helpers import camera_of  # noqa: E402

NAMES = [n for n, _ in SECTIONS]
IMG_TOL = 1e-4
GRAD_REL = 1e-3


def attrs_of(d, p):
    return AttributeArrays(*(d[p + k] for k in NAMES))


def assert_grads_close(got, want, where=""):
    for k in NAMES:
        g = np.asarray(getattr(got, k) if not isinstance(got, dict) else got[k], dtype=np.float64)
        w = np.asarray(want[k], dtype=np.float64)
        scale = np.max(np.abs(w)) if w.size else 0.0
        tol = GRAD_REL * (np.abs(w) + 1e-2 * scale) + 1e-300
        bad = np.abs(g - w) > tol
        assert not bad.any(), (f"{where} {k}: max rel err "
                               f"{np.max(np.abs(g - w) / (np.abs(w) + 1e-2 * scale + 1e-300)):.3e}")


def test_render_golden_forward_backward_loss():
    d = golden("render_cases.npz")
    for k in range(int(d["n_cases"])):
        cam = camera_of(d, f"r{k}_")
        a = attrs_of(d, f"r{k}_a_")
        ctx = Rn.render_forward(a, cam)
        err = np.max(np.abs(ctx.image - d[f"r{k}_image"]))
        assert err <= IMG_TOL, (k, err)
        g = Rn.backward(ctx, d[f"r{k}_upstream"])
        want = {n: d[f"r{k}_g_{n}"] for n in NAMES}
        assert_grads_close(g, want, where=f"case {k}")
        lv, lg = Rn.loss(d[f"r{k}_image"], d[f"r{k}_target"], 0.2)
        assert abs(lv - float(d[f"r{k}_loss"])) <= 1e-6 * max(1.0, abs(float(d[f"r{k}_loss"])))
        ref = d[f"r{k}_loss_grad"]
        assert np.max(np.abs(lg - ref)) <= 1e-4 * np.max(np.abs(ref))


def test_render_empty_and_offscreen():
    d = golden("render_cases.npz")
    cam = camera_of(d, "r0_")
    img = Rn.render(AttributeArrays.zeros(0), cam)
    assert img.shape == (cam.resolution[1], cam.resolution[0], 3) and np.all(img == 0)
    a = AttributeArrays.zeros(1)
    a.means[0] = [0, 0, -50]        # behind the camera
    a.opacities[:] = 1.0
    a.base_colors[0] = [1, 1, 1]
    assert np.all(Rn.render(a, cam) == 0)


def test_render_rejects_non_finite():
    d = golden("render_cases.npz")
    cam = camera_of(d, "r0_")
    a = AttributeArrays.zeros(3)
    a.means[1, 2] = np.nan
    with pytest.raises(Rn.InvalidInputError, match="Gaussian 1"):
        Rn.render(a, cam)


def test_single_opaque_center_kat():
    """Known answer (test_renderer.py:105-114): centre pixel = 0.99·colour."""
    d = golden("render_cases.npz")
    cam = camera_of(d, "r0_")
    a = AttributeArrays.zeros(1)
    a.opacities[:] = 1.0
    a.base_colors[0] = [0.2, 0.5, 0.9]
    img = Rn.render(a, cam)
    np.testing.assert_allclose(img[8, 8], 0.99 * a.base_colors[0], rtol=1e-6)


@pytest.mark.parametrize("n_leaves,res", [(20_000, (256, 256)), (60_000, (640, 360))])
def test_render_designed_scene_vs_oracle(n_leaves, res):
    """Render sets from the LoD cut of a generated scene (thousands of
    Gaussians, saturated pixels) against the numpy oracle."""
    from paper_2507_01110_b200 import hspt as H
    from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene, orbit_views, scene_extent
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=n_leaves, spt_leaves=1024, seed=2))
    E = scene_extent(n_leaves)
    cam = orbit_views(1, 1.4 * E, 0.6 * E, resolution=res, seed=4)[0]
    rs = H.cut_hspt(hs, h, cam, cfg)
    a = h.attrs.take(rs.nodes)
    ctx = Rn.render_forward(a, cam)
    A = {k: getattr(a, k) for k in NAMES}
    img, octx = O.render_forward(A, O.Cam.of(cam))
    assert np.max(np.abs(ctx.image - img)) <= IMG_TOL
    up = np.random.default_rng(0).normal(size=img.shape)
    assert_grads_close(Rn.backward(ctx, up), O.backward(octx, up), where="designed")


def test_adam_golden():
    from paper_2507_01110_b200 import _lib
    import ctypes as C
    d = golden("adam_cases.npz")
    n = d["p0_means"].shape[0]
    a = attrs_of(d, "p0_")
    P = torch.from_numpy(a.packed()).cuda()
    MV = torch.zeros(2 * P.numel(), dtype=torch.float64, device="cuda")   # [n][23][m, v]
    step = torch.zeros(n, dtype=torch.int64, device="cuda")
    lrs = (C.c_double * 6)(*[float(d["lr_" + k]) for k in NAMES])
    for it in range(3):
        ids = torch.from_numpy(d[f"it{it}_ids"].astype(np.int32)).cuda()
        g = AttributeArrays(*(d[f"it{it}_g_{k}"] for k in NAMES))
        G = torch.from_numpy(g.packed()).cuda()
        _lib.check(_lib.lib().glod_adam_step(_lib.ptr(P), _lib.ptr(MV), _lib.ptr(step), n,
                                             _lib.ptr(ids), _lib.ptr(G), None, ids.numel(), ids.numel(),
                                             lrs, None, 0, None, _lib.stream_ptr()))
        got = AttributeArrays.from_packed(P.cpu().numpy(), n)
        for k in NAMES:
            np.testing.assert_allclose(getattr(got, k), d[f"it{it}_p_{k}"], rtol=1e-12, atol=1e-14)
        np.testing.assert_array_equal(step.cpu().numpy(), d[f"it{it}_step"])
        mv = MV.view(n, 23, 2).cpu().numpy()
        off = 0
        for k, (_, cols) in zip(NAMES, SECTIONS):
            for j, tag in enumerate("mv"):
                want = d[f"it{it}_{tag}_{k}"].reshape(n, cols)
                np.testing.assert_allclose(mv[:, off:off + cols, j], want, rtol=1e-12, atol=1e-300)
            off += cols


def test_depth_order_exact_with_near_ties():
    """The depth sort radix-sorts only the top 32 bits of the key range and
    fixes up runs that tie there: opaque splats at depths 1e-12 apart (a
    tie in the top bits), exactly equal depths (index order decides) and a
    far splat widening the range must composite exactly as the reference's
    lexsort((idx, depth)) order — image equal to the oracle's."""
    from oracle.glod_oracle import Cam
    from paper_2507_01110_b200.core import Camera
    cam = Camera(position=np.zeros(3), orientation=np.array([1.0, 0.0, 0.0, 0.0]), focal=(40.0, 40.0),
                 principal_point=(16.0, 16.0), resolution=(32, 32))
    rng = np.random.default_rng(3)
    depths = [10.0, 10.0 + 1e-12, 10.0 + 2e-12, 10.0, 10.0 - 1e-13, 25.0, 25.0, 1000.0]
    n = len(depths) * 4
    a = AttributeArrays.zeros(n)
    for k in range(n):
        z = depths[k % len(depths)] + (k // len(depths)) * 3e-13
        a.means[k] = [rng.uniform(-0.2, 0.2) * z / 10, rng.uniform(-0.2, 0.2) * z / 10, z]
    a.scales[:] = 0.3
    a.scales[:, 2] = 0.05
    a.rotations[:, 0] = 1.0
    a.opacities[:] = 0.97
    a.base_colors[:] = rng.uniform(0, 1, (n, 3))
    img = Rn.render(a, cam)
    want, _ = O.render_forward({k: getattr(a, k) for k in NAMES}, Cam.of(cam))
    assert np.abs(img - want).max() <= IMG_TOL


def _facade(n, rng, jitter_rel, far=16):
    """n splats on a fronto-parallel plane at depth ≈ 10 (depths within
    `jitter_rel` relative, some exactly equal) plus `far` splats at depth
    1000 that widen the key range: with the top-32-bit radix passes the
    whole facade is ONE tie run (renderer.py:127's lexsort order must
    still come out exactly)."""
    a = AttributeArrays.zeros(n + far)
    z = 10.0 * (1.0 + jitter_rel * rng.uniform(-1, 1, n))
    z[::5] = 10.0                              # exact ties: index order decides
    a.means[:n] = np.stack([rng.uniform(-4, 4, n), rng.uniform(-4, 4, n), z], 1)
    a.means[n:] = np.stack([rng.uniform(-300, 300, far), rng.uniform(-300, 300, far), np.full(far, 1000.0)], 1)
    a.scales[:] = rng.uniform(0.02, 0.08, (n + far, 3))
    a.rotations[:, 0] = 1.0
    a.opacities[:] = rng.uniform(0.3, 0.9, n + far)
    a.base_colors[:] = rng.uniform(0, 1, (n + far, 3))
    return a


def test_facade_depth_order_exact():
    """fixup_runs_kernel's worst case: a 20k-splat facade whose depths tie in
    the top 32 bits of the key range — the long run is detected and the
    order finished by full-width radix passes; the image equals the oracle's."""
    from paper_2507_01110_b200.core import Camera
    rng = np.random.default_rng(8)
    a = _facade(20_000, rng, 1e-9)
    cam = Camera(position=np.zeros(3), orientation=np.array([1.0, 0.0, 0.0, 0.0]), focal=(100.0, 100.0),
                 principal_point=(64.0, 64.0), resolution=(128, 128))
    ctx = Rn.render_forward(a, cam)
    assert Rn._rasterizer().stats()["depth_full_sort"]
    want, _ = O.render_forward({k: getattr(a, k) for k in NAMES}, O.Cam.of(cam))
    assert np.abs(ctx.image - want).max() <= IMG_TOL


def test_facade_render_time_bounded():
    """1M facade splats, depths within 1e-9 relative, must render within 2x
    the time of the same splats at random depths (no O(run²) fix-up)."""
    import time as _t
    from paper_2507_01110_b200.core import Camera
    rng = np.random.default_rng(9)
    cam = Camera(position=np.zeros(3), orientation=np.array([1.0, 0.0, 0.0, 0.0]), focal=(1400.0, 1400.0),
                 principal_point=(960.0, 540.0), resolution=(1920, 1080))
    fac = _facade(1_000_000, rng, 1e-9)
    rnd = AttributeArrays(*(np.array(getattr(fac, k), copy=True) for k in NAMES))
    rnd.means[:1_000_000, 2] = rng.uniform(5.0, 15.0, 1_000_000)
    rast = Rn.Rasterizer()
    times = {}
    for name, a in (("random", rnd), ("facade", fac)):
        t = torch.from_numpy(a.packed()).cuda()
        ts = []
        for r in range(4):
            torch.cuda.synchronize()
            t0 = _t.perf_counter()
            rast.forward(t, len(a), cam)
            torch.cuda.synchronize()
            ts.append(_t.perf_counter() - t0)
        times[name] = min(ts[1:])
        if name == "facade":
            assert rast.stats()["depth_full_sort"]
    assert times["facade"] <= 2.0 * times["random"], times
