"""Generate golden vectors by running the REFERENCE itself.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
Outputs tests/golden/*.npz (committed).  Nothing at test time reads
/root/reference: the fixtures carry the reference's inputs and outputs.

Cases mirror the reference's own seeded fixtures (pkg/tests/conftest.py:
random_hierarchy / random_scale_hierarchy / random_camera / look_at_camera)
and known-answer tests (test_spt.py:132-149, test_renderer.py:105-114).
"""
from __future__ import annotations

import importlib.util
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _import_ref():
    sys.dont_write_bytecode = True
    spec = importlib.util.spec_from_file_location(
        "glod", REF / "glod" / "__init__.py", submodule_search_locations=[str(REF / "glod")])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["glod"] = mod
    spec.loader.exec_module(mod)
    import glod.core, glod.hierarchy, glod.spt, glod.hspt, glod.renderer, glod.trainer  # noqa
    import glod.cache, glod.store  # noqa
    return sys.modules["glod"]


glod = _import_ref()
from glod.core import AttributeArrays, Camera, Frustum, LodConfig, rotmat_to_quat  # noqa: E402
from glod.hierarchy import bfs_cut, build_hierarchy  # noqa: E402
from glod.hspt import build_hspt, cut_hspt, default_size_threshold  # noqa: E402
from glod.renderer import backward, loss, render_forward  # noqa: E402
from glod.spt import build_spt, cut_spt  # noqa: E402


# ---- the reference's own conftest builders (pkg/tests/conftest.py:11-58) ----
def random_leaves(rng, n, span=10.0, scale_lo=0.05, scale_hi=0.5):
    leaves = AttributeArrays.zeros(n)
    leaves.means = rng.uniform(-span, span, (n, 3))
    leaves.scales = rng.uniform(scale_lo, scale_hi, (n, 3))
    q = rng.normal(size=(n, 4))
    leaves.rotations = q / np.linalg.norm(q, axis=1, keepdims=True)
    leaves.opacities = rng.uniform(0.05, 1.0, n)
    leaves.base_colors = rng.uniform(0.0, 1.0, (n, 3))
    return leaves


def look_at_camera(position, target, focal=(40.0, 40.0), resolution=(32, 32), near=0.1):
    position = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - position
    fwd = fwd / np.linalg.norm(fwd)
    up = np.array([0.0, 1.0, 0.0])
    if abs(fwd @ up) > 0.99:
        up = np.array([1.0, 0.0, 0.0])
    right = np.cross(up, fwd)
    right = right / np.linalg.norm(right)
    upv = np.cross(fwd, right)
    rot = np.stack([right, upv, fwd], axis=1)
    w, h = resolution
    return Camera(position=position, orientation=rotmat_to_quat(rot), focal=focal,
                  principal_point=(w / 2.0, h / 2.0), resolution=resolution, near=near)


def random_camera(rng, span=10.0, resolution=(32, 32)):
    pos = rng.uniform(-3 * span, 3 * span, 3)
    target = rng.uniform(-span, span, 3)
    while np.linalg.norm(target - pos) < 1e-3:
        target = rng.uniform(-span, span, 3)
    focal = tuple(rng.uniform(20.0, 80.0, 2))
    return look_at_camera(pos, target, focal=focal, resolution=resolution)


def cam_arrays(cam, prefix="cam_"):
    return {prefix + "position": cam.position, prefix + "orientation": cam.orientation,
            prefix + "focal": np.array(cam.focal, dtype=np.float64),
            prefix + "pp": np.array(cam.principal_point, dtype=np.float64),
            prefix + "res": np.array(cam.resolution, dtype=np.int64),
            prefix + "near": np.float64(cam.near), prefix + "far": np.float64(cam.far),
            prefix + "planes": Frustum.from_camera(cam).planes}


def hier_arrays(h):
    return {"children": h.children.astype(np.int32), "parent": h.parent.astype(np.int32),
            "root": np.int64(h.root), "means": h.attrs.means, "scales": h.attrs.scales,
            "rotations": h.attrs.rotations, "opacities": h.attrs.opacities,
            "base_colors": h.attrs.base_colors, "sh_rest": h.attrs.sh_rest}


def hspt_arrays(hspt):
    spts = hspt.spts
    cnt = np.array([s.subtree_size for s in spts], dtype=np.int64)
    return {"upper_nodes": hspt.upper_nodes.astype(np.int64),
            "pass_roots": hspt.passthrough_roots.astype(np.int64),
            "spt_root": np.array([s.root for s in spts], dtype=np.int64),
            "spt_center": (np.stack([s.root_center for s in spts]) if spts else np.zeros((0, 3))),
            "spt_count": cnt,
            "rec_node": (np.concatenate([s.nodes for s in spts]) if spts else np.zeros(0, np.int64)),
            "key_self": (np.concatenate([s.key_self for s in spts]) if spts else np.zeros(0)),
            "key_parent": (np.concatenate([s.key_parent for s in spts]) if spts else np.zeros(0)),
            "lod_threshold": np.float64(hspt.lod.threshold),
            "lod_metric": np.int64(0 if hspt.lod.metric == "max_scale" else 1),
            "size_threshold": np.float64(hspt.size_threshold),
            "min_subtree": np.int64(hspt.min_subtree)}


def rs_arrays(rs, prefix="rs_"):
    sel = [s.selected for s in rs.per_spt]
    return {prefix + "upper": rs.upper.astype(np.int64),
            prefix + "pass": rs.passthrough.astype(np.int64),
            prefix + "spt_id": np.array([s.spt_id for s in rs.per_spt], dtype=np.int64),
            prefix + "d_root": np.array([s.d_root for s in rs.per_spt], dtype=np.float64),
            prefix + "prefix_len": np.array([s.prefix_len for s in rs.per_spt], dtype=np.int64),
            prefix + "sel_count": np.array([x.size for x in sel], dtype=np.int64),
            prefix + "sel": (np.concatenate(sel).astype(np.int64) if sel else np.zeros(0, np.int64))}


def _designed_scales(rng, h, depth_cut):
    """Upper nodes small (never taken, md > dist), SPT/pass interiors i.i.d.
    — the bench generator's shape at golden size."""
    depth = np.full(h.capacity, -1)
    lv, fr = 0, np.array([h.root])
    while fr.size:
        depth[fr] = lv
        ch = h.children[fr]
        fr = ch[ch[:, 0] != -1].ravel()
        lv += 1
    s = rng.uniform(0.05, 0.6, h.attrs.scales.shape)
    s[depth < depth_cut] = 0.004
    s[depth == depth_cut] = 0.003
    h.attrs.scales = s
    return 0.004 ** 3 * 0.9


def make_lod_cases():
    """HSPT cuts on merged, re-scaled and "designed" hierarchies, both
    metrics, cull on/off, runtime thresholds from coarse (root-only) to
    1e9 (descend to leaves) — the reference's own fixture families
    (test_hspt.py, test_acceptance.py:98-127, big_scene T=1e9 :282-306)."""
    rng = np.random.default_rng(20250701)
    n_files = 0
    for case in range(24):
        n = int(rng.choice([40, 90, 200, 700, 1500, 3000]))
        family = case % 3            # 0 merged, 1 rescaled i.i.d., 2 designed
        h = build_hierarchy(random_leaves(rng, n))
        metric = ("max_scale", "surface_area")[case % 2]
        build_cfg = LodConfig(threshold=float(rng.uniform(0.5, 20.0)), metric=metric)
        if family == 1:   # random_scale_hierarchy (conftest.py:26-31)
            h.attrs.scales = rng.uniform(0.05, 2.0, h.attrs.scales.shape)
            vols = np.prod(h.attrs.scales, axis=1)
            thr = float(np.quantile(vols, rng.uniform(0.2, 0.8)))
        elif family == 2:
            thr = _designed_scales(rng, h, int(rng.integers(2, 6)))
        else:
            thr = float(rng.uniform(0.5, 4.0)) * default_size_threshold(h)
        min_sub = int(rng.choice([1, 4, 8, 16, 32]))
        if family == 2:
            min_sub = int(rng.choice([8, 16, 24]))
        hspt = build_hspt(h, thr, min_sub, build_cfg)
        d = {"n_leaves": np.int64(n), "family": np.int64(family)}
        d.update(hier_arrays(h))
        d.update(hspt_arrays(hspt))
        views = []
        for v in range(8):
            cam = random_camera(rng)
            if v >= 6:   # look at the scene centre from close by
                cam = look_at_camera(rng.uniform(-14, 14, 3), np.zeros(3), focal=(30.0, 30.0))
            if v in (0, 1):
                T = float(np.exp(rng.uniform(np.log(0.5), np.log(200.0))))
            elif v in (2, 3):
                T = float(10.0 ** rng.uniform(2.5, 9.0))
            else:
                T = float(rng.uniform(1.0, 60.0)) if family != 2 else float(rng.uniform(0.5, 8.0))
            cfg = LodConfig(threshold=T, metric=("max_scale", "surface_area")[int(rng.integers(2))])
            cull = bool(v % 2 == 0)
            rs = cut_hspt(hspt, h, cam, cfg, cull=cull)
            fr = Frustum.from_camera(cam)
            full = bfs_cut(h, cam, cfg, frustum=fr if cull else None)
            views.append((cam, cfg, cull, rs, full))
        for i, (cam, cfg, cull, rs, full) in enumerate(views):
            d.update(cam_arrays(cam, f"v{i}_"))
            d[f"v{i}_T"] = np.float64(cfg.threshold)
            d[f"v{i}_metric"] = np.int64(0 if cfg.metric == "max_scale" else 1)
            d[f"v{i}_cull"] = np.int64(cull)
            d.update(rs_arrays(rs, f"v{i}_rs_"))
            d[f"v{i}_bfs"] = full.node_ids.astype(np.int64)
        d["n_views"] = np.int64(len(views))
        np.savez_compressed(OUT / f"lod_{case:02d}.npz", **d)
        n_files += 1
    return n_files


def make_spt_cases():
    """cut_spt on single SPTs over a sweep of distances (test_spt.py:151-170),
    plus the hand-made toy SPT (test_spt.py:132-149)."""
    rng = np.random.default_rng(1234)
    d = {}
    k = 0
    for case in range(40):
        n = int(rng.integers(2, 400))
        h = build_hierarchy(random_leaves(rng, n))
        h.attrs.scales = rng.uniform(0.05, 2.0, h.attrs.scales.shape)
        cfg = LodConfig(threshold=float(rng.uniform(0.2, 20.0)),
                        metric=("max_scale", "surface_area")[case % 2])
        spt = build_spt(h, h.root, cfg)
        top = float(spt.key_self.max())
        dists = list(rng.uniform(0.0, 1.5 * top, 8)) + [float(spt.key_self[3 % spt.subtree_size]),
                                                         float(spt.key_self[0]), 0.0]
        for dist in dists:
            pl, sel = cut_spt(spt, float(dist))
            d[f"c{k}_root"] = np.int64(spt.root)
            d[f"c{k}_nodes"] = spt.nodes.astype(np.int64)
            d[f"c{k}_key_self"] = spt.key_self
            d[f"c{k}_key_parent"] = spt.key_parent
            d[f"c{k}_d"] = np.float64(dist)
            d[f"c{k}_prefix"] = np.int64(pl)
            d[f"c{k}_sel"] = sel.astype(np.int64)
            k += 1
    from glod.spt import Spt
    nodes = np.array([1, 2, 0], dtype=np.int64)
    ks = np.array([2.0, 3.0, 10.0])
    kp = np.array([10.0, 10.0, np.inf])
    o = np.argsort(-kp, kind="stable")
    toy = Spt(root=0, root_center=np.zeros(3), nodes=nodes[o], key_self=ks[o], key_parent=kp[o])
    for dist in (5.0, 20.0, 10.0, 2.0, 1.0):
        pl, sel = cut_spt(toy, dist)
        d[f"c{k}_root"] = np.int64(0)
        d[f"c{k}_nodes"] = toy.nodes
        d[f"c{k}_key_self"] = toy.key_self
        d[f"c{k}_key_parent"] = toy.key_parent
        d[f"c{k}_d"] = np.float64(dist)
        d[f"c{k}_prefix"] = np.int64(pl)
        d[f"c{k}_sel"] = sel.astype(np.int64)
        k += 1
    d["n_cases"] = np.int64(k)
    np.savez_compressed(OUT / "spt_cases.npz", **d)


def _cam_axis(resolution=(16, 16), focal=(40.0, 40.0), z=-10.0):
    w, h = resolution   # test_renderer.py:_make_camera
    return Camera(position=np.array([0.0, 0.0, z]), orientation=np.array([1.0, 0.0, 0.0, 0.0]),
                  focal=focal, principal_point=(w / 2.0, h / 2.0), resolution=resolution,
                  near=0.1)


def attrs_arrays(a, prefix):
    return {prefix + k: np.array(v, dtype=np.float64, copy=True) for k, v in a.arrays()}


def make_render_cases():
    """Forward image, backward gradients for a random upstream, and the
    L1+SSIM loss — micro scenes like test_renderer.py plus a denser scene
    with saturated pixels (exercises the T>1e-4 gate and the 0.99 clamp)."""
    rng = np.random.default_rng(777)
    d = {}
    k = 0
    specs = []
    for i in range(10):
        specs.append(("micro", int(rng.integers(1, 9)), (16, 16), (40.0, 40.0), 0.8))
    specs += [("mid", 60, (48, 40), (60.0, 55.0), 1.5), ("dense", 300, (64, 48), (70.0, 70.0), 1.2),
              ("saturate", 400, (40, 40), (50.0, 50.0), 0.6), ("wide", 150, (96, 64), (80.0, 80.0), 2.5)]
    for kind, n, res, focal, span in specs:
        a = random_leaves(rng, n, span=span, scale_lo=0.05, scale_hi=0.4)
        a.sh_rest = rng.normal(0, 0.1, a.sh_rest.shape)
        if kind == "saturate":
            a.opacities = rng.uniform(0.7, 1.0, n)
        cam = _cam_axis(resolution=res, focal=focal)
        if kind == "wide":
            cam = look_at_camera(np.array([1.0, -2.0, -9.0]), np.zeros(3), focal=focal,
                                 resolution=res, near=0.1)
        ctx = render_forward(a, cam)
        up = rng.normal(size=(res[1], res[0], 3))
        g = backward(ctx, up)
        target = rng.uniform(0, 1, ctx.image.shape)
        lv, lg = loss(ctx.image, target, 0.2)
        d.update(attrs_arrays(a, f"r{k}_a_"))
        d.update(cam_arrays(cam, f"r{k}_"))
        d[f"r{k}_image"] = ctx.image
        d[f"r{k}_upstream"] = up
        for name, arr in [("means", g.means), ("scales", g.scales), ("rotations", g.rotations),
                          ("opacities", g.opacities), ("base_colors", g.base_colors),
                          ("sh_rest", g.sh_rest)]:
            d[f"r{k}_g_{name}"] = arr
        d[f"r{k}_target"] = target
        d[f"r{k}_loss"] = np.float64(lv)
        d[f"r{k}_loss_grad"] = lg
        k += 1
    d["n_cases"] = np.int64(k)
    np.savez_compressed(OUT / "render_cases.npz", **d)


def make_adam_cases():
    from glod.trainer import DEFAULT_LEARNING_RATES, OptimizerState, _adam_update
    from glod.renderer import GaussianGradients
    rng = np.random.default_rng(99)
    n = 50
    a = random_leaves(rng, n)
    a.sh_rest = rng.normal(0, 0.1, a.sh_rest.shape)
    opt = OptimizerState.zeros(a)
    d = attrs_arrays(a, "p0_")
    lrs = dict(DEFAULT_LEARNING_RATES)
    lrs["means"] = lrs["means"] * 17.0
    for it in range(3):
        ids = np.sort(rng.choice(n, size=30, replace=False))
        g = GaussianGradients(means=rng.normal(size=(30, 3)), scales=rng.normal(size=(30, 3)),
                              rotations=rng.normal(size=(30, 4)), opacities=rng.normal(size=30),
                              base_colors=rng.normal(size=(30, 3)), sh_rest=rng.normal(size=(30, 9)))
        _adam_update(a, opt, ids, g, np.arange(30), lrs)
        d[f"it{it}_ids"] = ids
        for name in ("means", "scales", "rotations", "opacities", "base_colors", "sh_rest"):
            d[f"it{it}_g_{name}"] = getattr(g, name)
        d.update(attrs_arrays(a, f"it{it}_p_"))
        for name in opt.m:
            d[f"it{it}_m_{name}"] = opt.m[name].copy()
            d[f"it{it}_v_{name}"] = opt.v[name].copy()
        d[f"it{it}_step"] = opt.step.copy()
    for k, v in lrs.items():
        d[f"lr_{k}"] = np.float64(v)
    np.savez_compressed(OUT / "adam_cases.npz", **d)


if __name__ == "__main__" and len(sys.argv) == 1:
    print("lod files", make_lod_cases())
    make_spt_cases()
    make_render_cases()
    make_adam_cases()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, os.path.getsize(f))


def make_scheduler_cases():
    """View sequences from scheduler.build_view_graph/next_view (scheduler.py:38-77)."""
    from glod.scheduler import build_view_graph, next_view
    rng = np.random.default_rng(5)
    d = {}
    for c in range(4):
        n = int(rng.integers(5, 40))
        pos = rng.normal(size=(n, 3)) * 10
        if c == 3:
            pos[1] = pos[0]          # duplicate positions: ties broken by index
        k = int(rng.integers(1, 20))
        g = build_view_graph(pos, k=k, random_every=int(rng.integers(2, 15)))
        r = np.random.default_rng(100 + c)
        cur, seq = 0, []
        for it in range(1, 200):
            cur = next_view(g, cur, it, r)
            seq.append(cur)
        d[f"s{c}_pos"] = pos
        d[f"s{c}_k"] = np.int64(k)
        d[f"s{c}_random_every"] = np.int64(g.random_every)
        d[f"s{c}_neighbors"] = g.neighbors
        d[f"s{c}_weights"] = g.weights
        d[f"s{c}_seq"] = np.array(seq, dtype=np.int64)
    d["n_cases"] = np.int64(4)
    np.savez_compressed(OUT / "scheduler_cases.npz", **d)


def make_cache_cases():
    """Random operation traces on the reference DeviceCache (cache.py:42-109)
    with the resulting hit/miss/evicted/resident sequences."""
    from glod.cache import CacheConfig, CacheEntry, DeviceCache
    from glod.store import AttributeBlock
    rng = np.random.default_rng(1007)
    d = {}
    for c in range(5):
        budget = int(rng.integers(500, 5000))
        flush = int(rng.integers(5, 50))
        cache = DeviceCache(config=CacheConfig(budget_bytes=budget, flush_interval=flush))
        ops, res = [], []
        for op in range(1, 1501):
            kind = rng.uniform()
            sid = int(rng.integers(0, 30))
            if kind < 0.5:
                dd = float(rng.uniform(0.0, 3.0))
                hit = cache.lookup(sid, dd) is not None
                ops.append((0, sid, dd, 0, 0))
                res.append([int(hit)])
            elif kind < 0.9:
                dd = float(rng.uniform(0.5, 2.0))
                nb = int(rng.integers(1, budget + 1))
                dirty = int(rng.integers(2))
                blk = AttributeBlock(spt_id=sid, prefix_len=0, attrs=AttributeArrays.zeros(0))
                ev = cache.insert(CacheEntry(spt_id=sid, cached_distance=dd, prefix_len=0, block=blk,
                                             nbytes=nb, dirty=bool(dirty)))
                ops.append((1, sid, dd, nb, dirty))
                res.append([e[0] for e in ev])
            else:
                fl = cache.tick_and_maybe_flush(op)
                ops.append((2, op, 0.0, 0, 0))
                res.append([e[0] for e in fl])
            res[-1] = res[-1] + [-7] + list(cache.resident_ids()) + [-8, cache.resident_bytes,
                                                                      cache.hits, cache.misses]
        d[f"c{c}_budget"] = np.int64(budget)
        d[f"c{c}_flush"] = np.int64(flush)
        d[f"c{c}_ops"] = np.array(ops, dtype=np.float64)
        lens = np.array([len(r) for r in res], dtype=np.int64)
        d[f"c{c}_reslen"] = lens
        d[f"c{c}_res"] = np.concatenate([np.array(r, dtype=np.int64) for r in res])
    d["n_cases"] = np.int64(5)
    np.savez_compressed(OUT / "cache_cases.npz", **d)


def make_serve_cases():
    """ServeSession.handle_pose message streams (protocol.py:152-193) over
    camera paths: first pose, repeated pose (stats only), moves that load
    and evict SPTs, a pose facing away (everything culled) and back."""
    from glod.protocol import ServeSession
    rng = np.random.default_rng(777)
    d = {}
    for case in range(4):
        n = int(rng.choice([300, 900, 2000]))
        h = build_hierarchy(random_leaves(rng, n))
        if case % 2:
            thr = _designed_scales(rng, h, int(rng.integers(2, 5)))
            min_sub = 8
        else:
            h.attrs.scales = rng.uniform(0.05, 2.0, h.attrs.scales.shape)
            thr = float(np.quantile(np.prod(h.attrs.scales, axis=1), 0.5))
            min_sub = int(rng.choice([4, 8, 16]))
        lod = LodConfig(threshold=float(rng.uniform(1.0, 20.0) if case % 2 == 0 else rng.uniform(0.5, 6.0)),
                        metric=("max_scale", "surface_area")[case % 2])
        hspt = build_hspt(h, thr, min_sub, lod)
        sess = ServeSession(hierarchy=h, hspt=hspt, lod=lod)
        p = f"c{case}_"
        d.update({p + k: v for k, v in hier_arrays(h).items()})
        d.update({p + k: v for k, v in hspt_arrays(hspt).items()})
        cams = []
        for v in range(8):
            if v == 2:
                cam = cams[1]                                     # repeated pose
            elif v == 5:
                c = cams[4]                                       # facing away
                cam = look_at_camera(c.position, 2 * c.position, focal=(40.0, 40.0))
            else:
                pos = rng.uniform(-25, 25, 3) * (0.3 + 0.2 * v)
                cam = look_at_camera(pos, rng.uniform(-3, 3, 3), focal=(40.0, 40.0))
            cams.append(cam)
            msgs = sess.handle_pose(cam)
            d.update(cam_arrays(cam, p + f"v{v}_"))
            d[p + f"v{v}_lens"] = np.array([len(m) for m in msgs], dtype=np.int64)
            d[p + f"v{v}_bytes"] = np.frombuffer(b"".join(msgs), dtype=np.uint8)
        d[p + "n_views"] = np.int64(len(cams))
    d["n_cases"] = np.int64(4)
    np.savez_compressed(OUT / "serve_cases.npz", **d)


def make_scenefile_cases():
    """write_scene bytes (store.py:157-234) and what open_scene reads back
    (read_hierarchy / read_hspt / load_spt_prefix, store.py:304-393)."""
    from glod.store import MemoryBacking, open_scene, write_scene
    rng = np.random.default_rng(4242)
    d = {}
    for case in range(3):
        n = int([150, 600, 1200][case])
        h = build_hierarchy(random_leaves(rng, n))
        h.attrs.sh_rest = rng.normal(0, 0.1, h.attrs.sh_rest.shape)
        h.attrs.scales = rng.uniform(0.05, 2.0, h.attrs.scales.shape)
        thr = float(np.quantile(np.prod(h.attrs.scales, axis=1), 0.5))
        lod = LodConfig(threshold=float(rng.uniform(1.0, 20.0)), metric=("max_scale", "surface_area")[case % 2])
        hspt = build_hspt(h, thr, [4, 8, 16][case], lod)
        mb = MemoryBacking()
        write_scene(h, hspt, mb)
        p = f"c{case}_"
        d.update({p + k: v for k, v in hier_arrays(h).items()})
        d.update({p + k: v for k, v in hspt_arrays(hspt).items()})
        d[p + "file"] = np.frombuffer(mb.tobytes(), dtype=np.uint8)
        sc = open_scene(MemoryBacking(mb.tobytes()))
        h2, hs2 = sc.read_hierarchy(), sc.read_hspt()
        d.update({p + "rd_" + k: v for k, v in hier_arrays(h2).items()})
        d.update({p + "rd_" + k: v for k, v in hspt_arrays(hs2).items()})
        sid = len(hs2.spts) // 2
        blk = sc.load_spt_prefix(sid, hs2.spts[sid].subtree_size // 2)
        d[p + "pf_spt"] = np.int64(sid)
        d[p + "pf_len"] = np.int64(blk.prefix_len)
        d[p + "pf_means"] = blk.attrs.means
        d[p + "pf_sh"] = blk.attrs.sh_rest
        d[p + "pf_slot"] = np.int64(sc.spt_slot_start(sid))
        d[p + "bytes_read"] = np.int64(sc.attribute_bytes_read)
    d["n_cases"] = np.int64(3)
    np.savez_compressed(OUT / "scenefile_cases.npz", **d)


def make_densify_cases():
    """trainer.densify (trainer.py:411-443) on reference TrainStates: dead
    leaves respawned, opacity-sampled spawns, moments reset/grown, the HSPT
    rebuilt with the surface-area metric; plus the RNG's next draw."""
    from glod.cache import DeviceCache
    from glod.store import MemoryBacking, open_scene, write_scene
    from glod.trainer import OptimizerState, TrainConfig, TrainState, densify
    rng = np.random.default_rng(99)
    d = {}
    for case in range(3):
        n = int([200, 700, 1500][case])
        h = build_hierarchy(random_leaves(rng, n))
        h.attrs.sh_rest = rng.normal(0, 0.1, h.attrs.sh_rest.shape)
        h.attrs.scales = rng.uniform(0.05, 2.0, h.attrs.scales.shape)
        leaves = h.leaf_ids
        dead = rng.choice(leaves, size=max(2, n // 25), replace=False)
        h.attrs.opacities[dead] = rng.uniform(0.0, 0.004, dead.size)
        thr = float(np.quantile(np.prod(h.attrs.scales, axis=1), 0.5))
        lod = LodConfig(threshold=float(rng.uniform(1.0, 20.0)), metric="max_scale")
        hspt = build_hspt(h, thr, [4, 8, 16][case], lod)
        mb = MemoryBacking()
        write_scene(h, hspt, mb)
        opt = OptimizerState.zeros(h.attrs)
        for k in opt.m:
            opt.m[k] = rng.normal(0, 1e-3, opt.m[k].shape)
            opt.v[k] = rng.uniform(0, 1e-5, opt.v[k].shape)
        opt.step = rng.integers(0, 50, h.capacity).astype(np.int64)
        spawns = [None, 7, 0][case]
        cfg = TrainConfig(total_iterations=1000, spawns_per_densify=spawns)
        p = f"c{case}_"
        # copies: densify mutates the hierarchy's arrays in place
        d.update({p + k: np.array(v, copy=True) for k, v in hier_arrays(h).items()})
        d.update({p + k: np.array(v, copy=True) for k, v in hspt_arrays(hspt).items()})
        for k in opt.m:
            d[p + "m_" + k] = opt.m[k].copy()
            d[p + "v_" + k] = opt.v[k].copy()
        d[p + "step"] = opt.step.copy()
        d[p + "seed"] = np.int64(1000 + case)
        d[p + "spawns"] = np.int64(-1 if spawns is None else spawns)
        state = TrainState(config=cfg, hierarchy=h, hspt=hspt, scene=open_scene(mb),
                           cache=DeviceCache(config=cfg.cache), graph=None, views=[], opt=opt,
                           rng=np.random.default_rng(1000 + case), extent=1.0,
                           skybox_ids=np.zeros(0, dtype=np.int64))
        out = densify(state)
        d[p + "out_spawned"] = np.int64(out["spawned"])
        d[p + "out_respawned"] = np.int64(out["respawned"])
        d.update({p + "out_" + k: v for k, v in hier_arrays(state.hierarchy).items()})
        d[p + "out_free"] = np.array(state.hierarchy.free, dtype=np.int64)
        d.update({p + "out_" + k: v for k, v in hspt_arrays(state.hspt).items()})
        for k in state.opt.m:
            d[p + "out_m_" + k] = state.opt.m[k]
            d[p + "out_v_" + k] = state.opt.v[k]
        d[p + "out_step"] = state.opt.step
        d[p + "out_next_draw"] = np.float64(state.rng.random())
    d["n_cases"] = np.int64(3)
    np.savez_compressed(OUT / "densify_cases.npz", **d)



def make_train_cases():
    """trainer.train_step (trainer.py:312-378) on reference TrainStates built
    from a .glod file (write_scene → open_scene → read_hierarchy/read_hspt,
    so every value is f32-representable and the SPT keys are f32): per step
    the scheduled view, every returned counter, the loss and the rendered
    node-id order; the rendered image and the raw gradients for the first
    steps; the full state (params, moments, step counts, store sections,
    cache entries with their blocks) at checkpoints.  The traces cover
    misses, hits, LRU evictions, same-step re-misses of a replaced dirty
    entry (the stale-store quirk, trainer.py:333-341) and periodic flushes
    (cache.py:98-106)."""
    sys.path.insert(0, str(OUT.parent.parent))
    from glod.cache import CacheConfig, DeviceCache
    from glod.hierarchy import Hierarchy as RefHierarchy
    from glod.scheduler import build_view_graph
    from glod.store import MemoryBacking, open_scene, write_scene
    import glod.trainer as TR
    from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene, orbit_views, scene_extent

    events = {}
    orig_insert = DeviceCache.insert
    orig_tick = DeviceCache.tick_and_maybe_flush

    def insert(self, entry):
        out = orig_insert(self, entry)
        for sid, _ in out:
            k = "replace_dirty" if sid == entry.spt_id else "evict_dirty"
            events[k] = events.get(k, 0) + 1
        return out

    def tick(self, it):
        out = orig_tick(self, it)
        if out:
            events["flush"] = events.get("flush", 0) + len(out)
        return out

    DeviceCache.insert, DeviceCache.tick_and_maybe_flush = insert, tick
    cap_rows = {}
    orig_cut, orig_pos, orig_fwd, orig_bwd = TR.cut_hspt, TR._spt_positions, TR.render_forward, TR.backward

    def cut(*a, **k):
        rs = orig_cut(*a, **k)
        cap_rows["rows"] = [np.asarray(rs.upper, np.int64), np.asarray(rs.passthrough, np.int64)]
        return rs

    def pos(spt, d):
        out = orig_pos(spt, d)
        cap_rows["rows"].append(np.asarray(out[2], np.int64))
        return out

    def fwd(attrs, cam):
        ctx = orig_fwd(attrs, cam)
        cap_rows["image"] = ctx.image.copy()
        return ctx

    def bwd(ctx, dimg):
        g = orig_bwd(ctx, dimg)
        cap_rows["grads"] = np.concatenate([np.asarray(getattr(g, n), np.float64).reshape(-1, c)
                                            for n, c in (("means", 3), ("scales", 3), ("rotations", 4),
                                                         ("opacities", 1), ("base_colors", 3), ("sh_rest", 9))],
                                           axis=1)
        return g

    TR.cut_hspt, TR._spt_positions, TR.render_forward, TR.backward = cut, pos, fwd, bwd
    d = {}
    specs = [  # leaves, seed, spt_leaves, budget (share of all records), flush, steps, res, views, k
        (1500, 3, 256, 0.6, 7, 16, (64, 48), 8, 4),
        (1500, 5, 128, 0.3, 5, 16, (64, 48), 8, 3),
    ]
    try:
        for case, (n, seed, sptl, bfrac, flush, steps, res, nviews, k) in enumerate(specs):
            events.clear()
            h, hs, cfg = designed_scene(SceneSpec(n_leaves=n, spt_leaves=sptl, seed=seed, pass_fraction=0.1))
            a = h.attrs
            rh = RefHierarchy(attrs=AttributeArrays(a.means.copy(), a.scales.copy(), a.rotations.copy(),
                                                    a.opacities.copy(), a.base_colors.copy(), a.sh_rest.copy()),
                              parent=h.parent.astype(np.int32).copy(), children=h.children.astype(np.int32).copy(),
                              root=int(h.root))
            lod = LodConfig(cfg.threshold, cfg.metric)
            rhs = build_hspt(rh, hs.size_threshold, hs.min_subtree, lod)
            mb = MemoryBacking()
            write_scene(rh, rhs, mb)
            file_bytes = mb.tobytes()
            scene = open_scene(mb)
            h2, hs2 = scene.read_hierarchy(), scene.read_hspt()
            E = scene_extent(n)
            cams = orbit_views(nviews, 1.5 * E, 0.6 * E, resolution=res, focal=(70.0, 70.0), seed=seed,
                               jitter=0.2)
            cams = [Camera(position=c.position, orientation=c.orientation, focal=c.focal,
                           principal_point=c.principal_point, resolution=c.resolution, near=c.near)
                    for c in cams]
            rng = np.random.default_rng(seed)
            # f32-representable targets: the device keeps targets in f32
            targets = [np.clip(rng.normal(0.5, 0.2, (res[1], res[0], 3)), 0, 1).astype(np.float32)
                       .astype(np.float64) for _ in cams]
            nrec = sum(s.subtree_size for s in hs2.spts)
            budget = int(bfrac * nrec * 92)
            tcfg = TR.TrainConfig(total_iterations=steps, lod=lod,
                                  cache=CacheConfig(budget_bytes=budget, flush_interval=flush),
                                  scheduler_k=k, seed=seed)
            graph = build_view_graph(np.stack([c.position for c in cams]), k=k)
            extent = 2.0 * E
            st = TR.TrainState(config=tcfg, hierarchy=h2, hspt=hs2, scene=scene,
                               cache=DeviceCache(config=tcfg.cache), graph=graph,
                               views=list(zip(cams, targets)), opt=TR.OptimizerState.zeros(h2.attrs),
                               rng=np.random.default_rng(seed), extent=extent,
                               skybox_ids=np.zeros(0, dtype=np.int64))
            p = f"c{case}_"
            d[p + "file"] = np.frombuffer(file_bytes, dtype=np.uint8)
            d.update({p + k2: v for k2, v in hier_arrays(h2).items()})
            d.update({p + k2: v for k2, v in hspt_arrays(hs2).items()})
            for v, c in enumerate(cams):
                d.update(cam_arrays(c, p + f"cam{v}_"))
            d[p + "targets"] = np.stack(targets).astype(np.float32)
            d[p + "n_views"] = np.int64(nviews)
            d[p + "budget"] = np.int64(budget)
            d[p + "flush"] = np.int64(flush)
            d[p + "k"] = np.int64(k)
            d[p + "seed"] = np.int64(seed)
            d[p + "extent"] = np.float64(extent)
            d[p + "steps"] = np.int64(steps)
            d[p + "lod_T"] = np.float64(lod.threshold)
            d[p + "lod_metric"] = np.int64(0 if lod.metric == "max_scale" else 1)
            checkpoints = (1, steps)
            counters = []
            for it in range(1, steps + 1):
                r = TR.train_step(st, it)
                counters.append([r["view"], r["gaussians_rendered"], r["gaussians_loaded_from_store"],
                                 r["cache_hits"], r["bytes_streamed"]])
                q = p + f"it{it}_"
                d[q + "loss"] = np.float64(r["loss"])
                d[q + "rows"] = np.concatenate(cap_rows["rows"]).astype(np.int32)
                if it <= 2:
                    d[q + "image"] = cap_rows["image"]
                    d[q + "grads"] = cap_rows["grads"]
                if it in checkpoints:
                    d.update({q + "p_" + k2: np.array(v, copy=True) for k2, v in hier_arrays(h2).items()
                              if k2 in ("means", "scales", "rotations", "opacities", "base_colors", "sh_rest")})
                    for k2 in st.opt.m:
                        d[q + "m_" + k2] = st.opt.m[k2].copy()
                        d[q + "v_" + k2] = st.opt.v[k2].copy()
                    d[q + "step"] = st.opt.step.copy()
                    sc = st.scene
                    for name, cols in (("means", 3), ("scales", 3), ("rotations", 4), ("opacities", 1),
                                       ("base_colors", 3), ("sh_rest", 9)):
                        off, length = sc.sections[name]
                        d[q + "store_" + name] = np.frombuffer(bytes(sc.backing.buf[off:off + length]),
                                                               dtype="<f4").copy()
                    ents = list(st.cache.entries.values())
                    d[q + "cache_sid"] = np.array([e.spt_id for e in ents], dtype=np.int64)
                    d[q + "cache_dist"] = np.array([e.cached_distance for e in ents], dtype=np.float64)
                    d[q + "cache_prefix"] = np.array([e.prefix_len for e in ents], dtype=np.int64)
                    d[q + "cache_dirty"] = np.array([e.dirty for e in ents], dtype=np.int64)
                    d[q + "cache_blocks"] = (np.concatenate([np.concatenate(
                        [np.asarray(getattr(e.block.attrs, nm), np.float64).reshape(e.prefix_len, -1)
                         for nm in ("means", "scales", "rotations", "opacities", "base_colors", "sh_rest")],
                        axis=1) for e in ents]) if ents else np.zeros((0, 23)))
            d[p + "counters"] = np.array(counters, dtype=np.int64)
            d[p + "checkpoints"] = np.array(checkpoints, dtype=np.int64)
            d[p + "events"] = np.array([events.get("evict_dirty", 0), events.get("replace_dirty", 0),
                                        events.get("flush", 0)], dtype=np.int64)
            print("train case", case, "counters", counters, "events", dict(events))
    finally:
        DeviceCache.insert, DeviceCache.tick_and_maybe_flush = orig_insert, orig_tick
        TR.cut_hspt, TR._spt_positions, TR.render_forward, TR.backward = orig_cut, orig_pos, orig_fwd, orig_bwd
    d["n_cases"] = np.int64(len(specs))
    np.savez_compressed(OUT / "train_cases.npz", **d)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"make_{name}_cases"]()
        sys.exit(0)
    make_scheduler_cases()
    make_cache_cases()
    make_serve_cases()
    make_scenefile_cases()
    make_densify_cases()
    make_train_cases()
