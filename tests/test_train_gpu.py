"""GPU train_step parity against the oracle's restatement of
trainer.train_step (store + device-cache semantics included).

Each GPU step is checked from an identical state: the oracle is re-synced
from a snapshot of the GPU state (params, moments, step counts, pinned
store, cache entries and blocks) taken just before the step.  Checked:
scheduled view, every counter (exact), render-set size (exact), loss
(1e-5 relative), per-row gradients (1e-3 relative, see test_render_gpu),
and the post-step parameters (ADAM: tight except where a near-zero
gradient's sign is ambiguous — there the update may differ by ≤ 2·lr).
"""
from __future__ import annotations

from collections import OrderedDict

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import glod_oracle as O  # noqa: E402
from oracle.train_oracle import OracleTrainer  # noqa: E402
from paper_2507_01110_b200.cache import CacheConfig  # noqa: E402
from paper_2507_01110_b200.core import SECTIONS, AttributeArrays  # noqa: E402
from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene, orbit_views, scene_extent  # noqa: E402
from paper_2507_01110_b200.trainer import TrainConfig, Trainer  # noqa: E402

from .test_render_gpu import assert_grads_close  # noqa: E402

NAMES = [n for n, _ in SECTIONS]



def same_state(a, b):
    """Equal state across two runs of the same steps.  The backward blend
    accumulates per-Gaussian partials with fp64 atomics whose order is not
    fixed, so a sum that is not exact in fp64 may round differently between
    runs (last-bit differences); everything else is deterministic."""
    a, b = a.double(), b.double()
    return torch.equal(a, b) or torch.allclose(a, b, rtol=1e-10, atol=1e-14)

def _dict(a: AttributeArrays):
    return {k: np.array(getattr(a, k), copy=True) for k in NAMES}


def snapshot(tr: Trainer):
    torch.cuda.synchronize()
    sc = tr.scene
    cap = sc.cap
    m, v = sc.moments_packed()
    snap = {"P": _dict(AttributeArrays.from_packed(sc.params.cpu().numpy(), cap)),
            "M": _dict(AttributeArrays.from_packed(m.cpu().numpy(), cap)),
            "V": _dict(AttributeArrays.from_packed(v.cpu().numpy(), cap)),
            "step": sc.step.cpu().numpy().copy(),
            "store": [s.numpy().copy() for s in sc.store.sections],
            "cache": OrderedDict(), "resident": tr.cache.resident_bytes}
    for sid, cd, pl, addr, dirty in tr.cache.entries():
        blk = _dict(AttributeArrays.from_packed(tr.cache.read_block(addr, pl), pl))
        snap["cache"][sid] = [cd, pl, blk, dirty]
    return snap


def restore(orc: OracleTrainer, snap):
    orc.P = {k: v.copy() for k, v in snap["P"].items()}
    orc.M = {k: v.copy() for k, v in snap["M"].items()}
    orc.V = {k: v.copy() for k, v in snap["V"].items()}
    orc.step = snap["step"].copy()
    orc.store = [s.copy() for s in snap["store"]]
    orc.cache = OrderedDict((k, [e[0], e[1], {n: a.copy() for n, a in e[2].items()}, e[3]])
                            for k, e in snap["cache"].items())
    orc.resident = snap["resident"]


def make_case(n_leaves=6000, res=(96, 64), n_views=10, budget_frac=0.35, seed=3, store_location="host"):
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=n_leaves, spt_leaves=256, seed=seed,
                                          pass_fraction=0.1))
    E = scene_extent(n_leaves)
    cams = orbit_views(n_views, 1.5 * E, 0.6 * E, resolution=res, focal=(70.0, 70.0), seed=seed,
                       jitter=0.2)
    rng = np.random.default_rng(seed)
    targets = [np.clip(rng.normal(0.5, 0.2, (res[1], res[0], 3)), 0, 1) for _ in cams]
    budget = int(budget_frac * hs.flat_records()["nodes"].size * 92)
    tcfg = TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=budget, flush_interval=7),
                       scheduler_k=4, seed=seed, store_location=store_location)
    tr = Trainer(h, hs, list(zip(cams, targets)), tcfg, extent=2 * E)
    flat = hs.flat_records()
    kind = np.full(h.capacity, -1, np.int32)
    kind[flat["roots"]] = np.arange(flat["roots"].size)
    kind[hs.passthrough_roots] = -2
    st = tr.scene.store
    lrs = dict(tcfg.learning_rates)
    lrs["means"] *= 2 * E
    orc = OracleTrainer(_dict(h.attrs), h.children, h.root, kind, flat,
                        [s.cpu().numpy() for s in st.sections],
                        [st.spt_slot_start(i) for i in range(len(hs.spts))],
                        [(O.Cam.of(c), t) for c, t in zip(cams, targets)], cfg.threshold,
                        cfg.metric_code, budget, flush_interval=7, lrs=lrs)
    return tr, orc, lrs


def test_train_steps_match_oracle():
    tr, orc, lrs = make_case()
    saw_miss = saw_hit = False
    for it in range(1, 13):
        snap = snapshot(tr)
        got = tr.train_step(it)
        restore(orc, snap)
        want, extra = orc.train_step(it, view=got["view"])
        for k in ("view", "gaussians_rendered", "gaussians_loaded_from_store", "cache_hits",
                  "bytes_streamed"):
            assert got[k] == want[k], (it, k, got[k], want[k])
        assert abs(got["loss"] - want["loss"]) <= 1e-5 * abs(want["loss"]), it
        R = got["gaussians_rendered"]
        g = AttributeArrays.from_packed(tr._last_grads[:23 * R].cpu().numpy(), R)
        assert_grads_close(g, extra["grads"], where=f"step {it}")
        post = AttributeArrays.from_packed(tr.scene.params.cpu().numpy(), tr.scene.cap)
        for k, (name, _) in enumerate(SECTIONS):
            a, b = getattr(post, name), orc.P[name]
            d = np.abs(a - b)
            lr = lrs[name] if name not in ("scales", "opacities") else 1.0
            assert np.all(d <= 2.5 * lr * np.maximum(1.0, np.abs(b)) + 1e-12), (it, name, d.max())
            assert np.mean(d <= 1e-7 * np.maximum(1.0, np.abs(b))) > 0.98, (it, name)
        saw_miss |= got["gaussians_loaded_from_store"] > 0
        saw_hit |= got["cache_hits"] > 0
    assert saw_miss and saw_hit


def test_warm_cache_zero_loads():
    """test_trainer.py:154-168: revisiting the same view with a warm cache
    loads nothing from the store."""
    tr, _, _ = make_case(budget_frac=2.0)
    tr.graph.random_every = 1   # uniform draws; then pin the view below
    first = None
    for it in range(1, 4):
        tr.rng = np.random.default_rng(0)
        r = tr.train_step(it * 1)
        if first is None:
            first = r
        else:
            assert r["view"] == first["view"]
            assert r["gaussians_loaded_from_store"] == 0
            assert r["bytes_streamed"] == 0


def test_prefetch_is_invisible():
    """The copy-engine prefetch of the predicted next view changes where a
    missed prefix is read from (an HBM copy made during the previous step),
    never what: 20 steps with misses, evictions, same-step re-misses and
    flushes leave params, moments, step counts, the pinned store and every
    cache block bit-identical to a run without prefetch."""
    a, _, _ = make_case()
    b, _, _ = make_case()
    b.cfg.prefetch = False
    for it in range(1, 21):
        ra, rb = a.train_step(it), b.train_step(it)
        assert ra == rb, it
    torch.cuda.synchronize()
    st = a.cache.stats()
    assert st["prefetch_used_rows"] > 0 and b.cache.stats()["prefetched_rows"] == 0
    assert same_state(a.scene.params, b.scene.params)
    assert same_state(a.scene.mv, b.scene.mv)
    assert torch.equal(a.scene.step, b.scene.step)
    for sa, sb in zip(a.scene.store.sections, b.scene.store.sections):
        assert same_state(sa, sb)
    ea, eb = a.cache.entries(), b.cache.entries()
    assert [e[:3] + e[4:] for e in ea] == [e[:3] + e[4:] for e in eb]
    for x, y in zip(ea, eb):
        ba, bb = a.cache.read_block(x[3], x[2]), b.cache.read_block(y[3], y[2])
        assert np.array_equal(ba, bb) or np.allclose(ba, bb, rtol=1e-10, atol=1e-14)


def test_device_store_matches_host_store():
    """C2's device-resident store (sections in HBM) runs the same transfer
    paths device-to-device: identical counters, parameters and store."""
    a, _, _ = make_case()
    b, _, _ = make_case(store_location="device")
    for it in range(1, 11):
        assert a.train_step(it) == b.train_step(it), it
    torch.cuda.synchronize()
    assert same_state(a.scene.params, b.scene.params)
    for sa, sb in zip(a.scene.store.sections, b.scene.store.sections):
        assert same_state(sa, sb.cpu())


def test_empty_view_trains():
    """A view whose cut is empty (camera facing away from the scene) renders
    the black background, has a finite loss and updates nothing."""
    from paper_2507_01110_b200.scenegen import look_at
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=4000, spt_leaves=256, seed=2))
    E = scene_extent(4000)
    cams = [look_at([3 * E, E, 0.0], [6 * E, E, 0.0], (70.0, 70.0), (64, 48)) for _ in range(3)]
    cams[1] = look_at([3 * E, E, 1.0], [6 * E, 2 * E, 1.0], (70.0, 70.0), (64, 48))
    targets = [np.full((48, 64, 3), 0.5) for _ in cams]
    tr = Trainer(h, hs, list(zip(cams, targets)), TrainConfig(lod=cfg, scheduler_k=2), extent=2 * E)
    before = tr.scene.params.clone()
    for it in range(1, 4):
        r = tr.train_step(it)
        assert r["gaussians_rendered"] == 0 and np.isfinite(r["loss"])
    torch.cuda.synchronize()
    assert torch.equal(before, tr.scene.params)


def test_host_targets_match_device_targets():
    """e2e mode: targets in pinned host memory are uploaded on a side stream
    (double-buffered, overlapping the cut/gather/forward); losses and
    parameters are identical to device-resident targets."""
    a, _, _ = make_case()
    b, _, _ = make_case()
    b.targets = [t.cpu().pin_memory() for t in b.targets]
    b.device_targets = False
    for it in range(1, 13):
        assert a.train_step(it) == b.train_step(it), it
    torch.cuda.synchronize()
    assert same_state(a.scene.params, b.scene.params)


def test_non_finite_loss_raises_before_adam():
    """trainer.py:360-367: a non-finite loss raises NonFiniteLossError and
    leaves the parameters untouched (the backward may already have run; the
    check precedes ADAM, the first write to the parameters)."""
    from paper_2507_01110_b200.trainer import NonFiniteLossError
    tr, _, _ = make_case()
    tr.train_step(1)
    torch.cuda.synchronize()
    before = tr.scene.records.clone()
    for t in tr.targets:
        t.fill_(float("nan"))
    with pytest.raises(NonFiniteLossError):
        tr.train_step(2)
    torch.cuda.synchronize()
    assert torch.equal(before, tr.scene.records)


def test_render_prefetch_is_invisible():
    """render_view with the next frame known prefetches that frame's misses
    on the copy engines: identical images and counters to the path without."""
    a, _, _ = make_case(budget_frac=0.3)
    b, _, _ = make_case(budget_frac=0.3)
    n = len(a.views)
    used = 0
    for f in range(12):
        v, nv = (3 * f) % n, (3 * f + 3) % n
        ia = a.render_view(v)
        ib = b.render_view(v, next_view=nv)
        assert a.last_render == b.last_render, f
        assert torch.equal(ia, ib), f
    torch.cuda.synchronize()
    assert b.cache.stats()["prefetch_used_rows"] > 0


def test_disk_store_matches_host_store(tmp_path):
    """Disk mode (FileBacking, store.py:84-112): the store
    stays in the .glod file — misses pread + H2D (prefetches overlapping the
    step), write-backs D2H + pwrite before the next read.  Against the
    pinned-DRAM store of the same file: identical counters every step
    (misses, hits, evictions, re-misses, flushes), the same parameters, and
    after a flush the file holds exactly the pinned store's bytes."""
    import shutil
    from paper_2507_01110_b200 import scenefile as SF
    h0, hs0, cfg = designed_scene(SceneSpec(n_leaves=6000, spt_leaves=256, seed=3, pass_fraction=0.1))
    pa, pb = tmp_path / "a.glod", tmp_path / "b.glod"
    SF.write_scene(h0, hs0, pa)
    shutil.copy(pa, pb)
    sa, sb = SF.open_scene(pa), SF.open_scene(pb)
    h, hs = sa.read_hierarchy(), sa.read_hspt()
    E = scene_extent(6000)
    cams = orbit_views(10, 1.5 * E, 0.6 * E, resolution=(96, 64), focal=(70.0, 70.0), seed=3, jitter=0.2)
    rng = np.random.default_rng(3)
    targets = [np.clip(rng.normal(0.5, 0.2, (64, 96, 3)), 0, 1) for _ in cams]
    budget = int(0.3 * hs.flat_records()["nodes"].size * 92)
    mk = lambda store: Trainer(h, hs, list(zip(cams, targets)),
                               TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=budget, flush_interval=7),
                                           scheduler_k=4, seed=3), extent=2 * E, store=store)
    a, b = mk(sa.host_store()), mk(sb.disk_store())
    assert b.scene.store.location == "disk"
    for it in range(1, 16):
        ra, rb = a.train_step(it), b.train_step(it)
        assert ra == rb, it
    a.flush_cache()
    b.flush_cache()
    torch.cuda.synchronize()
    io = b.cache.flush_io()
    assert io["file_bytes_read"] > 0 and io["file_bytes_written"] > 0
    assert same_state(a.scene.params, b.scene.params)
    assert same_state(a.scene.mv, b.scene.mv)
    for sa_, sb_ in zip(a.scene.store.sections, b.scene.store.sections):
        assert same_state(sa_, sb_)


def test_fused_gather_matches_gathered_rows():
    """glod_render_forward_plan (the K4 gather fused into the preprocess:
    render rows read in place from the master records and cache blocks,
    touched rows from the master) against the rasteriser on the K4-gathered
    packed copy: identical images, losses, gradients, row node ids and
    parameters over 12 train steps (misses, hits, flushes), and identical
    render_view frames (gradients and parameters up to the fp64-atomic
    ordering of the backward blend, see same_state)."""
    a, _, _ = make_case()
    b, _, _ = make_case()
    a.cfg.fuse_gather = True
    b.cfg.fuse_gather = False
    for it in range(1, 13):
        ra, rb = a.train_step(it), b.train_step(it)
        la, lb = ra.pop("loss"), rb.pop("loss")
        assert ra == rb and abs(la - lb) <= 1e-6 * abs(lb), it
        R = ra["gaussians_rendered"]
        assert torch.allclose(a._last_image, b._last_image, rtol=0, atol=1e-6), it
        assert same_state(a._last_grads[:23 * R], b._last_grads[:23 * R]), it
        assert torch.equal(a._last_rows, b._last_rows), it
    torch.cuda.synchronize()
    assert same_state(a.scene.records, b.scene.records)
    for v in range(len(a.views)):
        assert torch.allclose(a.render_view(v), b.render_view(v), rtol=0, atol=1e-6), v
        assert torch.equal(a._row_node[:a._plan_R], b._row_node[:b._plan_R]), v
        assert same_state(a.gathered_rows(), b.gathered_rows()), v


def test_fused_gather_render_bit_identical():
    """On one state and one plan, the frame rendered through the gather plan
    equals the frame rendered from the K4-gathered rows of that plan bit for
    bit (the forward is deterministic; only the backward's fp64 atomics are
    order-dependent)."""
    a, _, _ = make_case()
    for it in range(1, 6):
        a.train_step(it)
    a.cfg.fuse_gather = True
    for v in range(len(a.views)):
        i1 = a.render_view(v).clone()
        n1 = a._row_node[:a._plan_R].clone()
        rows = a.gathered_rows()
        assert torch.equal(n1, a._row_node[:a._plan_R]), v
        i2 = a.rast.forward(rows, a._plan_R, a.views[v][0])
        d = (i1 - i2).abs()
        assert torch.equal(i1, i2), (v, float(d.max()), int((d > 0).sum()))


def test_pipelined_render_matches():
    """render_view(view, next_view) with the next frame's select enqueued
    between this frame's tile sort and its blend (TrainConfig.pipeline_render)
    against the unpipelined path: identical frames and counters, also when
    the announced next view is not the one rendered next (the preselect is
    dropped) or no next view is given."""
    a, _, _ = make_case(budget_frac=0.3)
    b, _, _ = make_case(budget_frac=0.3)
    b.cfg.pipeline_render = False
    n = len(a.views)
    seq = [(3 * f) % n for f in range(14)]
    for f, v in enumerate(seq):
        nv = seq[f + 1] if f + 1 < len(seq) else None
        if f == 6:
            nv = (v + 1) % n if (v + 1) % n != seq[f + 1] else (v + 2) % n   # wrong guess
        if f == 9:
            nv = None
        ia = a.render_view(v, next_view=nv)
        ib = b.render_view(v, next_view=nv)
        assert a.last_render == b.last_render, f
        assert torch.equal(ia, ib), f
    torch.cuda.synchronize()


def test_deferred_blend_capi():
    """glod_render_defer_blend / glod_render_blend: the deferred frame equals
    the direct one; a blend with none pending and a backward before the
    deferred blend are refused."""
    from paper_2507_01110_b200 import _lib
    a, _, _ = make_case()
    a.train_step(1)
    rows = a.gathered_rows()
    R, cam = a._plan_R, a.views[a.current_view][0]
    want = a.rast.forward(rows, R, cam).clone()
    a.rast.defer_blend(True)
    img = a.rast.forward(rows, R, cam)
    a.rast.defer_blend(False)
    with pytest.raises((_lib.GlodError, ValueError)):
        a.rast.backward(torch.zeros_like(img))
    a.rast.blend()
    assert torch.equal(img, want)
    with pytest.raises((_lib.GlodError, ValueError)):
        a.rast.blend()
