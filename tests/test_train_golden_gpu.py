"""GPU train_step against the reference's own trainer.train_step traces
(tests/golden/train_cases.npz, minted by make_golden.py:make_train_cases):
the device Trainer and the drop-in `train_step(state, iteration)` run the
same steps from the same .glod file, free-running (no re-sync), and must
reproduce every scheduled view, every counter and the rendered node-id
order exactly; the loss to 1e-6 relative; the image of the first steps to
1e-4 max-abs and their raw gradients to 1e-3 relative; and at the
checkpoints the cache entries (id, cached distance, prefix, dirty) exactly,
the step counts exactly, and params / moments / store within the bounds an
fp32-per-pixel rasteriser allows (ADAM's first steps move a parameter by
≈ lr·sign(g), so a near-zero gradient whose sign differs moves it the other
way: the bound is 2·lr per step, and ≥ 98 % of values must agree to 1e-6)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2507_01110_b200 import trainer as TR  # noqa: E402
from paper_2507_01110_b200.cache import CacheConfig, DeviceCache  # noqa: E402
from paper_2507_01110_b200.core import SECTIONS, AttributeArrays, LodConfig  # noqa: E402
from paper_2507_01110_b200.scheduler import build_view_graph  # noqa: E402

from .test_render_gpu import assert_grads_close  # noqa: E402
from .train_golden import NAMES, cases  # noqa: E402

LR = {"means": None, "scales": 5e-3, "rotations": 1e-3, "opacities": 5e-2, "base_colors": 2.5e-3,
      "sh_rest": 2.5e-3 / 20.0}


def _cfg(tc, sc):
    return TR.TrainConfig(total_iterations=tc.steps, lod=LodConfig(sc.lod.threshold, sc.lod.metric),
                          cache=CacheConfig(budget_bytes=tc.budget, flush_interval=tc.flush),
                          scheduler_k=tc.k, seed=tc.seed)


def _close_frac(a, b, bound, where):
    """|a-b| ≤ bound everywhere, and ≥ 98 % of entries within 1e-6 rel."""
    d = np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))
    assert np.all(d <= bound + 1e-12), (where, float(d.max()), float(np.max(bound)))
    frac = float(np.mean(d <= 1e-6 * np.maximum(1.0, np.abs(b))))
    assert frac >= 0.98, (where, frac)


def check_step(got, want, image, grads, rows, where):
    for k in ("view", "gaussians_rendered", "gaussians_loaded_from_store", "cache_hits", "bytes_streamed"):
        assert got[k] == want[k], (where, k, got[k], want[k])
    assert abs(got["loss"] - want["loss"]) <= 1e-6 * abs(want["loss"]), (where, got["loss"], want["loss"])
    if rows is not None:
        np.testing.assert_array_equal(rows.cpu().numpy().astype(np.int64), want["rows"], err_msg=where)
    if "image" in want and image is not None:
        err = float(np.abs(image.cpu().numpy().astype(np.float64) - want["image"]).max())
        assert err <= 1e-4, (where, err)
        R = got["gaussians_rendered"]
        g = AttributeArrays.from_packed(grads[:23 * R].cpu().numpy(), R)
        parts = np.split(want["grads"], np.cumsum([c for _, c in SECTIONS])[:-1], axis=1)
        ref = {n: (x if x.shape[1] > 1 else x[:, 0]) for n, x in zip(NAMES, parts)}
        assert_grads_close(g, ref, where=where)


def check_state(P, M, V, step, store, entries, ref, it, lrs, where):
    np.testing.assert_array_equal(step, ref["step"], err_msg=f"{where} step")
    for n in NAMES:
        lr = lrs[n] if n not in ("scales", "opacities") else 1.0     # log / logit space: relative
        scale = np.maximum(1.0, np.abs(ref["P"][n]))
        _close_frac(P[n], ref["P"][n], 2.5 * it * lr * scale, f"{where} params {n}")
        mm = np.abs(ref["M"][n]).max() + 1e-30
        assert np.mean(np.abs(M[n] - ref["M"][n]) <= 1e-3 * (np.abs(ref["M"][n]) + 1e-3 * mm)) >= 0.98, where
        vv = np.abs(ref["V"][n]).max() + 1e-30
        assert np.mean(np.abs(V[n] - ref["V"][n]) <= 2e-3 * (np.abs(ref["V"][n]) + 1e-3 * vv)) >= 0.98, where
    for k, (a, b) in enumerate(zip(store, ref["store"])):
        n = NAMES[k]
        lr = lrs[n] if n not in ("scales", "opacities") else 1.0
        _close_frac(a.reshape(-1), b, 2.5 * it * lr * np.maximum(1.0, np.abs(b)) + 1e-6 * np.abs(b),
                    f"{where} store {n}")
    assert [(e[0], e[1], e[2], int(e[4])) for e in entries] == ref["cache"], where


def trainer_state(tr):
    torch.cuda.synchronize()
    sc = tr.scene
    P = AttributeArrays.from_packed(sc.params.cpu().numpy(), sc.cap)
    m, v = sc.moments_packed()
    M = AttributeArrays.from_packed(m.cpu().numpy(), sc.cap)
    V = AttributeArrays.from_packed(v.cpu().numpy(), sc.cap)
    return ({n: getattr(P, n) for n in NAMES}, {n: getattr(M, n) for n in NAMES},
            {n: getattr(V, n) for n in NAMES}, sc.step.cpu().numpy(),
            [s.cpu().numpy() for s in sc.store.sections], tr.cache.entries())


def test_trainer_matches_reference_trace(tmp_path):
    for ci, tc in enumerate(cases(tmp_path)):
        sc = tc.scene()
        h, hs = sc.read_hierarchy(), sc.read_hspt()
        cfg = _cfg(tc, hs)
        tr = TR.Trainer(h, hs, list(zip(tc.cams, tc.targets)), cfg, extent=tc.extent, store=sc.host_store())
        lrs = dict(LR, means=1.6e-4 * tc.extent)
        for it in range(1, tc.steps + 1):
            got = tr.train_step(it)
            where = f"case {ci} step {it}"
            check_step(got, tc.step(it), tr._last_image, tr._last_grads, tr._last_rows, where)
            if it in tc.checkpoints:
                check_state(*trainer_state(tr), tc.state(it), it, lrs, where)


def test_dropin_train_step_matches_reference_trace(tmp_path):
    """train_step(state, iteration) at the reference's signature
    (trainer.py:312) on a TrainState built like the reference's: same
    counters / loss / views, state.rng advanced by the draws, and
    sync_state writing params, moments, steps and the store back."""
    for ci, tc in enumerate(cases(tmp_path)):
        sc = tc.scene()
        h, hs = sc.read_hierarchy(), sc.read_hspt()
        cfg = _cfg(tc, hs)
        graph = build_view_graph(np.stack([c.position for c in tc.cams]), k=tc.k)
        st = TR.TrainState(config=cfg, hierarchy=h, hspt=hs, scene=sc, cache=DeviceCache(config=cfg.cache),
                           graph=graph, views=list(zip(tc.cams, tc.targets)),
                           opt=TR.OptimizerState.zeros(h.attrs), rng=np.random.default_rng(tc.seed),
                           extent=tc.extent, skybox_ids=np.zeros(0, np.int64))
        lrs = dict(LR, means=1.6e-4 * tc.extent)
        for it in range(1, tc.steps + 1):
            got = TR.train_step(st, it)
            want = tc.step(it)
            assert st.current_view == want["view"] and st.iteration == it
            tr = st._device_trainer
            check_step(got, want, tr._last_image, tr._last_grads, tr._last_rows, f"drop-in case {ci} step {it}")
        # sync_state flushes the device cache into the store and copies the
        # master state into the host objects
        TR.sync_state(st)
        ref = tc.state(tc.steps)
        np.testing.assert_array_equal(st.opt.step, ref["step"])
        for n in NAMES:
            lr = lrs[n] if n not in ("scales", "opacities") else 1.0
            _close_frac(getattr(h.attrs, n), ref["P"][n],
                        2.5 * tc.steps * lr * np.maximum(1.0, np.abs(ref["P"][n])), f"sync {n}")
        # the file now holds the flushed store: every resident dirty block of
        # the reference's cache, written back, equals what the device wrote
        sc2 = type(sc)(tc.path)
        blk_ref = ref["blocks"]
        off = 0
        for sid, dist, pl, dirty in ref["cache"]:
            b = sc2.load_spt_prefix(sid, pl)
            got = np.concatenate([np.asarray(getattr(b.attrs, n), np.float64).reshape(pl, -1) for n in NAMES],
                                 axis=1)
            want = blk_ref[off:off + pl].astype(np.float32).astype(np.float64)
            assert np.mean(np.abs(got - want) <= 1e-6 * np.maximum(1.0, np.abs(want))) >= 0.98
            off += pl
