"""The train-step oracle (oracle/train_oracle.py) pinned to the reference's
own trainer.train_step traces (tests/golden/train_cases.npz): scheduled
view, every counter, the rendered node-id order, the loss, the image and
raw gradients of the first steps and the full state (params, moments, step
counts, store bytes, cache entries and blocks) at the checkpoints —
including LRU evictions, same-step re-misses of a replaced dirty entry
(trainer.py:333-341) and flushes.  CPU only."""
from __future__ import annotations

import numpy as np

from oracle import glod_oracle as O
from oracle.train_oracle import NAMES, OracleTrainer
from paper_2507_01110_b200.scheduler import build_view_graph, next_view

from .train_golden import cases


def oracle_for(tc):
    sc = tc.scene()
    h, hs = sc.read_hierarchy(), sc.read_hspt()
    flat = hs.flat_records()
    kind = np.full(h.capacity, -1, np.int32)
    kind[flat["roots"]] = np.arange(flat["roots"].size)
    kind[hs.passthrough_roots] = -2
    store = sc.host_store()
    lrs = {"means": 1.6e-4 * tc.extent, "scales": 5e-3, "rotations": 1e-3, "opacities": 5e-2,
           "base_colors": 2.5e-3, "sh_rest": 2.5e-3 / 20.0}
    params = {n: np.array(getattr(h.attrs, n), copy=True) for n in NAMES}
    orc = OracleTrainer(params, h.children, h.root, kind, flat, [s.numpy() for s in store.sections],
                        [store.spt_slot_start(i) for i in range(len(hs.spts))],
                        [(O.Cam.of(c), t) for c, t in zip(tc.cams, tc.targets)], hs.lod.threshold,
                        0 if hs.lod.metric == "max_scale" else 1, tc.budget, flush_interval=tc.flush, lrs=lrs)
    graph = build_view_graph(np.stack([c.position for c in tc.cams]), k=tc.k)
    return orc, graph


def test_train_oracle_matches_reference_trace(tmp_path):
    for ci, tc in enumerate(cases(tmp_path)):
        orc, graph = oracle_for(tc)
        rng = np.random.default_rng(tc.seed)
        view = 0
        for it in range(1, tc.steps + 1):
            want = tc.step(it)
            view = next_view(graph, view, it, rng)
            got, extra = orc.train_step(it, view)
            where = f"case {ci} step {it}"
            for k in ("view", "gaussians_rendered", "gaussians_loaded_from_store", "cache_hits", "bytes_streamed"):
                assert got[k] == want[k], (where, k, got[k], want[k])
            np.testing.assert_array_equal(extra["row_nodes"], want["rows"], err_msg=where)
            assert got["loss"] == want["loss"] or abs(got["loss"] - want["loss"]) <= 1e-13 * abs(want["loss"]), where
            if "image" in want:
                assert np.abs(extra["image"] - want["image"]).max() <= 1e-13, where
                G = np.concatenate([np.asarray(extra["grads"][n]).reshape(got["gaussians_rendered"], -1)
                                    for n in NAMES], axis=1)
                np.testing.assert_allclose(G, want["grads"], rtol=1e-9, atol=1e-14, err_msg=where)
            if it in tc.checkpoints:
                ref = tc.state(it)
                for n in NAMES:
                    np.testing.assert_allclose(orc.P[n], ref["P"][n], rtol=1e-12, atol=1e-15, err_msg=f"{where} P {n}")
                    np.testing.assert_allclose(orc.M[n], ref["M"][n], rtol=1e-9, atol=1e-18, err_msg=f"{where} M {n}")
                    np.testing.assert_allclose(orc.V[n], ref["V"][n], rtol=1e-9, atol=1e-24, err_msg=f"{where} V {n}")
                np.testing.assert_array_equal(orc.step, ref["step"], err_msg=where)
                for a, b in zip(orc.store, ref["store"]):
                    np.testing.assert_array_equal(a.reshape(-1), b, err_msg=f"{where} store")
                ents = [(sid, e[0], e[1], int(e[3])) for sid, e in orc.cache.items()]
                assert ents == ref["cache"], where
                if ents:
                    blocks = np.concatenate([np.concatenate([np.asarray(e[2][n]).reshape(e[1], -1) for n in NAMES],
                                                            axis=1) for e in orc.cache.values()])
                    np.testing.assert_allclose(blocks, ref["blocks"], rtol=1e-12, atol=1e-15, err_msg=where)


def test_train_trace_covers_the_cache_state_machine(tmp_path):
    """The fixture exercises misses, hits, dirty evictions, same-step
    re-misses of a replaced dirty entry and flushes (make_train_cases)."""
    from .conftest import golden
    d = golden("train_cases.npz")
    ev = sum(d[f"c{c}_events"] for c in range(int(d["n_cases"])))
    cnt = np.concatenate([d[f"c{c}_counters"] for c in range(int(d["n_cases"]))])
    assert (cnt[:, 2] > 0).any() and (cnt[:, 3] > 0).any() and (cnt[:, 2] == 0).any()
    assert ev[0] > 0 and ev[1] > 0 and ev[2] > 0
