"""Loader for tests/golden/train_cases.npz — traces of the reference's own
trainer.train_step (trainer.py:312-378), minted by
tests/golden/make_golden.py:make_train_cases — shared by the CPU oracle test
(test_train_golden.py) and the GPU tests (test_train_golden_gpu.py)."""
from __future__ import annotations

import numpy as np

from paper_2507_01110_b200 import scenefile as SF
from paper_2507_01110_b200.core import SECTIONS, Camera

from .conftest import golden

NAMES = [n for n, _ in SECTIONS]
COUNTER_KEYS = ("view", "gaussians_rendered", "gaussians_loaded_from_store", "cache_hits", "bytes_streamed")


class TrainCase:
    def __init__(self, d, c, tmp_path):
        p = f"c{c}_"
        self.d = {k[len(p):]: d[k] for k in d.files if k.startswith(p)}
        g = self.d
        self.path = tmp_path / f"train{c}.glod"
        self.path.write_bytes(g["file"].tobytes())
        self.n_views = int(g["n_views"])
        self.cams = [Camera(position=g[f"cam{v}_position"], orientation=g[f"cam{v}_orientation"],
                            focal=tuple(g[f"cam{v}_focal"]), principal_point=tuple(g[f"cam{v}_pp"]),
                            resolution=tuple(int(x) for x in g[f"cam{v}_res"]), near=float(g[f"cam{v}_near"]),
                            far=float(g[f"cam{v}_far"]))
                     for v in range(self.n_views)]
        self.targets = [t.astype(np.float64) for t in g["targets"]]
        self.budget, self.flush = int(g["budget"]), int(g["flush"])
        self.k, self.seed = int(g["k"]), int(g["seed"])
        self.extent, self.steps = float(g["extent"]), int(g["steps"])
        self.counters = g["counters"]
        self.checkpoints = [int(x) for x in g["checkpoints"]]

    def scene(self):
        return SF.open_scene(self.path)

    def step(self, it):
        g, q = self.d, f"it{it}_"
        out = dict(zip(COUNTER_KEYS, (int(x) for x in self.counters[it - 1])))
        out["iteration"] = it
        out["loss"] = float(g[q + "loss"])
        out["rows"] = g[q + "rows"].astype(np.int64)
        for k in ("image", "grads"):
            if q + k in g:
                out[k] = g[q + k]
        return out

    def state(self, it):
        """Reference state after step `it` (a checkpoint)."""
        g, q = self.d, f"it{it}_"
        return {"P": {n: g[q + "p_" + n] for n in NAMES}, "M": {n: g[q + "m_" + n] for n in NAMES},
                "V": {n: g[q + "v_" + n] for n in NAMES}, "step": g[q + "step"],
                "store": [g[q + "store_" + n] for n in NAMES],
                "cache": list(zip(g[q + "cache_sid"].tolist(), g[q + "cache_dist"].tolist(),
                                  g[q + "cache_prefix"].tolist(), g[q + "cache_dirty"].tolist())),
                "blocks": g[q + "cache_blocks"]}


def cases(tmp_path):
    d = golden("train_cases.npz")
    return [TrainCase(d, c, tmp_path) for c in range(int(d["n_cases"]))]
