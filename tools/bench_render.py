"""C2: single-GPU LoD cut + forward render at 1080p of a 1M-leaf scene,
fully device-resident (`cli.cmd_render`-style serve path).

The f32 store itself lives in HBM (`store_location="device"`) and the cache
budget holds every SPT record, so nothing crosses PCIe: a cache miss (the
reference's distance-band rule, cache.py:56-73, still decides hits) is a
device-to-device prefix load.  Two scene shapes: G-spt (the designed
scene, SPT cuts) and G-leaf (every cut branch a passthrough subtree, so the
BFS selects leaves).  Timed with CUDA events over all frames; prints one
JSON line per shape.

    python tools/bench_render.py [--leaves 1000000] [--frames 64]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2507_01110_b200.cache import CacheConfig
from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene, orbit_views, scene_extent
from paper_2507_01110_b200.trainer import TrainConfig, Trainer


def run(shape, leaves, frames, views, w, h):
    spec = SceneSpec(n_leaves=leaves, seed=1, pass_fraction=1.0 if shape == "G-leaf" else 0.05,
                     spt_leaves=4096)
    t0 = time.time()
    hier, hs, cfg = designed_scene(spec, device="cuda")
    E = scene_extent(leaves)
    cams = orbit_views(views, 1.3 * E, 0.7 * E, resolution=(w, h), seed=1, jitter=0.15,
                       target_jitter=0.1 * E)
    build_s = time.time() - t0
    records = int(hs.flat_records()["nodes"].size) if hs.spts else 0
    budget = max(records * 92 * 2, 1 << 20)           # whole scene resident
    targets = [np.zeros((h, w, 3), np.float32)] * len(cams)
    tr = Trainer(hier, hs, list(zip(cams, targets)),
                 TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=budget), store_location="device"),
                 extent=2 * E)
    img = None
    for v in range(len(cams)):                         # warm-up: every view's prefixes resident
        img = tr.render_view(v, img)
    torch.cuda.synchronize()
    loaded = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for f in range(frames):
        img = tr.render_view(f % len(cams), img)
        loaded.append(tr.last_render["gaussians_loaded_from_store"])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / frames
    tr.enable_timing(True)
    for f in range(min(frames, 8)):
        tr.render_view(f % len(cams), img)
    stage = {k: float(np.mean(v)) for k, v in tr.timing.items()}
    return {"config": "C2", "shape": shape, "leaves": leaves, "resolution": [w, h], "views": views,
            "frames": frames, "render_fps": 1e3 / ms, "ms_per_frame": ms,
            "mean_rendered": tr.last_render["gaussians_rendered"],
            "n_instances": tr.rast.stats()["n_instances"], "spt_records": records,
            "cache_budget_mb": budget >> 20, "store": "HBM (device-resident)",
            "mean_loaded_rows_per_frame": float(np.mean(loaded)),
            "stage_ms": stage, "scene_build_s": round(build_s, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=1_000_000)
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--views", type=int, default=16)
    a = ap.parse_args()
    for shape in ("G-spt", "G-leaf"):
        print(json.dumps(run(shape, a.leaves, a.frames, a.views, 1920, 1080)), flush=True)


if __name__ == "__main__":
    main()
