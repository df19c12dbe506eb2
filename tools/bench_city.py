"""C5: city-scale out-of-core training and rendering on
one GPU — the per-GPU share of the 8×B200 configuration.

G-city scene (`scenegen.city_block_leaves`: 8×8 city blocks of varying
height separated by streets) with `--leaves` leaves (60M → 120M nodes,
11 GB f32 store in pinned host DRAM), mixed aerial orbit + street-level
views, a device cache of `--budget-mb`.  Trains `--steps` scheduled views
(one per step) and renders every view once; prints one JSON line with
iters/s, e2e iters/s, aerial and street render FPS, store traffic and the
HBM footprint.

    python tools/bench_city.py [--leaves 60000000] [--steps 30] [--budget-mb 4096]
"""
import argparse
import json
import resource
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2507_01110_b200.cache import CacheConfig
from paper_2507_01110_b200.scenegen import (SceneSpec, designed_scene, orbit_views, scene_extent,
                                            street_views)
from paper_2507_01110_b200.trainer import TrainConfig, Trainer


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=60_000_000)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=40)   # the 4 GB cache fills over ~20 steps
    ap.add_argument("--budget-mb", type=int, default=4096)
    ap.add_argument("--aerial", type=int, default=24)
    ap.add_argument("--street", type=int, default=24)
    a = ap.parse_args()
    W, H = 1920, 1080
    t0 = time.time()
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=a.leaves, spt_leaves=8192, seed=5, layout="blocks"),
                                device="cuda")
    E = scene_extent(a.leaves)
    cams = (orbit_views(a.aerial, 1.3 * E, 0.7 * E, resolution=(W, H), seed=5, jitter=0.15,
                        target_jitter=0.1 * E)
            + street_views(a.street, E, resolution=(W, H), seed=5))
    build_s = time.time() - t0
    targets = bench.synthetic_targets(len(cams), W, H, 5)
    t0 = time.time()
    tr = Trainer(h, hs, list(zip(cams, targets)),
                 TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=a.budget_mb << 20), seed=5),
                 extent=2 * E)
    setup_s = time.time() - t0
    nodes, spts, records = int(tr.scene.cap), int(tr.scene.lod.S), int(tr.scene.lod.R)
    del h
    it = 0
    for _ in range(a.warmup):
        it += 1
        tr.train_step(it)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st0 = tr.cache.stats()
    import ctypes as C
    from paper_2507_01110_b200 import _lib
    pr0 = np.zeros(8, np.int64)
    _lib.check(_lib.lib().glod_cache_debug_profile(tr.cache._h, pr0.ctypes.data_as(C.c_void_p)))
    e0.record()
    recs = []
    for _ in range(a.steps):
        it += 1
        recs.append(tr.train_step(it))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    st1 = tr.cache.stats()
    per_step = {k: (st1[k] - st0[k]) / a.steps for k in ("pf_copies", "prefetched_rows", "loaded_rows",
                                                        "host_ns_step", "host_ns_prefetch", "pool_allocs",
                                                        "grow_events")}
    pr1 = np.zeros(8, np.int64)
    _lib.check(_lib.lib().glod_cache_debug_profile(tr.cache._h, pr1.ctypes.data_as(C.c_void_p)))
    per_step["step_phase_ms"] = dict(zip(["decide", "disk", "materialize", "loads", "wb_staging"],
                                         ((pr1 - pr0)[:5] / a.steps / 1e6).round(3).tolist()))
    tr.enable_timing(True)
    for _ in range(6):
        it += 1
        tr.train_step(it)
    stage_ms = {k: float(np.mean(v)) for k, v in tr.timing.items()}
    tr.enable_timing(False)
    # e2e: targets from pinned host memory every step
    tr.targets = [t.cpu().pin_memory() for t in tr.targets]
    tr.device_targets = False
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(a.steps):
        it += 1
        tr.train_step(it)
    torch.cuda.synchronize()
    e2e = a.steps / (time.perf_counter() - t)
    fps = {}
    img = None
    for kind, idx in (("aerial", range(a.aerial)), ("street", range(a.aerial, a.aerial + a.street))):
        idx = list(idx)
        for v in idx[:2]:
            img = tr.render_view(v, img)
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        rendered, loaded = [], []
        for v in idx:
            img = tr.render_view(v, img)
            rendered.append(tr.last_render["gaussians_rendered"])
            loaded.append(tr.last_render["gaussians_loaded_from_store"])
        r1.record()
        torch.cuda.synchronize()
        fps[kind] = {"fps": len(idx) / (r0.elapsed_time(r1) / 1e3), "mean_rendered": float(np.mean(rendered)),
                     "mean_loaded_rows": float(np.mean(loaded))}
    st = tr.cache.stats()
    print(json.dumps({
        "config": "C5 (per-GPU share, 1 GPU)", "leaves": a.leaves, "nodes": nodes, "spts": spts,
        "spt_records": records, "resolution": [W, H], "views": {"aerial": a.aerial, "street": a.street},
        "cache_budget_mb": a.budget_mb, "store_gb_pinned_host": round(nodes * 92 / 1e9, 2),
        "train_iters_per_s": 1e3 / ms, "ms_per_step": ms, "e2e_iters_per_s": e2e,
        "mean_rendered": float(np.mean([r["gaussians_rendered"] for r in recs])),
        "mean_loaded_rows_per_step": float(np.mean([r["gaussians_loaded_from_store"] for r in recs])),
        "prefetched_rows": st["prefetched_rows"], "prefetch_used_rows": st["prefetch_used_rows"],
        "per_step_cache": per_step, "stage_ms": stage_ms,
        "render": fps, "hbm_peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
        "hbm_reserved_gb_incl_arenas": round((torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9, 1),
        "scene_build_s": round(build_s, 1), "setup_s": round(setup_s, 1),
        "host_peak_rss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 1),
        "data": "synthetic G-city (seeded), synthetic smooth targets"}), flush=True)


if __name__ == "__main__":
    main()
