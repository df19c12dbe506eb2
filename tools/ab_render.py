"""A/B of render_view options on the bench workload (C4): FPS over the
bench's frame sequence for each TrainConfig variant, alternated.

    python tools/ab_render.py [--frames 60] [--rounds 2]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2507_01110_b200.cache import CacheConfig
from paper_2507_01110_b200.trainer import TrainConfig, Trainer


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=60)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--budget-mb", type=int, default=None)
    a = ap.parse_args()
    args = bench.parse_args_for_tools()
    h, hs, cfg, cams, E, _ = bench.make_workload(args, device="cuda")
    targets = bench.synthetic_targets(len(cams), args.width, args.height, args.seed)
    budget = (a.budget_mb or args.budget_mb) << 20
    tr = Trainer(h, hs, list(zip(cams, targets)),
                 TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=budget), seed=args.seed), extent=2 * E)
    for it in range(1, 21):
        tr.train_step(it)
    nv = len(cams)
    variants = {"pipelined": True, "plain": False}
    res = {k: [] for k in variants}
    img = None
    for r in range(a.rounds):
        for name, pipe in variants.items():
            tr.cfg.pipeline_render = pipe
            for f in range(3):
                img = tr.render_view(f % nv, img, next_view=(f + 1) % nv)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            loaded = 0
            e0.record()
            for f in range(a.frames):
                img = tr.render_view((3 + f) % nv, img, next_view=(4 + f) % nv)
                loaded += tr.last_render["gaussians_loaded_from_store"]
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.frames
            res[name].append({"fps": 1e3 / ms, "loaded_mb_per_frame": loaded * 92 / a.frames / 1e6})
    print(json.dumps({"tool": "ab_render", "budget_mb": budget >> 20, "frames": a.frames, "results": res}))


if __name__ == "__main__":
    main()
