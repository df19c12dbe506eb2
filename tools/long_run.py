"""Long training run on the bench scene generator (1M leaves by default) through the
reference's loop, `Trainer.train` (trainer.py:446-458): every iteration a
scheduled view, densification every `--densify-interval` iterations (host
tree surgery + device HSPT rebuild + store/record re-layout).  Prints one
JSON line: loss curve (window means), throughput per window, densify cost,
scene growth, and the check that every loss stayed finite.

    python tools/long_run.py [--iters 3000] [--densify-interval 1000] [--leaves 1000000]
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
from paper_2507_01110_b200.trainer import TrainConfig, Trainer


class Sink:
    """metrics_out for Trainer.train: wall time per record."""

    def __init__(self):
        self.t = []
        self.recs = []

    def write(self, line):
        self.t.append(time.perf_counter())
        self.recs.append(json.loads(line))
        n = len(self.recs)
        if n % 250 == 0 or "spawned" in self.recs[-1]:
            print(f"[long_run] it {n}: loss {self.recs[-1]['loss']:.5f} "
                  f"t {self.t[-1] - self.t0:.1f}s {'densify' if 'spawned' in self.recs[-1] else ''}",
                  file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=1_000_000)
    ap.add_argument("--iters", type=int, default=3000)
    ap.add_argument("--densify-interval", type=int, default=1000)
    ap.add_argument("--window", type=int, default=250)
    a = ap.parse_args()
    args = bench.parse_args_for_tools(leaves=a.leaves)
    h, hs, cfg, cams, E, _ = bench.make_workload(args, device="cuda")
    targets = bench.synthetic_targets(len(cams), args.width, args.height, args.seed)
    leaves0 = int(h.leaf_count)
    tr = Trainer(h, hs, list(zip(cams, targets)),
                 TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=args.budget_mb << 20), seed=args.seed,
                             total_iterations=a.iters, densify_interval=a.densify_interval),
                 extent=2 * E)
    del h
    sink = Sink()
    t0 = time.perf_counter()
    sink.t0 = t0
    tr.train(metrics_out=sink)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    recs = sink.recs
    losses = np.array([r["loss"] for r in recs])
    ts = np.array(sink.t)
    dens = [i for i, r in enumerate(recs) if "respawned" in r or "spawned" in r or "densify_s" in r]
    windows = []
    for w0 in range(0, len(recs), a.window):
        w1 = min(len(recs), w0 + a.window)
        dt = ts[w1 - 1] - (ts[w0 - 1] if w0 > 0 else t0)
        windows.append({"iters": [w0 + 1, w1], "mean_loss": float(losses[w0:w1].mean()),
                        "iters_per_s_wall": (w1 - w0) / dt,
                        "mean_rendered": float(np.mean([r["gaussians_rendered"] for r in recs[w0:w1]]))})
    print(json.dumps({
        "tool": "long_run", "workload": f"bench scene generator, {a.leaves} leaves, 1080p, 32 views",
        "iterations": len(recs), "densify_interval": a.densify_interval, "wall_s": wall,
        "all_losses_finite": bool(np.all(np.isfinite(losses))),
        "loss_first_window": windows[0]["mean_loss"], "loss_last_window": windows[-1]["mean_loss"],
        "leaves_start": leaves0, "leaves_end": int(tr.hierarchy.leaf_count),
        "densify_records": [{k: v for k, v in recs[i].items() if k not in ("loss",)} for i in dens],
        "windows": windows,
        "note": "Trainer.train (the reference's loop) with densification; wall-clock windows include the "
                "densify iterations; synthetic smooth targets"}))


if __name__ == "__main__":
    main()
