"""Host-side cost of the train step's synchronous phases (bench workload):
wall time of the calls the host makes between its synchronisations, so the
GPU-idle share of the select → cache → compact chain can be attributed.

    python tools/host_profile.py [--leaves 10000000] [--steps 20]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2507_01110_b200 import _lib
from paper_2507_01110_b200.cache import CacheConfig
from paper_2507_01110_b200.trainer import TrainConfig, Trainer

T = {}


def wrap(obj, name, key=None):
    f = getattr(obj, name)
    key = key or name

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        T.setdefault(key, []).append(time.perf_counter() - t)
        return r
    setattr(obj, name, g)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    args = bench.parse_args_for_tools(leaves=a.leaves)
    h, hs, cfg, cams, E, _ = bench.make_workload(args, device="cuda")
    targets = bench.synthetic_targets(len(cams), args.width, args.height, args.seed)
    tr = Trainer(h, hs, list(zip(cams, targets)),
                 TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=args.budget_mb << 20), seed=args.seed),
                 extent=2 * E)
    it = 0
    for _ in range(10):
        it += 1
        tr.train_step(it)
    torch.cuda.synchronize()
    wrap(tr, "select")
    wrap(tr.cache, "step", "cache.step")
    wrap(tr.cache, "prefetch", "cache.prefetch")
    wrap(tr.cache, "end_step", "cache.end_step")
    wrap(tr.scene.lod, "compact", "lod.compact")
    wrap(_lib, "upload")
    wrap(tr.rast, "forward", "rast.forward")
    wrap(tr.rast, "backward", "rast.backward")
    wrap(tr.rast, "loss", "rast.loss")
    wrap(tr, "_gather_view")
    wrap(tr, "train_step")
    s0 = tr.cache.stats()
    for _ in range(a.steps):
        it += 1
        tr.train_step(it)
    torch.cuda.synchronize()
    s1 = tr.cache.stats()
    print(f"C++ cache_step {(s1['host_ns_step'] - s0['host_ns_step']) / a.steps / 1e6:.3f} ms/step, "
          f"cache_prefetch {(s1['host_ns_prefetch'] - s0['host_ns_prefetch']) / a.steps / 1e6:.3f} ms/step")
    for k, v in sorted(T.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:18s} calls/step {len(v) / a.steps:4.1f}  mean {1e3 * np.mean(v):7.3f} ms  "
              f"per step {1e3 * sum(v) / a.steps:7.3f} ms")


if __name__ == "__main__":
    main()
