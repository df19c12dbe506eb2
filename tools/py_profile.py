"""cProfile of the host side of the bench's train step (where the Python
time between the step's host synchronisations goes).

    python tools/py_profile.py [--leaves 10000000] [--steps 30]
"""
import argparse
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2507_01110_b200.cache import CacheConfig
from paper_2507_01110_b200.trainer import TrainConfig, Trainer


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=30)
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
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(a.steps):
        it += 1
        tr.train_step(it)
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(30)


if __name__ == "__main__":
    main()
