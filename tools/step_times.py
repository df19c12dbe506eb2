"""Per-step device time (CUDA events, synchronised per step) and cache
counters for the bench workload — where the steady state starts and which
steps are slow.

    python tools/step_times.py [--steps 80] [--leaves 10000000]
"""
import argparse
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
    ap.add_argument("--steps", type=int, default=80)
    ap.add_argument("--no-prefetch", action="store_true")
    a = ap.parse_args()
    args = bench.parse_args_for_tools(leaves=a.leaves)
    h, hs, cfg, cams, E, _ = bench.make_workload(args, device="cuda")
    targets = bench.synthetic_targets(len(cams), args.width, args.height, args.seed)
    tr = Trainer(h, hs, list(zip(cams, targets)),
                 TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=args.budget_mb << 20),
                             seed=args.seed, prefetch=not a.no_prefetch), extent=2 * E)
    used0 = 0
    for it in range(1, a.steps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = tr.train_step(it)
        e1.record()
        torch.cuda.synchronize()
        st = tr.cache.stats()
        print(f"it {it:3d} view {r['view']:2d} ms {e0.elapsed_time(e1):7.2f} rendered {r['gaussians_rendered']:8d} "
              f"loaded {r['gaussians_loaded_from_store']:8d} pf_used {st['prefetch_used_rows'] - used0:8d} "
              f"hits {r['cache_hits']:4d} inst {tr.last_stats.get('n_instances', 0):9d}", flush=True)
        used0 = st["prefetch_used_rows"]


if __name__ == "__main__":
    main()
