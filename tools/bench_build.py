"""HSPT/SPT build timing: the device build K12 against
the numpy restatement on the same hierarchy, with a record-for-record
equality check.  One JSON line.

  python tools/bench_build.py --leaves 10000000
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2507_01110_b200 import hspt as H  # noqa: E402
from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=10_000_000)
    ap.add_argument("--spt-leaves", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-host", action="store_true")
    a = ap.parse_args()
    t0 = time.perf_counter()
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=a.leaves, spt_leaves=a.spt_leaves, seed=1, relabel=False),
                                device="cuda")
    scene_s = time.perf_counter() - t0
    args = (h, hs.size_threshold, hs.min_subtree, cfg)
    H.build_hspt(*args)                      # warm-up (module load, pool)
    dev_s = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        got = H.build_hspt(*args)
        dev_s.append(time.perf_counter() - t)
    line = {"tool": "bench_build", "leaves": a.leaves, "nodes": int(h.capacity), "spts": len(got.spts),
            "records": int(got.flat["nodes"].size), "upper": int(got.upper_nodes.size),
            "passthrough": int(got.passthrough_roots.size),
            "device_s": min(dev_s), "device_s_all": dev_s, "scene_build_s": scene_s,
            "note": "device_s includes the H2D upload of parent/children/means/scales and the D2H of the "
                    "records (build_hspt end to end, host arrays in and out)"}
    if not a.no_host:
        t = time.perf_counter()
        want = H.build_hspt_host(*args)
        line["host_numpy_s"] = time.perf_counter() - t
        line["host_cores"] = 1
        ok = (np.array_equal(got.upper_nodes, want.upper_nodes)
              and np.array_equal(got.passthrough_roots, want.passthrough_roots))
        for k in ("nodes", "key_self", "key_parent", "offset", "count", "roots"):
            x, y = np.asarray(got.flat[k]), np.asarray(want.flat[k])
            ok = ok and x.shape == y.shape and np.array_equal(x.view(np.uint8), y.astype(x.dtype).view(np.uint8))
        line["bitexact_vs_host"] = bool(ok)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
