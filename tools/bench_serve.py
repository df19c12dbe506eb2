"""Serve-path throughput: ServeSession.handle_pose over a
1080p camera path on a designed scene — device cut + diff + wire payloads
(glod_wire_pack into mapped pinned memory).  Reports poses/s, the bytes
streamed and the payload packing bandwidth.  One JSON line.

  python tools/bench_serve.py --leaves 1000000
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

from paper_2507_01110_b200 import protocol as P  # noqa: E402
from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene, orbit_views, scene_extent  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=1_000_000)
    ap.add_argument("--spt-leaves", type=int, default=2048)
    ap.add_argument("--poses", type=int, default=200)
    a = ap.parse_args()
    t0 = time.perf_counter()
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=a.leaves, spt_leaves=a.spt_leaves, seed=1), device="cuda")
    build_s = time.perf_counter() - t0
    E = scene_extent(a.leaves)
    # a smooth orbit (small steps: the delta protocol's steady state) ...
    path = orbit_views(a.poses, 1.5 * E, 0.6 * E, seed=2)
    sess = P.ServeSession(hierarchy=h, hspt=hs, lod=cfg)
    first = sess.handle_pose(path[0])          # cold: full set
    first_bytes = sum(len(m) for m in first)
    torch.cuda.synchronize()
    nbytes = 0
    loaded = 0
    t = time.perf_counter()
    for cam in path[1:]:
        msgs = sess.handle_pose(cam)
        nbytes += sum(len(m) for m in msgs)
        loaded += P.decode_message(msgs[-1])[0]["loaded"]
    dt = time.perf_counter() - t
    # ... and cold full-set poses (every SPT re-sent): packing bandwidth
    cold_s, cold_bytes = [], 0
    for cam in path[:10]:
        s2 = P.ServeSession(hierarchy=h, hspt=hs, lod=cfg)
        s2._dev = sess._dev
        t1 = time.perf_counter()
        msgs = s2.handle_pose(cam)
        cold_s.append(time.perf_counter() - t1)
        cold_bytes += sum(len(m) for m in msgs)
    n = len(path) - 1
    print(json.dumps({
        "tool": "bench_serve", "leaves": a.leaves, "nodes": int(h.capacity), "spts": len(hs.spts),
        "resolution": [1920, 1080], "poses": n, "poses_per_s": n / dt, "ms_per_pose": 1e3 * dt / n,
        "mean_bytes_per_pose": nbytes / n, "mean_loaded_per_pose": loaded / n,
        "first_pose_bytes": first_bytes,
        "cold_pose_ms": 1e3 * float(np.median(cold_s)), "cold_pose_bytes": cold_bytes / len(cold_s),
        "cold_stream_gbs": cold_bytes / sum(cold_s) / 1e9,
        "scene_build_s": build_s,
        "note": "handle_pose end to end (device cut, host diff, one glod_wire_pack launch into mapped "
                "pinned memory, message assembly in Python)"}))


if __name__ == "__main__":
    main()
