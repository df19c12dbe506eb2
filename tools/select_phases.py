"""Phase times of the LoD select kernel (K2) on the bench workload, from the
kernel's own %globaltimer stamps (glod_debug_select_phases).

    python tools/select_phases.py [--leaves 10000000] [--views 8]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2507_01110_b200 import _lib
from paper_2507_01110_b200.device import DeviceLodScene

NAMES = ["flags", "upper walks", "pass walks", "bitmap counts", "id lists", "d_root+prefix"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=10_000_000)
    ap.add_argument("--views", type=int, default=8)
    a = ap.parse_args()
    args = bench.parse_args_for_tools(leaves=a.leaves)
    h, hs, cfg, cams, E, _ = bench.make_workload(args, device="cuda")
    lod = DeviceLodScene(h, hs)
    print("candidates", lod.num_cand, "upper", lod.num_cand_upper, "spts", lod.S, "grid", _lib.lib().glod_lod_select_grid() if hasattr(_lib.lib(), "glod_lod_select_grid") else "?")
    rows = []
    for rep in range(3):
        for cam in cams[:a.views]:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sel = lod.select(cam, cfg, cull=True)
            e1.record()
            torch.cuda.synchronize()
            t = np.zeros(7, np.int64)
            _lib.check(_lib.lib().glod_debug_select_phases(t.ctypes.data_as(C.c_void_p)))
            if rep:
                rows.append(np.concatenate([[e0.elapsed_time(e1) * 1e3], np.diff(t) / 1e3]))
    r = np.mean(rows, axis=0)
    print(f"select launch (events, incl. memset): {r[0]:.1f} us")
    for n, v in zip(NAMES, r[1:]):
        print(f"  {n:14s} {v:7.1f} us")


if __name__ == "__main__":
    main()
