"""CPU reference timing at the bench workload (C4), without the GPU.

Times ONE real train iteration of the oracle port of the reference
(oracle/train_oracle.py: cut, store/cache gather, full 1080p render
forward, L1+SSIM, backward, ADAM — no extrapolation) on one core, and next
to it the bounded-sample estimator bench.py's `cpu_baseline` uses (uniform
random sample of the render set), so the two can be compared on the same
view.  Prints one JSON line.

    CUDA_VISIBLE_DEVICES= python tools/cpu_reference.py [--leaves N] [--view V]
"""
import argparse
import json
import os
import platform
import sys
import time
from pathlib import Path

os.environ["CUDA_VISIBLE_DEVICES"] = ""
for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "GLOD_THREADS"):
    os.environ[v] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=10_000_000)
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--sample", type=int, default=20_000)
    a = ap.parse_args()
    args = bench.parse([])
    args.leaves = a.leaves
    t0 = time.time()
    w = bench.cpu_workload(args)
    build_s = time.time() - t0
    orc = w["oracle"]
    tim = {}
    t0 = time.perf_counter()
    counters, extra = orc.train_step(1, a.view, timing=tim)
    real_s = time.perf_counter() - t0
    R = counters["gaussians_rendered"]
    est = bench.cpu_sample_estimate(w, a.view, extra_rows=None, n_sample=a.sample,
                                    n_contrib=tim["splats_backward"])
    print(json.dumps({"leaves": a.leaves, "view": a.view, "rendered": R, "build_s": build_s,
                      "real_iteration_s": real_s, "real_stages_s": tim, "estimate": est,
                      "ratio_estimate_over_real": est["seconds"] / real_s,
                      "cpu": platform.processor() or platform.machine(), "cores_used": 1}), flush=True)


if __name__ == "__main__":
    main()
