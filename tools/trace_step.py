"""GPU timeline of a few train steps (torch.profiler / CUPTI): per-kernel
device intervals on every stream, the idle gaps of the main stream and the
host-side ranges around them.  Prints a summary and writes the chrome trace.

    python tools/trace_step.py [--leaves 10000000] [--steps 3] [--out gpurun_out/trace.json]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2507_01110_b200.cache import CacheConfig
from paper_2507_01110_b200.trainer import TrainConfig, Trainer


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leaves", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/trace.json")
    ap.add_argument("--render", action="store_true", help="trace render_view frames (next view known)")
    a = ap.parse_args()
    args = bench.parse_args_for_tools(leaves=a.leaves)
    h, hs, cfg, cams, E, _ = bench.make_workload(args, device="cuda")
    targets = bench.synthetic_targets(len(cams), args.width, args.height, args.seed)
    tr = Trainer(h, hs, list(zip(cams, targets)),
                 TrainConfig(lod=cfg, cache=CacheConfig(budget_bytes=args.budget_mb << 20),
                             seed=args.seed), extent=2 * E)
    it = 0
    for _ in range(a.warmup):
        it += 1
        tr.train_step(it)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
    nv = len(cams)
    if a.render:
        for f in range(3):
            tr.render_view(f % nv, next_view=(f + 1) % nv)
    with torch.profiler.profile(activities=acts) as prof:
        for f in range(a.steps):
            it += 1
            with torch.profiler.record_function(f"step{it}"):
                if a.render:
                    tr.render_view((3 + f) % nv, next_view=(4 + f) % nv)
                else:
                    tr.train_step(it)
        torch.cuda.synchronize()
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    prof.export_chrome_trace(a.out)
    ev = json.load(open(a.out))["traceEvents"]
    kern = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    steps = sorted([e for e in ev if e.get("name", "").startswith("step") and e.get("ph") == "X"],
                   key=lambda e: e["ts"])
    streams = {}
    for k in kern:
        streams.setdefault(k["args"].get("stream", k.get("tid")), []).append(k)
    main_sid = max(streams, key=lambda s: sum(k["dur"] for k in streams[s]))
    mk = sorted(streams[main_sid], key=lambda k: k["ts"])
    busy = {s: sum(k["dur"] for k in v) for s, v in streams.items()}
    print("streams busy us:", {str(s): round(v, 1) for s, v in busy.items()})
    t0, t1 = mk[0]["ts"], mk[-1]["ts"] + mk[-1]["dur"]
    print(f"main stream span {t1 - t0:.0f} us over {a.steps} steps, busy {busy[main_sid]:.0f} us")
    def short(n):
        n = n.replace("(anonymous namespace)::", "").replace("glod::", "").replace("void ", "")
        return n.split("(")[0][-48:]
    gaps = []
    others = [k for sid, v in streams.items() if sid != main_sid for k in v]
    for p, q in zip(mk[:-1], mk[1:]):
        g = q["ts"] - (p["ts"] + p["dur"])
        if g > 5:
            gaps.append((g, short(p["name"]), short(q["name"])))
        if g > 150:
            # what ran on the other streams during the gap
            t_a, t_b = p["ts"] + p["dur"], q["ts"]
            ov = [k for k in others if k["ts"] < t_b and k["ts"] + k["dur"] > t_a]
            by = {}
            for k in ov:
                key = (k["args"].get("stream"), k["name"][:24])
                b = by.setdefault(key, [0, 0.0, 0])
                b[0] += 1
                b[1] += min(k["ts"] + k["dur"], t_b) - max(k["ts"], t_a)
                b[2] += k["args"].get("bytes", 0) or 0
            last_end = max([k["ts"] + k["dur"] for k in ov if k["ts"] + k["dur"] <= t_b + 2] or [0])
            print(f"gap {g:.0f} us before {short(q['name'])}: other streams "
                  + "; ".join(f"s{s_} {n} x{c} {t:.0f}us {b / 1e6:.1f}MB" for (s_, n), (c, t, b) in by.items())
                  + f"; last other op ended {t_b - last_end:.0f} us before the gap end")
    agg = {}
    for g, p, q in gaps:
        key = (p.split("(")[0][-40:], q.split("(")[0][-40:])
        agg.setdefault(key, [0, 0.0])
        agg[key][0] += 1
        agg[key][1] += g
    print(f"idle gaps >5us on main stream: total {sum(g for g, _, _ in gaps):.0f} us")
    for (p, q), (n, tot) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"  {tot / a.steps:8.1f} us/step  x{n:3d}  after {p}  ->  before {q}")
    # per-stream activity relative to each step's first main-stream kernel
    firsts = []
    for st_ev in steps:
        ks = [k for k in mk if st_ev["ts"] <= k["ts"] <= st_ev["ts"] + st_ev["dur"] + 20000]
        if ks:
            firsts.append(ks[0]["ts"])
    for s_id, v in streams.items():
        v = sorted(v, key=lambda k: k["ts"])
        cats = {}
        for k in v:
            cats[k.get("cat")] = cats.get(k.get("cat"), 0) + 1
        print(f"stream {s_id}: {len(v)} ops {cats}")
        if s_id == main_sid:
            continue
        for f in firsts:
            w = [k for k in v if f - 8000 <= k["ts"] < f + 8000]
            if w:
                print(f"   rel. step start {f:.0f}: first {w[0]['ts'] - f:+.0f} us, last end "
                      f"{max(k['ts'] + k['dur'] for k in w) - f:+.0f} us, busy {sum(k['dur'] for k in w):.0f} us, "
                      f"n={len(w)}")
    kagg = {}
    for k in mk:
        n = k["name"].split("(")[0][-45:]
        kagg[n] = kagg.get(n, 0) + k["dur"]
    print("main stream kernels (us/step):")
    for n, d in sorted(kagg.items(), key=lambda x: -x[1])[:25]:
        print(f"  {d / a.steps:8.1f}  {n}")


if __name__ == "__main__":
    main()
