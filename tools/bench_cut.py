"""C3: LoD-cut-only sweep over 1M-100M SPT records.

Keys T/s + r with i.i.d. s (f32), key_parent sorted descending, root key the
maximum so the interval-test path runs; d swept over quantiles of key_self.
Every cut is checked bit-exact against the C oracle (cut_spt); the
compaction kernel K1 is timed with CUDA events (L2 flushed between reps by
writing a 512 MB buffer) and reported as GB/s of algorithmic bytes:
4 B/record of the key_self prefix + 16 B per selected record (rec_node read,
seg/pos/node writes) against the measured HBM peak.

    python tools/bench_cut.py [--sizes 1e6,1e7,1e8] [--spts 1,1024]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from oracle import glod_oracle as O
from paper_2507_01110_b200.device import DeviceLodScene
from paper_2507_01110_b200.hierarchy import Hierarchy
from paper_2507_01110_b200.hspt import Hspt
from paper_2507_01110_b200.spt import Spt
from paper_2507_01110_b200.core import LodConfig


def make_spts(n, S, rng):
    per = n // S
    spts = []
    for s in range(S):
        ks = (25.0 / rng.uniform(0.03, 0.3, per) + rng.uniform(0, 5, per)).astype(np.float32).astype(np.float64)
        kp = np.sort(ks)[::-1].copy()
        kp[0] = np.inf
        nodes = (s * per + rng.permutation(per)).astype(np.int64)
        ks[0] = ks.max()        # root = record 0 holds the max key: the filter path runs
        spts.append(Spt(root=int(nodes[0]), root_center=np.zeros(3), nodes=nodes, key_self=ks,
                        key_parent=kp))
    return spts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1e6,1e7,1e8")
    ap.add_argument("--spts", default="1,1024")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--check", type=int, default=1)
    args = ap.parse_args()
    peak = 6542.1
    try:
        peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        pass
    rng = np.random.default_rng(0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for n in [int(float(x)) for x in args.sizes.split(",")]:
        for S in [int(x) for x in args.spts.split(",")]:
            spts = make_spts(n, S, rng)
            cap = n
            # topology is irrelevant to the prefix cut; a flat stub of the right capacity
            stub = Hierarchy(attrs=None, parent=np.full(cap, -1, np.int32),
                             children=np.full((cap, 2), -1, np.int32), root=0)
            hs = Hspt(upper_nodes=np.zeros(0, np.int64), spts=spts,
                      passthrough_roots=np.zeros(0, np.int64), size_threshold=1.0, min_subtree=1,
                      lod=LodConfig(1.0))
            dev = DeviceLodScene(stub, hs)
            allks = np.concatenate([s.key_self for s in spts])
            ids = torch.arange(S, dtype=torch.int32, device="cuda")
            nsp = torch.tensor([S], dtype=torch.int32, device="cuda")
            for q in (0.1, 0.3, 0.5, 0.7, 0.9):
                d = float(np.quantile(allks, q))
                dist = torch.full((S,), d, dtype=torch.float64, device="cuda")
                times = []
                # the compaction captured once as a CUDA graph (its launches
                # are stream-ordered, no host syncs): replays time the
                # device work alone, L2 flushed before each
                res = dev.compact(nsp, ids, dist)
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    res = dev.compact(nsp, ids, dist)
                for r in range(args.reps + 2):
                    flush.fill_(r & 0xff)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    graph.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    if r >= 2:
                        times.append(e0.elapsed_time(e1))
                total = int(res.total[0].item())
                prefix = int(res.prefix_len[:S].sum().item())
                ok = None
                if args.check:
                    nodes = res.sel_node[:total].cpu().numpy()
                    want = []
                    for s in spts:
                        _, sel = O.cut_spt(s.key_self, s.key_parent, s.nodes, s.root, d)
                        want.append(sel)
                    ok = bool(np.array_equal(nodes, np.concatenate(want)))
                ms = float(np.median(times))
                alg = 4 * prefix + 16 * total + 48 * S
                gbs = alg / (ms * 1e-3) / 1e9
                print(json.dumps({"records": n, "spts": S, "quantile": q, "prefix": prefix,
                                  "selected": total, "ms": ms, "GB/s": gbs, "frac_of_peak": gbs / peak,
                                  "bitexact_vs_oracle": ok}), flush=True)
            del dev


if __name__ == "__main__":
    main()
