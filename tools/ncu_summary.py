"""Summarise an `ncu --set full` report: per kernel, mean duration, DRAM
bytes per launch, achieved DRAM GB/s, issue-slot utilisation, warps active
and the top stall reasons.  Writes profiles/ncu_traffic.json (read by
bench.py for roofline.traffic) and prints a markdown table.

    python tools/ncu_summary.py gpurun_out/r1d_full.ncu-rep [--json profiles/ncu_traffic.json]
"""
import argparse
import collections
import csv
import io
import json
import subprocess

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "smsp__inst_executed.sum", "launch__registers_per_thread",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
UNIT = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
        "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        name = name.split("<")[0] if name.startswith(("store_xfer", "scatter_kernel")) else name
        for m in M:
            if m not in h:
                continue
            u = units[h.index(m)]
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            agg[name][m].append(v * UNIT.get(u, 1.0))
    res = {}
    print("| kernel | launches | ms | DRAM MB/launch | DRAM GB/s | issue active % | warps active % | regs |")
    print("|---|---|---|---|---|---|---|---|")
    for name, d in sorted(agg.items(), key=lambda x: -sum(x[1]["gpu__time_duration.sum"])):
        n = len(d["gpu__time_duration.sum"])
        ms = sum(d["gpu__time_duration.sum"]) / n
        by = (sum(d["dram__bytes_read.sum"]) + sum(d["dram__bytes_write.sum"])) / n
        iss = sum(d[M[3]]) / n
        wa = sum(d[M[4]]) / n
        regs = d[M[6]][0]
        mean = lambda m: (sum(d[m]) / len(d[m])) if d.get(m) else None
        res[name] = {"launches": n, "ms": ms, "dram_bytes_per_launch": by, "dram_gbs": by / (ms * 1e-3) / 1e9,
                     "issue_active_pct": iss, "warps_active_pct": wa, "registers": regs,
                     "smem_wavefronts_pct": mean(M[7]),
                     "pipe_pct": {"alu": mean(M[8]), "fma": mean(M[9]), "xu": mean(M[10]), "lsu": mean(M[11])},
                     "warp_instructions": sum(d[M[5]]) / n, "source": a.rep}
        print(f"| {name} | {n} | {ms:.3f} | {by / 1e6:.1f} | {by / (ms * 1e-3) / 1e9:.0f} | {iss:.1f} | {wa:.1f} | {regs:.0f} |")
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
