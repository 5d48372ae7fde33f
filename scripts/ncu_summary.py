#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (markdown + JSON).

    python scripts/ncu_summary.py --rep gpurun_out/prof_r1.ncu-rep --launches gpurun_out/launches_r1.csv \
        --tag r1 --config small --frames 4096 --N 128

* --rep: a `ncu --set full` report; per kernel: duration, DRAM bytes, throughput, occupancy, IPC,
  pipe utilisation, registers, shared memory, bank conflicts.
* --launches: a `ncu --metrics gpu__time_duration.sum --csv` launch list; per kernel name: count,
  total / mean device time and share of the listed time (cold-cache, serialised: compare SHARES).
Writes profiles/<tag>_ncu.md and merges DRAM bytes per launch into profiles/ncu_traffic.json
(keyed by config, then kernel) for bench.py's roofline "traffic" field.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RAW = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pct",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block_dynamic": "smem_dyn",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_conflicts",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}


def raw_rows(rep):
    # a .csv is a saved `ncu -i <rep> --page raw --csv` export (reports too large to bring back)
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for i, h in enumerate(hdr):
            if h in RAW:
                d[RAW[h]] = (r[i], units[i])
        res.append(d)
    return res


def to_bytes(v):
    val, unit = v
    val = float(val.replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return val * mult


def to_seconds(v):
    val, unit = v
    val = float(val.replace(",", ""))
    return val * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
                  "second": 1.0, "s": 1.0}.get(unit, 1e-9)


def short(name):
    return name.split("(")[0].replace("void ", "").replace("pty::", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="small")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--N", type=int, default=128)
    args = ap.parse_args()
    md = [f"# ncu summary {args.tag} (config {args.config})", ""]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    if args.rep:
        md += [f"`ncu --set full --clock-control none` capture: `{os.path.basename(args.rep)}`", "",
               "| kernel | dur us | DRAM R MB | DRAM W MB | DRAM % | B/px | occ % | IPC | FMA % | ALU % | XU % | regs | smem KB | bank confl |",
               "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        px = args.frames * args.N * args.N
        for d in raw_rows(args.rep):
            nm = short(d["kernel"])
            dur = to_seconds(d["duration"]) * 1e6 if "duration" in d else float("nan")
            rd = to_bytes(d["dram_read"]) if "dram_read" in d else 0.0
            wr = to_bytes(d["dram_write"]) if "dram_write" in d else 0.0
            bpx = (rd + wr) / px if px else float("nan")
            g = lambda k: d[k][0] if k in d else "-"
            md.append(f"| {nm} | {dur:.1f} | {rd/1e6:.1f} | {wr/1e6:.1f} | {g('dram_pct')} | {bpx:.1f} | "
                      f"{g('occupancy_pct')} | {g('ipc')} | {g('fma_pct')} | {g('alu_pct')} | {g('xu_pct')} | "
                      f"{g('regs')} | {float(g('smem_dyn'))/1024 if g('smem_dyn') != '-' else 0:.1f} | {g('smem_conflicts')} |")
            key = nm.split("<")[0]
            traffic.setdefault(args.config, {})[key] = {"dram_bytes_per_launch": rd + wr, "dram_bytes_per_px": bpx,
                                                      "tag": args.tag}
        md.append("")
    if args.launches:
        rows = [r for r in csv.reader(open(args.launches)) if len(r) > 5]
        hdr = rows[0]
        ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        ui = hdr.index("Metric Unit")
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows[1:]:
            if r[mi] != "gpu__time_duration.sum":
                continue
            t = to_seconds((r[vi], r[ui]))
            agg[short(r[ki])][0] += 1
            agg[short(r[ki])][1] += t
        tot = sum(v[1] for v in agg.values())
        md += [f"Launch list `{os.path.basename(args.launches)}` (`--metrics gpu__time_duration.sum`, serialised,"
               " cold-cache: compare shares)", "",
               "| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| {k} | {n} | {t*1e3:.3f} | {t/n*1e6:.1f} | {t/tot*100:.1f}% |")
        md.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{args.tag}_ncu.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
