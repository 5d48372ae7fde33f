#!/usr/bin/env python
"""Per-source-line warp-stall attribution of one kernel in an ncu report (needs -lineinfo and
--import-source on).  Prints the top lines by stall samples with their dominant stall reasons,
and the whole-kernel stall mix.

    python scripts/ncu_lines.py gpurun_out/prof_ls_r2a.ncu-rep [--top 40]
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()
if a.rep.endswith(".csv"):   # a saved `ncu -i <rep> --page source --csv --print-source cuda,sass` export
    out = open(a.rep).read()
else:
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
fname = "?"
cur = None
lines = {}
tot = defaultdict(float)
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0].isdigit():            # a CUDA source line: the SASS rows below it belong to it
        cur = (fname, int(r[0]))
        lines.setdefault(cur, [0.0, 0.0, r[1][:90], defaultdict(float)])
        continue
    if cur is None or len(r) < 4 or not r[2].startswith("0x"):
        continue
    d = dict(zip(hdr, r))         # SASS row: columns aligned with the header

    def f(k):
        try:
            return float(d.get(k, "0"))
        except ValueError:
            return 0.0
    e = lines[cur]
    e[0] += f("Warp Stall Sampling (All Samples)")
    e[1] += f("Instructions Executed")
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            e[3][k[6:]] += f(k)
            tot[k[6:]] += f(k)
S = sum(v[0] for v in lines.values())
I = sum(v[1] for v in lines.values())
print(f"total stall samples {S:.0f}, warp instructions {I:.3g}")
print("mix:", ", ".join(f"{k} {100*v/S:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]))
for (fn, ln), (s, ins, src, rs) in sorted(lines.items(), key=lambda x: -x[1][0])[:a.top]:
    top = ", ".join(f"{k} {100*v/max(s,1):.0f}%" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:3] if v > 0)
    print(f"{100*s/S:5.1f}% {ins/1e6:7.2f}M {fn}:{ln:<4d} {src.strip()[:70]:70s} | {top}")
