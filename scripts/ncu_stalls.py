#!/usr/bin/env python
"""Warp-stall samples of an ncu --set full --import-source capture, grouped by
CUDA source line (where the kernel's time goes).

usage: python scripts/ncu_stalls.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[2]
ix = {k: i for i, k in enumerate(hdr)}
col = next(k for k in hdr if k.startswith("Warp Stall Sampling (All"))
cur_line, cur_src = None, ""
agg = defaultdict(lambda: [0.0, ""])
for r in rows[3:]:
    if not r:
        continue
    if r[0].isdigit():
        cur_line, cur_src = int(r[0]), r[1][:110]
        continue
    try:
        v = float(r[ix[col]] or 0)
    except (ValueError, IndexError):
        continue
    if v and cur_line is not None:
        agg[cur_line][0] += v
        agg[cur_line][1] = cur_src
tot = sum(v[0] for v in agg.values()) or 1
print(f"total warp-stall samples {tot:.0f}")
for ln, (v, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} {100 * v / tot:5.1f}%  {src}")
