#!/usr/bin/env python
"""Per-instruction L2 sector demand (global loads / stores / atomics) of an
ncu --set full --import-source capture, grouped by CUDA source line.

usage: python scripts/ncu_sectors.py REPORT.ncu-rep [channel_frames] [top]
Prints, per source line: L2 theoretical sectors (total and per channel-frame),
access kinds and the line text, sorted by sectors."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
cf = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[2]
ix = {k: i for i, k in enumerate(hdr)}
cur_line, cur_src = None, ""
agg = defaultdict(lambda: [0, set(), ""])
for r in rows[3:]:
    if not r:
        continue
    if r[0].isdigit():  # a CUDA source row; the SASS rows that follow belong to it
        cur_line, cur_src = int(r[0]), r[1][:100]
        continue
    try:
        sec = int(r[ix["L2 Theoretical Sectors Global"]] or 0)
    except (ValueError, IndexError):
        continue
    if sec and cur_line is not None:
        a = agg[cur_line]
        a[0] += sec
        a[1].add((r[ix["Access Operation"]] or "?") + "/" + (r[ix["Access Size"]] or "?"))
        a[2] = cur_src
tot = sum(v[0] for v in agg.values()) or 1
print(f"total L2 theoretical sectors {tot:.4g} = {tot / cf:.0f} per channel-frame")
for ln, (s, kinds, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} {100 * s / tot:5.1f}% {s / cf:9.0f}/cf  {','.join(sorted(kinds)):24s} {src}")
