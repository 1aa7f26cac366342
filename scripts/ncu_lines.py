#!/usr/bin/env python
"""Per-source-line stall samples / instructions / L2 sectors from an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[2]
ix = {k: i for i, k in enumerate(hdr)}
recs = []
for r in rows[3:]:
    if r and r[0].isdigit():
        try:
            recs.append((int(r[0]), r[1][:90], int(r[4] or 0), int(r[ix["Instructions Executed"]] or 0),
                         int(r[ix["L2 Theoretical Sectors Global"]] or 0)))
        except (ValueError, KeyError):
            pass
ts = sum(x[2] for x in recs) or 1
ti = sum(x[3] for x in recs) or 1
tl = sum(x[4] for x in recs) or 1
print(f"samples {ts} instr {ti} l2sectors {tl}")
for x in sorted(recs, key=lambda x: -x[2])[:n]:
    print(f"{x[0]:5d} samp {100*x[2]/ts:5.1f}% inst {100*x[3]/ti:5.1f}% l2 {100*x[4]/tl:5.1f}%  {x[1]}")
