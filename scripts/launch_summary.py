#!/usr/bin/env python
"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import io
import json
import sys

text = open(sys.argv[1]).read()
start = text.index('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
tot = {}
cnt = {}
for r in rows:
    k = r["Kernel Name"].split("(")[0]
    tot[k] = tot.get(k, 0.0) + float(r["Metric Value"])
    cnt[k] = cnt.get(k, 0) + 1
s = sum(tot.values())
out = [{"kernel": k, "launches": cnt[k], "ms": v / 1e6, "share": v / s}
       for k, v in sorted(tot.items(), key=lambda x: -x[1])]
json.dump(out, sys.stdout, indent=1)
print()
