#!/bin/bash
# Experiment builds: libraries with different batching / occupancy macros.
# usage: scripts/build_variants.sh "tag:-DFLAGS ..." ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  tag="${spec%%:*}"; flags="${spec#*:}"
  python - "$tag" $flags -DAB_BENCH_ONLY -diag-suppress 177,550 <<'PY'
import sys
from pathlib import Path
import __graft_entry__ as g
tag, flags = sys.argv[1], tuple(sys.argv[2:])
g.build_lib(g.PKG / f"libarcboost_b200_{tag}.so", flags, tag)
PY
done
