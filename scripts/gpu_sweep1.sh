#!/bin/bash
# Launch-shape / L2-fetch sweep on C3 (100 frames, 1 segment).
mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4))"; }
: > gpurun_out/sweep1.log
for cfg in "X=0" "AB_L2FETCH=32" "AB_L2FETCH=128" "AB_GRID=296" "AB_GRID=148" "AB_BLOCK=512" "AB_BLOCK=512 AB_L2FETCH=32" "AB_BLOCK=512 AB_GRID=148" "AB_BLOCK=128"; do
  echo "== $cfg : $(run $cfg)" >> gpurun_out/sweep1.log
done
