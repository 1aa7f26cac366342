#!/bin/bash
# C3 kernel-only bench of experiment libraries: scripts/gpu_variants.sh TAG...
mkdir -p gpurun_out
run() { timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 1 --no-e2e --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))"; }
: > gpurun_out/variants.log
for t in "$@"; do
  echo "== $t : $(ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_$t.so run)" >> gpurun_out/variants.log
done
echo "== main : $(run)" >> gpurun_out/variants.log
