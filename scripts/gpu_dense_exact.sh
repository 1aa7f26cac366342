#!/bin/bash
# C4 biasing overhead with and without the expansion-time cutoff (--exact:
# every candidate relaxed, the reference's work): how much of the discount's
# overhead is the biased search itself.   $1 = tag
T=${1:-dx}
mkdir -p gpurun_out
out=gpurun_out/dense_exact_$T.jsonl
: > $out
for d in 0.01 0.05; do
  for k in words arcs; do
    for x in "" "--exact"; do
      timeout 600 python bench.py --workload c4 --density $d --c4-kind $k --steps 2 --warmup 2 --no-e2e --no-cpu $x 2>/dev/null | grep '^{' >> $out
    done
  done
done
