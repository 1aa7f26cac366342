#!/bin/bash
# Other BASELINE configs as bench lines (config.workload names density / kind):
# C3 with Alg. 1 multi-word contexts (LIST), C4 density sweep (word and
# random-arc contexts), C2, C1.   $1 = tag
T=${1:-wl}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
out=gpurun_out/workloads_$T.jsonl
: > $out
timeout 900 python bench.py --ctx-kind entities --steps 2 --warmup 2 --no-e2e --cpu-seconds 3 2>gpurun_out/wl_entities_$T.err | grep '^{' >> $out
for d in 0.001 0.01 0.05; do
  for k in words arcs; do
    timeout 600 python bench.py --workload c4 --density $d --c4-kind $k --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' >> $out
  done
done
timeout 600 python bench.py --workload c2 --steps 3 --warmup 3 2>/dev/null | grep '^{' >> $out
timeout 600 python bench.py --workload c1 --steps 3 --warmup 3 2>/dev/null | grep '^{' >> $out
