#!/bin/bash
# Other BASELINE configs as bench lines: C4 density sweep (word and random-arc contexts), C2, C1.
mkdir -p gpurun_out
: > gpurun_out/workloads.jsonl
for d in 0.001 0.01 0.05; do
  for k in words arcs; do
    timeout 600 python bench.py --workload c4 --density $d --c4-kind $k --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['c4']={'density':$d,'kind':'$k'}; print(json.dumps(d))" >> gpurun_out/workloads.jsonl
  done
done
timeout 600 python bench.py --workload c2 --steps 3 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/workloads.jsonl
timeout 600 python bench.py --workload c1 --steps 3 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/workloads.jsonl
