#!/bin/bash
# C1 / C2 with and without thread-block clusters (AB_CLUSTER=1 disables)
mkdir -p gpurun_out
: > gpurun_out/c12.log
for w in c1 c2; do
  for c in auto 1 2 4 8; do
    if [ "$c" = auto ]; then e=""; else e="AB_CLUSTER=$c"; fi
    env $e timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('$w cluster=$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms/step', round(d['ms_per_step'],2))" >> gpurun_out/c12.log 2>&1
  done
done
