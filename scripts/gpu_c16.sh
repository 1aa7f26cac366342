#!/bin/bash
# C1 with 8- and 16-CTA clusters (16 = non-portable size), and cluster-size parity.  $1 = tag
T=${1:-c16}
mkdir -p gpurun_out
: > gpurun_out/c16_$T.log
for c in 8 16 8 16; do
  AB_CLUSTER=$c timeout 600 python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('c1 cluster=$c', round(d['value']), 'e2e', round(d['e2e']['value']))" >> gpurun_out/c16_$T.log 2>&1
done
AB_CLUSTER=16 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "small_cases or c1_full" >> gpurun_out/c16_$T.log 2>&1; echo "pytest16 rc=$?" >> gpurun_out/c16_$T.log
