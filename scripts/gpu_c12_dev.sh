#!/bin/bash
# C1 / C2 development loop: cluster parity tests, C1 / C2 bench lines, and
# the phase profile (libarcboost_b200_prof.so, AB_PROFILE clock64 per phase of
# the leader CTA) of both.   $1 = tag
T=${1:-dev}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "cluster or small or c2 or switch" > gpurun_out/c12dev_tests_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c12dev_tests_$T.log
: > gpurun_out/c12dev_$T.log
for w in c1 c2; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('$w', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms/step', round(d['ms_per_step'],2))" >> gpurun_out/c12dev_$T.log 2>&1
  ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_prof.so timeout 600 python bench.py --workload $w --steps 1 --warmup 1 --no-cpu --no-overhead --no-e2e 2>&1 | grep AB_PROFILE | tail -2 >> gpurun_out/c12dev_$T.log
done
