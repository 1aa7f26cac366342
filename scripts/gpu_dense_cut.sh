#!/bin/bash
# C4 cutoff-mode overhead lines (words / arcs at 1% and 5%) and the Alg. 1
# entity C3 line, plus the cutoff parity tests.   $1 = tag
T=${1:-dc}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -m gpu -p no:cacheprovider -x -k "cutoff or dense or c4 or scale" > gpurun_out/dense_tests_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/dense_tests_$T.log
out=gpurun_out/dense_cut_$T.jsonl
: > $out
for d in 0.01 0.05; do
  for k in words arcs; do
    timeout 600 python bench.py --workload c4 --density $d --c4-kind $k --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' >> $out
  done
done
timeout 900 python bench.py --ctx-kind entities --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' >> $out
