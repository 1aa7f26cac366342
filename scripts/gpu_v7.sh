#!/bin/bash
# v7 (direct token table + batched phases): correctness, then variant sweep + phase profile.
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
# timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4))"; }
: > gpurun_out/sweep_v7.log
for v in A B C D E F; do
  echo "== $v : $(ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_$v.so run)" >> gpurun_out/sweep_v7.log
done
