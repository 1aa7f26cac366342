#!/bin/bash
# v6 (batched expand/relax/snapshot): correctness, then variant sweep + phase profile.
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4))"; }
: > gpurun_out/sweep_v6.log
for v in m2u4s4 m3u4s4 m4u2s2 m2u2s4 m3u2s2 m2u8s4; do
  echo "== $v : $(ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_$v.so run)" >> gpurun_out/sweep_v6.log
done
ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_prof.so timeout 300 python bench.py --frames 100 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_v6.log 2>&1
