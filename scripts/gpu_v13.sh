#!/bin/bash
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 1 --no-e2e --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))"; }
echo "== default : $(run)" > gpurun_out/v13.log
ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_prof.so timeout 300 python bench.py --frames 100 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-overhead > gpurun_out/prof_v13.log 2>&1
