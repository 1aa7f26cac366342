#!/bin/bash
# GPU tests + a short C3 kernel-only bench of the current build.
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 1 --no-e2e --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))"; }
echo "== default : $(run)" > gpurun_out/quick.log
echo "== default again : $(run)" >> gpurun_out/quick.log
