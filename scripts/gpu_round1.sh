#!/bin/bash
# First GPU shakedown: smoke, GPU tests, small + default bench.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
make -C oracle > /dev/null 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload c1 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c1.log
timeout 600 python bench.py --channels 128 --frames 100 --steps 2 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_small.log 2>&1; echo "rc=$?" >> gpurun_out/bench_small.log
