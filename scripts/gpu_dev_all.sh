#!/bin/bash
# Development check after a kernel change: the full GPU suite, the C1/C2 loop
# (scripts/gpu_c12_dev.sh) and a short C3 bench line.   $1 = tag
T=${1:-dev}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/dev_pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/dev_pytest_$T.log
bash scripts/gpu_c12_dev.sh $T
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-overhead > gpurun_out/dev_c3_$T.log 2>&1; echo "rc=$?" >> gpurun_out/dev_c3_$T.log
