#!/bin/bash
T=${1:-cut3}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 600 python scripts/diag_cutoff.py > gpurun_out/diag_$T.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$T.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$T.log
