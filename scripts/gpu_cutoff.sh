#!/bin/bash
# Expansion-time cutoff: GPU parity (both modes), then C3 bench with the cutoff and exact.
T=${1:-cut}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$T.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$T.log
timeout 900 python bench.py --no-cpu --no-e2e --no-overhead --exact > gpurun_out/bench_${T}_exact.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${T}_exact.log
