#!/bin/bash
T=${1:-cut4}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$T.log
bash scripts/gpu_variants_full.sh main n2k
