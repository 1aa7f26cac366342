#!/bin/bash
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/v12.jsonl
timeout 600 python bench.py --workload c1 --steps 3 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/v12.jsonl
timeout 600 python bench.py --workload c2 --steps 3 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/v12.jsonl
timeout 900 python bench.py --no-cpu 2>/dev/null | grep '^{' >> gpurun_out/v12.jsonl
