#!/bin/bash
# LIST contexts: the GPU suite, then the C3 entity (Alg. 1, LIST) line.   $1 = tag
T=${1:-ls}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/list_pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/list_pytest_$T.log
timeout 900 python bench.py --ctx-kind entities --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' > gpurun_out/list_entities_$T.jsonl
timeout 900 python bench.py --ctx-kind entities --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' >> gpurun_out/list_entities_$T.jsonl
