#!/bin/bash
# Harness benchmark on the GPU box (bench_tools/harness_bench.py): the default
# 32x2x50 workload (compared against the reference run in the container) and a
# 512-channel one.
mkdir -p gpurun_out
python bench_tools/harness_bench.py --make /tmp/hb > /dev/null
timeout 600 python bench_tools/harness_bench.py --dir /tmp/hb --impl ours --repeats 3 > gpurun_out/harness_ours.json 2> gpurun_out/harness_ours.err
python bench_tools/harness_bench.py --make /tmp/hb512 --channels 512 > /dev/null
timeout 600 python bench_tools/harness_bench.py --dir /tmp/hb512 --impl ours --repeats 3 > gpurun_out/harness_ours512.json 2> gpurun_out/harness_ours512.err
