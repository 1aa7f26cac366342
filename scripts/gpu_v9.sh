#!/bin/bash
# random-access ceiling + full ncu capture of the default library's decode kernel
mkdir -p gpurun_out
timeout 300 ./bench_tools/random_access_peak > gpurun_out/random_access_peak.json 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 -o gpurun_out/prof_v8 python bench.py --frames 20 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_v8.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_v8.log
