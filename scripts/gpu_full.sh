#!/bin/bash
# Full round measurement: tests, smoke, default bench, launch list, one ncu --set full capture.
# $1 = tag for output names (e.g. r01_v9)
T=${1:-cur}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$T.log
timeout 1200 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$T.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --frames 20 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-overhead > gpurun_out/ncu_launch_$T.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch_$T.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 -o gpurun_out/prof_$T python bench.py --frames 20 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-overhead > gpurun_out/ncu_full_$T.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full_$T.log
