#!/bin/bash
# Round measurement: GPU tests, smoke, default bench, launch list, and one
# `ncu --set full` capture of a STEADY-STATE decode launch (segment 2 of the
# warm-up step: channels 250 frames in, after two context switches), the
# launch the timed region is made of.   $1 = tag (outputs gpurun_out/*_TAG*)
# $2 = "notest" to skip pytest / smoke.
T=${1:-cur}
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
if [ "$2" != "notest" ]; then
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$T.log
fi
timeout 1200 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$T.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-overhead > gpurun_out/ncu_launch_$T.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch_$T.log
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_$T python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-overhead > gpurun_out/ncu_full_$T.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full_$T.log
