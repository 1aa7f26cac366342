#!/bin/bash
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 2 --no-e2e --no-cpu 2>&1 | grep '^{' ; }
for L in default u1 u3; do
  for B in 128 256; do
    if [ $L = default ]; then lib=paper_2306_15685_b200/libarcboost_b200.so; else lib=build_variants/lib_$L.so; fi
    echo "== $L B$B $(ARCBOOST_B200_LIB=$lib AB_BLOCK=$B run)" >> gpurun_out/sweep.log
  done
done
timeout 600 python bench.py --no-cpu > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
