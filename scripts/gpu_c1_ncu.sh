#!/bin/bash
# ncu --set full of the C1 decode kernel (one channel over a cluster, 500
# frames) with source-level stall sampling, and the C1/C2 phase profile.  $1 = tag
T=${1:-c1}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 -o gpurun_out/prof_c1_$T python bench.py --workload c1 --steps 1 --warmup 0 --no-e2e --no-cpu --no-overhead > gpurun_out/ncu_c1_$T.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_c1_$T.log
for w in c1 c2; do
  ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_prof.so timeout 600 python bench.py --workload $w --steps 1 --warmup 1 --no-cpu --no-overhead --no-e2e 2>&1 | grep AB_PROFILE | tail -1 >> gpurun_out/c12prof_$T.log
done
