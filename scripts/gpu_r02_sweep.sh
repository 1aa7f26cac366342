#!/bin/bash
# Round-2 layout sweep: DRAM bytes per channel-frame and frames/s of the C3
# steady-state launch for CTA size x token-table layout, plus the DRAM bytes a
# random 16-B load / CAS-128 really moves (access granularity).
mkdir -p gpurun_out
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_sw.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sw.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rap bench_tools/random_access_peak.cu
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_requests_srcunit_tex.sum,gpu__time_duration.sum -k regex:"read16|cas16" --csv --log-file gpurun_out/gran.csv /tmp/rap > gpurun_out/gran.log 2>&1
run() { # tag, env..., args
  tag=$1; shift
  env "$@" timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-overhead $ARGS > gpurun_out/sw_$tag.log 2>&1
  env "$@" timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:decode_kernel -s 2 -c 1 --csv --log-file gpurun_out/sw_$tag.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-overhead $ARGS > /dev/null 2>&1
}
ARGS=""
run b256d AB_BLOCK=256
run b1024d AB_BLOCK=1024
ARGS="--table-slots 65536"
run b256h16 AB_BLOCK=256
run b512h16 AB_BLOCK=512
run b1024h16 AB_BLOCK=1024
ARGS="--table-slots 131072"
run b1024h17 AB_BLOCK=1024
