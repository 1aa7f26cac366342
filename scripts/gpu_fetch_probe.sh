#!/bin/bash
# DRAM bytes per random access (bench_tools/fetch_probe.cu) under ncu.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp bench_tools/fetch_probe.cu
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_requests_srcunit_tex.sum,gpu__time_duration.sum -k regex:rd --csv --log-file gpurun_out/fetch_probe.csv /tmp/fp > gpurun_out/fetch_probe.log 2>&1
/tmp/fp > gpurun_out/fetch_probe_plain.log 2>&1
