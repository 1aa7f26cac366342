for t in main n2k; do
  if [ "$t" = main ]; then lib=paper_2306_15685_b200/libarcboost_b200.so; else lib=paper_2306_15685_b200/libarcboost_b200_$t.so; fi
  AB_VERBOSE=1 ARCBOOST_B200_LIB=$lib timeout 300 python bench.py --frames 20 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-overhead 2>&1 | grep arcboost | head -2 | sed "s/^/$t /" >> gpurun_out/occ.log
done
