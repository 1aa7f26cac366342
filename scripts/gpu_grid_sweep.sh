: > gpurun_out/grid.log
for g in 512 592 1024; do
  AB_GRID=$g timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('grid $g', round(d['value']))" >> gpurun_out/grid.log
done
