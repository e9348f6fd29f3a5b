#!/bin/bash
out=gpurun_out/${1:-fill2}; mkdir -p $out
b() { timeout 300 python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu --no-e2e 2>>$out/err.log | tail -1; }
for G in 1 2 4; do echo "G$G $(VXG_FILL_G=$G b)" >> $out/res.txt; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiles_fill -c 1 -o $out/fill \
  python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu --no-e2e > $out/ncu_fill.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiles_scatter -c 1 -o $out/scatter \
  python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu --no-e2e > $out/ncu_scatter.log 2>&1
