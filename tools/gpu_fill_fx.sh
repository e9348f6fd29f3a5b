#!/bin/bash
# Fill A/B: fixed-point stepping (default) against the exact-FP64 fill (VXG_FILL_PF=9), bitmap
# parity tests, and one ncu capture of the fill.   bash tools/gpu_fill_fx.sh TAG
out=gpurun_out/${1:-fx}; mkdir -p $out
timeout 1200 python -m pytest tests -x -q -m gpu -k "bitmap or config3 or config5 or ties or fixed_point" > $out/pytest_bitmap.log 2>&1; echo "rc=$?" >> $out/pytest_bitmap.log
for w in cfg5 cfg3; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_$w.json 2> $out/bench_$w.err
  VXG_FILL_PF=9 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_${w}_exact.json 2> $out/bench_${w}_exact.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tiles_fill" -s 1 -c 1 \
  -o $out/prof_fill5 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_fill5.log 2>&1
