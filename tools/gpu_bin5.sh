#!/bin/bash
# cfg5/cfg3 bitmap pipeline: bitmap parity tests, bench lines, one ncu capture of the binning and
# fill kernels.   bash tools/gpu_bin5.sh TAG [noprof]
out=gpurun_out/${1:-bin5}; mkdir -p $out
timeout 1200 python -m pytest tests -x -q -m gpu -k "bitmap or config3 or config5 or ties or fixed_point or slab" > $out/pytest_bitmap.log 2>&1; echo "rc=$?" >> $out/pytest_bitmap.log
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_cfg5.json 2> $out/bench_cfg5.err
timeout 600 python bench.py --workload cfg3 --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_cfg3.json 2> $out/bench_cfg3.err
[ "$2" = noprof ] && exit 0
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tiles_(count|scatter|fill)" -s 3 -c 3 \
  -o $out/prof_cfg5 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_prof5.log 2>&1
