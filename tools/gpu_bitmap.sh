#!/bin/bash
# Bitmap iteration: tests, cfg3/cfg5 bench lines, launch list + ncu of the tile kernels (cfg3).
tag=${1:-b}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for w in cfg3 cfg5; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu > $out/bench_$w.json 2> $out/bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  --log-file $out/launches_cfg3.csv python bench.py --workload cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tiles_(count|scatter|fill)" -s 3 -c 3 \
  -o $out/prof python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_prof.log 2>&1
