#!/bin/bash
# Quick GPU iteration: tests, cfg4/cfg1 bench lines, one ncu --set full of a kernel.
# Usage: bash tools/gpu_quick.sh tag [kernel-regex] [bench args for the ncu run...]
tag=${1:-q}; shift
k=${1:-list_kernel}; shift
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for w in cfg4 cfg1; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $out/bench_$w.json 2> $out/bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $out/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 2 \
  -o $out/prof python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > $out/ncu_$k.log 2>&1
