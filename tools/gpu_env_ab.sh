#!/bin/bash
# Fill variants on cfg5/cfg3 (bench lines only): bash tools/gpu_env_ab.sh TAG "ENV1" "ENV2" ...
out=gpurun_out/${1:-ab}; shift; mkdir -p $out
i=0
for e in "$@"; do
  for w in cfg5 cfg3; do
    env $e timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_${w}_$i.json 2> $out/bench_${w}_$i.err
  done
  echo "$i $e" >> $out/variants.txt
  i=$((i+1))
done
