#!/bin/bash
# cfg1 (small-batch one-launch kernel): its parity tests, then bench lines per env variant.
#   bash tools/gpu_cfg1_ab.sh TAG "ENV1" "ENV2" ...
out=gpurun_out/${1:-c1}; shift; mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu -k "one_launch or device_batch or torch or golden_batch or config_scaled or fixed_point" > $out/pytest_small.log 2>&1; echo "rc=$?" >> $out/pytest_small.log
i=0
for e in "$@"; do
  env $e timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu --no-e2e > $out/bench_cfg1_$i.json 2> $out/bench_cfg1_$i.err
  echo "$i $e" >> $out/variants.txt; i=$((i+1))
done
