#!/bin/bash
# The driver's default bench line (cfg5) plus the other configs' lines and the reference arm.
out=gpurun_out/${1:-bench}; mkdir -p $out
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err
for w in cfg4 cfg1 cfg3 cfg2; do
  timeout 600 python bench.py --workload $w > $out/bench_$w.json 2> $out/bench_$w.err
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $out/ref_cfg5.json 2> $out/ref_cfg5.err
