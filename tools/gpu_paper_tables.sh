#!/bin/bash
# The reference harness's three scenarios (paper Tables 2-4 shapes) at the reference's default
# desk scale: `voxgpu bench` (GPU path) beside oracle/_ref/ref_bench (the reference's own
# src/bench.cpp on the host cores). Usage (under gpurun): bash tools/gpu_paper_tables.sh TAG
tag=${1:-pt}
out=gpurun_out/$tag
mkdir -p $out
nproc > $out/nproc.txt
for sc in single fixed-batch arbitrary; do
  timeout 900 paper_2009_09500_b200/bin/voxgpu bench --scenario $sc --report $out/gpu_$sc.csv \
    --report-json $out/gpu_$sc.json > $out/gpu_$sc.txt 2>&1
  timeout 900 oracle/_ref/ref_bench $sc --report $out/ref_$sc.csv > $out/ref_$sc.txt 2>&1
done
