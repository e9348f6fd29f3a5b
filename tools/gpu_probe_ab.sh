#!/bin/bash
# slab_probe (every rank's cfg5 step at N) per env variant: bash tools/gpu_probe_ab.sh TAG N "ENV1" ...
out=gpurun_out/${1:-pab}; N=$2; shift 2; mkdir -p $out
i=0
for e in "$@"; do
  env $e timeout 900 python tools/slab_probe.py $N > $out/probe_$i.txt 2>&1
  echo "$i $e" >> $out/variants.txt; i=$((i+1))
done
