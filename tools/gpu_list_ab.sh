#!/bin/bash
# cfg4 A/B of library variants (interleaved, 2 rounds)
out=gpurun_out/${1:-lab}; shift; mkdir -p $out
for round in 1 2; do
for v in "$@"; do
  if [ $v = default ]; then L=paper_2009_09500_b200/lib/libvoxgpu.so; else L=paper_2009_09500_b200/lib/var/libvoxgpu_$v.so; fi
  echo "$v $(VXG_LIBRARY=$L timeout 300 python bench.py --workload cfg4 --steps 10 --no-cpu --no-e2e 2>>$out/err.log | tail -1)" >> $out/res.txt
done; done
