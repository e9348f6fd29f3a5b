#!/bin/bash
# cfg5 A/B of library variants (interleaved, 2 rounds); args: tag variant...
out=gpurun_out/${1:-bab}; shift; mkdir -p $out
timeout 600 python -m pytest tests -x -q -m gpu -k "(bitmap or slab) and not full" > $out/pytest_bitmap.log 2>&1; echo "rc=$?" >> $out/pytest_bitmap.log
for round in 1 2; do
for v in "$@"; do
  if [ $v = default ]; then L=paper_2009_09500_b200/lib/libvoxgpu.so; else L=paper_2009_09500_b200/lib/var/libvoxgpu_$v.so; fi
  echo "$v $(VXG_LIBRARY=$L timeout 300 python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu --no-e2e 2>>$out/err.log | tail -1)" >> $out/res.txt
done; done
