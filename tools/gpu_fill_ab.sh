#!/bin/bash
# A/B of the bitmap fill: old uniform loop vs per-lane trip counts, and blocked tile claim orders.
out=gpurun_out/${1:-fill_ab}; mkdir -p $out
timeout 600 python -m pytest tests -x -q -m gpu -k "bitmap or slab" > $out/pytest_bitmap.log 2>&1; echo "rc=$?" >> $out/pytest_bitmap.log
b() { timeout 300 python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu --no-e2e 2>>$out/err.log | tail -1; }
echo "uni $(VXG_LIBRARY=paper_2009_09500_b200/lib/var/libvoxgpu_uni.so b)" >> $out/res.txt
echo "new $(b)" >> $out/res.txt
for o in 2,2,2 4,4,4 8,4,4 4,4,2 8,8,8 32,2,2 32,4,2 16,4,4; do
  echo "order $o $(VXG_FILL_ORDER=$o b)" >> $out/res.txt
done
