#!/bin/bash
# A/B: fill record prefetch modes, scatter pipeline depth, tile order (DRAM bytes of the fill)
out=gpurun_out/${1:-fill3}; mkdir -p $out
timeout 600 python -m pytest tests -x -q -m gpu -k "bitmap or slab" > $out/pytest_bitmap.log 2>&1; echo "rc=$?" >> $out/pytest_bitmap.log
b() { timeout 300 python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu --no-e2e 2>>$out/err.log | tail -1; }
for pf in 1 2 3 6 0; do echo "pf$pf $(VXG_FILL_PF=$pf b)" >> $out/res.txt; done
for d in 1 2 3 4; do echo "scatterD$d $(VXG_SCATTER_D=$d b)" >> $out/res.txt; done
for o in 0 4,4,4 32,4,2; do
VXG_FILL_ORDER=$o timeout 600 ncu --clock-control none -k regex:tiles_fill -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct \
  python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu --no-e2e > $out/ncu_order_$o.txt 2>&1
done
