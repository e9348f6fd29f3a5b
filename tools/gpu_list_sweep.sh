#!/bin/bash
# cfg4 fused list kernel: ranges per warp x count look-ahead sweep (VXG_FUSED_RPW / VXG_FUSED_LA)
out=gpurun_out/${1:-lsweep}; mkdir -p $out
for rpw in 32 16 48; do for la in 1.0 0.5 2.0; do
  echo "rpw$rpw la$la $(VXG_FUSED_RPW=$rpw VXG_FUSED_LA=$la timeout 300 python bench.py --workload cfg4 --steps 10 --no-cpu --no-e2e 2>>$out/err.log | tail -1)" >> $out/res.txt
done; done
