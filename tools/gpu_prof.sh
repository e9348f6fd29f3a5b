#!/bin/bash
# ncu --set full captures of the list kernels at 1M segments of config 4 (run under gpurun).
tag=${1:-p}
out=gpurun_out/$tag
mkdir -p $out
for k in list_count_kernel list_emit_kernel emit_bitmap_kernel plan_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o $out/$k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --segments 1048576 \
    $( [ $k = emit_bitmap_kernel ] && echo --workload cfg3 --segments 2097152 ) > $out/ncu_$k.log 2>&1
done
