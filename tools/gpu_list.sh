#!/bin/bash
# List path: parity tests, cfg4/cfg1 bench lines (fixed point vs FP64 fast runs), one ncu capture
# of the fused kernel.   bash tools/gpu_list.sh TAG [noprof]
out=gpurun_out/${1:-list}; mkdir -p $out
timeout 1500 python -m pytest tests -x -q -m gpu -k "list or config4 or ties or golden or corpora or uniform or batch or fixed_point or chain or int32 or error or round_pos" > $out/pytest_list.log 2>&1; echo "rc=$?" >> $out/pytest_list.log
for w in cfg4 cfg1; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu --no-e2e > $out/bench_$w.json 2> $out/bench_$w.err
  VXG_LIST_FX=0 timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu --no-e2e > $out/bench_${w}_fp64.json 2> $out/bench_${w}_fp64.err
done
[ "$2" = noprof ] && exit 0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"list_(fused|count|emit)_kernel" -s 1 -c 1 \
  -o $out/prof_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_prof4.log 2>&1
