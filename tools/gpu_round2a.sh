#!/bin/bash
out=gpurun_out/${1:-r2}; mkdir -p $out
timeout 1800 python -m pytest tests -q -m gpu --durations=10 > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:list_fused -c 1 -o $out/fused python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu --no-e2e > $out/ncu_fused.log 2>&1
bash tools/gpu_sanitize.sh ${1:-r2}/sanitize
