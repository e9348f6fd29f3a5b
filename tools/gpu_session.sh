#!/bin/bash
# One GPU-box session: tests, bench lines per workload, ncu launch list of the default bench.
# Usage (from the repo root, under gpurun): bash tools/gpu_session.sh [tag]
tag=${1:-s}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
nproc > $out/nproc.txt; lscpu > $out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for w in cfg4 cfg1 cfg3 cfg5 cfg2; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > $out/bench_$w.json 2> $out/bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_bench.log 2>&1
