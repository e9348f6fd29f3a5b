#!/bin/bash
# One GPU-box session: tests, bench lines per workload (with the CPU reference baseline), the
# reference arm, launch lists and one ncu --set full capture of each dominant kernel.
# Usage (from the repo root, under gpurun): bash tools/gpu_session.sh [tag]
tag=${1:-s}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
nproc > $out/nproc.txt; lscpu > $out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for w in cfg4 cfg1 cfg3 cfg5 cfg2; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > $out/bench_$w.json 2> $out/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_reference_cfg5.json 2> $out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $out/launches_cfg4.csv python bench.py --workload cfg4 --steps 2 --warmup 3 --no-e2e --no-cpu > $out/ncu_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $out/launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu > $out/ncu_bench5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"list_(fused|count|emit)_kernel" -s 1 -c 1 \
  -o $out/prof_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_prof4.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tiles_(count|scatter|fill)" -s 3 -c 3 \
  -o $out/prof_cfg5 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_prof5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tiles_fill" -s 1 -c 1 \
  -o $out/prof_cfg3 python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > $out/ncu_prof3.log 2>&1
# the reference harness's scenarios: voxgpu bench beside the reference's own harness
bash tools/gpu_paper_tables.sh $tag/pt
[ -x tools/latency_probe ] || g++ -std=c++17 -O2 -I/usr/local/cuda/include -o tools/latency_probe tools/latency_probe.cpp \
  -Lpaper_2009_09500_b200/lib -lvoxgpu -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -lpthread -Wl,-rpath,'$ORIGIN/../paper_2009_09500_b200/lib'
( for a in "1 1000" "1 100000" "65536 128"; do echo "== $a"; ./tools/latency_probe $a; done ) > $out/latency_probe.txt 2>&1
