#!/bin/bash
out=gpurun_out/${1:-small}; mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu -k "run_batch_device or count_voxels or list or batch" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python bench.py --workload cfg1 --no-cpu --no-e2e > $out/bench_cfg1.json 2> $out/bench_cfg1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:list_small -s 3 -c 1 -o $out/small python bench.py --workload cfg1 --steps 1 --warmup 3 --no-cpu --no-e2e > $out/ncu_small.log 2>&1
for lib in default; do
  if [ $lib = default ]; then L=paper_2009_09500_b200/lib/libvoxgpu.so; else L=paper_2009_09500_b200/lib/var/libvoxgpu_4cta.so; fi
  VXG_LIBRARY=$L timeout 300 python bench.py --workload cfg4 --steps 10 --no-cpu --no-e2e > $out/bench_cfg4_$lib.json 2>> $out/err.log
done
