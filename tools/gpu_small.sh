#!/bin/bash
out=gpurun_out/${1:-small}; mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu -k "run_batch_device or count_voxels or list or batch" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python bench.py --workload cfg1 --no-cpu > $out/bench_cfg1.json 2> $out/bench_cfg1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $out/launches_cfg1.csv python bench.py --workload cfg1 --steps 3 --warmup 3 --no-cpu --no-e2e > $out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:list_small -s 3 -c 1 -o $out/small python bench.py --workload cfg1 --steps 1 --warmup 3 --no-cpu --no-e2e > $out/ncu_small.log 2>&1
