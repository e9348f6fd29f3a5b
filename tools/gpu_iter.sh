#!/bin/bash
# One GPU iteration: list tests + cfg4/cfg1 bench + ncu metrics of the bitmap fill.
out=gpurun_out/${1:-iter}; mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu -k "not full" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for w in cfg4 cfg1; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_$w.json 2>>$out/err.log
done
timeout 600 ncu --clock-control none -k regex:tiles_fill -c 1 \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_mio_throttle,smsp__average_warp_latency_issue_stalled_short_scoreboard,dram__bytes_read.sum \
  python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu --no-e2e > $out/ncu_fill.txt 2>&1
