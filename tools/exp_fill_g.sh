mkdir -p gpurun_out/e1
for G in 8 16 32; do
  VXG_FILL_G=$G timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:tiles_fill -c 2 --csv --log-file gpurun_out/e1/fill_G$G.csv python bench.py --workload cfg5 --segments 8388608 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
  VXG_FILL_G=$G timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:tiles_fill -c 2 --csv --log-file gpurun_out/e1/fill3_G$G.csv python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
