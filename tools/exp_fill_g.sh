# G sweep of the bitmap fill (lanes per piece) on cfg5 (8M segments) and cfg3; plus one ncu capture
d=gpurun_out/${1:-e1}
mkdir -p $d
for G in 4 8; do
  VXG_FILL_G=$G timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:tiles_fill -c 2 --csv --log-file $d/fill_G$G.csv python bench.py --workload cfg5 --segments 8388608 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
  VXG_FILL_G=$G timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:tiles_fill -c 2 --csv --log-file $d/fill3_G$G.csv python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"tiles_fill" -s 1 -c 1 -o $d/prof5 python bench.py --workload cfg5 --segments 2097152 --steps 1 --warmup 1 --no-e2e --no-cpu > $d/ncu5.log 2>&1
