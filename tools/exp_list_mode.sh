# list path: fused vs two-pass on cfg4 (tests first)
d=gpurun_out/${1:-lm}
mkdir -p $d
timeout 900 python -m pytest tests -x -q -m gpu > $d/pytest_gpu.log 2>&1; echo "rc=$?" >> $d/pytest_gpu.log
VXG_LIST_MODE=fused timeout 900 python -m pytest tests -x -q -m gpu -k "list or config4 or batch or acceptance or golden or random" > $d/pytest_fused.log 2>&1; echo "rc=$?" >> $d/pytest_fused.log
for m in fused twopass; do
  VXG_LIST_MODE=$m timeout 600 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu --no-e2e > $d/bench_$m.json 2> $d/bench_$m.err
done
VXG_LIST_MODE=fused timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"list_fused" -s 1 -c 1 -o $d/prof python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $d/ncu.log 2>&1
