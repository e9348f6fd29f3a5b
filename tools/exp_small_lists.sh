d=gpurun_out/fz3; mkdir -p $d
for m in fused twopass; do for w in cfg1 cfg2; do
VXG_LIST_MODE=$m timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu --no-e2e > $d/${w}_$m.json 2>/dev/null
done; done
