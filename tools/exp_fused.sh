# fused list kernel: ranges per warp x lookahead sweep on cfg4
d=gpurun_out/${1:-fz}
mkdir -p $d
for rpw in 16 32 64 128; do for la in 1 4; do
  VXG_FUSED_RPW=$rpw VXG_FUSED_LA=$la timeout 300 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu --no-e2e > $d/b_${rpw}_${la}.json 2>/dev/null
done; done
