out=gpurun_out/r2a
mkdir -p $out
(nproc; free -g; lscpu | head -30; nvidia-smi; df -h /dev/shm /tmp) > $out/host.txt 2>&1
for w in cfg4 cfg1 cfg5; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_$w.json 2> $out/bench_$w.err
done
