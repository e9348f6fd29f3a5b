#!/bin/bash
# Functional check of bench.py's N > 1 path on a one-GPU box: 2 ranks (gloo) share GPU 0, with
# --verify (every rank's output digest against the one-rank result) and the e2e leg
# (shard.distribute_segments for the z-slab configs).
out=gpurun_out/${1:-mr}
mkdir -p $out
port=29511
for w in cfg1 cfg4 cfg3 cfg5; do
  port=$((port+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 2 --steps 3 --warmup 2 --workload $w --verify \
    --dist-backend gloo > $out/bench2_$w.json 2> $out/bench2_$w.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29599 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --workload cfg1 > $out/ref2.json 2> $out/ref2.err
