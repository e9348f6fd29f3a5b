#!/bin/bash
# Functional check of bench.py's N > 1 path on a one-GPU box: 2 ranks (gloo) share GPU 0.
out=gpurun_out/${1:-mr}
mkdir -p $out
for w in cfg5 cfg4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --workload $w --segments 4194304 \
    --dist-backend gloo --no-e2e > $out/bench2_$w.json 2> $out/bench2_$w.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > $out/ref2.json 2> $out/ref2.err
