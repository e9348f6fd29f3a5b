#!/bin/bash
# Multi-GPU evidence on a one-GPU box: every rank's cfg5 step timed in turn (tools/slab_probe.py,
# N = 1, 2, 4, 8) and bench.py's N > 1 path with 2 gloo ranks sharing the GPU (--verify).
out=gpurun_out/${1:-multi}; mkdir -p $out
( for N in 1 2 4 8; do echo "== N=$N"; timeout 900 python tools/slab_probe.py $N; done ) > $out/slab_probe_balanced.txt 2>&1
bash tools/gpu_multi_rank.sh ${1:-multi}/gloo2
