#!/bin/bash
# Copy one gpu_session.sh run's evidence from gpurun_out/TAG into profiles/DEST (run here).
tag=$1; dest=profiles/$2; src=gpurun_out/$tag
mkdir -p $dest
cp $src/bench_*.json $src/pytest_gpu.log $src/smoke.log $dest/ 2>/dev/null
cp $src/launches_*.csv $src/latency_probe.txt $src/nvidia-smi.txt $dest/ 2>/dev/null
[ -d $src/pt ] && cp -r $src/pt $dest/paper_tables
for r in $src/prof_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_kernels.py $r > $dest/ncu_${b}_kernels.txt 2>&1
  python tools/ncu_summary.py $r --top 30 > $dest/ncu_${b}_summary.txt 2>&1
done
ls $dest
