#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py
out=gpurun_out/${1:-sanitize}; mkdir -p $out
K='kns=plan_kernel|list_fused_kernel|list_small_kernel|tiles_scan_lb_kernel|tiles_fill_kernel|tiles_scatter_kernel|tiles_count_kernel'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-name "$K" --print-limit 50 \
    python tools/sanitize_driver.py > $out/$tool.log 2>&1
  echo "exit=$?" >> $out/$tool.log
done
