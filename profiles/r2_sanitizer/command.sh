#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py:
# every kernel of the driver's run is instrumented (plan, fused list, small-batch list, bitmap
# count / scan / scatter / fill, slab select), each output checked against the oracle.
out=gpurun_out/${1:-sanitize}; mkdir -p $out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 \
    python tools/sanitize_driver.py > $out/$tool.log 2>&1
  echo "exit=$?" >> $out/$tool.log
done
