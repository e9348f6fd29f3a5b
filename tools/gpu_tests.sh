#!/bin/bash
# Full GPU test suite with per-test durations (log under gpurun_out/<tag>/)
out=gpurun_out/${1:-tests}; shift; mkdir -p $out
timeout 3000 python -m pytest tests -q -m gpu --durations=15 "$@" > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
