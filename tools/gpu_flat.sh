out=gpurun_out/flat1; mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu -k "list or batch or config or golden or random or ties or corpora or segments or edges or concurrent or torch or device or run_batch or count" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
bash tools/gpu_list_ab.sh flat1 pf2 flat
timeout 300 python bench.py --workload cfg1 --no-cpu --no-e2e > $out/bench_cfg1.json 2>>$out/err.log
