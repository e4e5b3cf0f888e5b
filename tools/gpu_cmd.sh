# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 1800 python tools/sweep.py --out gpurun_out/sweep_v10.jsonl > gpurun_out/sweep_v10.log 2>&1; echo sweep rc=$?
timeout 600 python bench.py > gpurun_out/bench_v10.json 2> gpurun_out/bench_v10.err; echo bench rc=$?
