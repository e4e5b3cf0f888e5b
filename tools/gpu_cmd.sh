# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+ *\[" | tail -3
timeout 600 python bench.py --steps 10 --no-cpu > gpurun_out/bench_v8.json 2> gpurun_out/bench_v8.err; echo bench rc=$?
timeout 600 ncu --nvtx --nvtx-include "jm:run/" --metrics gpu__time_duration.sum --csv -c 3 python bench.py --steps 3 --warmup 3 --no-generic --no-e2e --no-cpu 2>&1 | grep -c k_update
