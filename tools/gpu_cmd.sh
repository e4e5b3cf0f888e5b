# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+ *\[" | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; echo bench rc=$?
timeout 1800 python tools/sweep.py --out gpurun_out/sweep_v9.jsonl > gpurun_out/sweep_v9.log 2>&1; echo sweep rc=$?
python tools/stream_sweep.py --sizes $(seq -s, 2 64) --dtypes f64,f32 --repeats 1,100 --gb 0.5 --steps 3 > gpurun_out/all_n_v4.jsonl 2>&1; echo alln rc=$?
timeout 1800 python tools/work_check.py --out gpurun_out/work_check4.jsonl > gpurun_out/work_check4.log 2>&1; echo wc rc=$?
