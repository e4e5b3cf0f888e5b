timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+ *\[" | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python tools/sweep.py --out gpurun_out/sweep_v6.jsonl > gpurun_out/sweep_v6.log 2>&1; echo sweep rc=$?
timeout 600 python bench.py > gpurun_out/bench_v6.json 2> gpurun_out/bench_v6.err; echo bench rc=$?
python tools/stream_sweep.py --sizes $(seq -s, 2 64) --dtypes f64,f32 --repeats 1,100 --gb 0.5 --steps 3 > gpurun_out/all_n_v2.jsonl 2>&1; echo alln rc=$?
