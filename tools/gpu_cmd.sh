# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+ *\[" | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_v7.json 2> gpurun_out/bench_v7.err; echo bench rc=$?
for cfg in "--size 8 --batch 67108864 --repeat 100" "--size 8 --batch 67108864 --repeat 1" "--size 32 --batch 4194304 --repeat 100" "--size 32 --batch 4194304 --repeat 1"; do
  timeout 900 python bench.py --no-cpu --no-e2e --steps 10 $cfg >> gpurun_out/c5_v7.jsonl 2>>gpurun_out/c5_v7.err; done; echo c5 rc=$?
python tools/stream_sweep.py --sizes $(seq -s, 2 64) --dtypes f64,f32 --repeats 1,100 --gb 0.5 --steps 3 > gpurun_out/all_n_v3.jsonl 2>&1; echo alln rc=$?
timeout 900 python tools/sweep.py --only c4 --out gpurun_out/c4_v7.jsonl > /dev/null 2>&1; echo c4 rc=$?
