timeout 1800 python tools/sweep.py --out gpurun_out/sweep_v5.jsonl > gpurun_out/sweep_v5.log 2>&1; echo sweep rc=$?
timeout 1800 python tools/work_check.py --out gpurun_out/work_check3.jsonl > gpurun_out/work_check3.log 2>&1; echo wc rc=$?
python tools/stream_sweep.py --sizes $(seq -s, 2 64) --dtypes f64,f32 --repeats 1,100 --gb 0.5 --steps 3 > gpurun_out/all_n.jsonl 2>&1; echo alln rc=$?
