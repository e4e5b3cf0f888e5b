timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/stream_sweep.py --sizes $(seq -s, 8 64) --dtypes f64 --repeats 1,100 --gb 1 --steps 3 > gpurun_out/f64_all.jsonl 2>&1; echo rc=$?
