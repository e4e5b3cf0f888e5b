timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -v "^\.\+ *\[" | tail -5
python tools/stream_sweep.py --sizes 8,10,16,24,26,32,40,48,56,64 --dtypes f64 --repeats 1,4,100 --gb 2 --steps 3 > gpurun_out/vecld.jsonl 2>&1; echo rc=$?
