timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/stream_sweep.py --sizes 9,10,17,18,25,26,33,34 --dtypes f64 --repeats 1,8,100 --gb 1 --steps 3 > gpurun_out/border.jsonl 2>&1; echo rc=$?
