timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -v "^\.\+ *\[" | tail -5
python tools/stream_sweep.py --sizes 5,6,7 --dtypes f64 --repeats 1,100 --gb 1 --steps 3 > gpurun_out/tpmpf.jsonl 2>&1
python tools/stream_sweep.py --sizes 8 --dtypes f32 --repeats 1,100 --gb 1 --steps 3 >> gpurun_out/tpmpf.jsonl 2>&1; echo rc=$?
