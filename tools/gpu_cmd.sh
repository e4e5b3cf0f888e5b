timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
python tools/stream_sweep.py --sizes 33,34,41,42,49,50,57,58 --dtypes f64 --repeats 1,4,100 --gb 1 --steps 3 > gpurun_out/bord2.jsonl 2>&1; echo rc=$?
