python tools/stream_sweep.py --sizes 49,50,52,54,56 --dtypes f64 --repeats 8,100 --gb 1 --steps 3 > gpurun_out/t87.jsonl 2>&1; echo rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "49 or 50 or 52 or 55 or 56 or 57" 2>&1 | tail -2
