timeout 900 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
timeout 1500 python tools/stream_sweep.py --sizes 16,32,48,64 --dtypes f64 --repeats 1,2,4,8,16,32,100 --gb 2 --steps 3 --out gpurun_out/stream_v3.jsonl > gpurun_out/stream_v3.log 2>&1; echo sweep rc=$?
