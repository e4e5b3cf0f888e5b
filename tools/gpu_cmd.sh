timeout 900 python -m pytest tests/test_gpu_stream.py -q -x 2>&1 | tail -2
python tools/stream_sweep.py --sizes 12,13,14,16 --dtypes f32 --repeats 1,2,4 --gb 1 --steps 3 > gpurun_out/f32pring.jsonl 2>&1; echo rc=$?
