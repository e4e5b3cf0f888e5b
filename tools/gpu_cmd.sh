timeout 900 python -m pytest tests/test_gpu_stream.py -q -x 2>&1 | tail -2
python tools/stream_sweep.py --sizes 17,20,24,28,32,40,48,56,64 --dtypes f32 --repeats 1,2,4,8 --gb 1 --steps 3 > gpurun_out/f32s.jsonl 2>&1; echo rc=$?
