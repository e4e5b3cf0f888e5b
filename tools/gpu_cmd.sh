# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q -x -k "17 or 18 or 19 or 20 or 25" 2>&1 | tail -2
python tools/stream_sweep.py --sizes 17,18,19,20,25 --dtypes f32 --repeats 1,100 --gb 0.5 --steps 3 > gpurun_out/f32ovr.jsonl 2>&1; echo rc=$?
