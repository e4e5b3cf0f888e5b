timeout 1500 python -m pytest tests/test_gpu_stream.py -q -x 2>&1 | tail -2
python tools/stream_sweep.py --sizes 18,20,22,24,26,28,30,34,36,40,44,50,56,62 --dtypes f64 --repeats 1,4 --gb 0.5 --steps 3 > gpurun_out/dslot.jsonl 2>&1; echo rc=$?
