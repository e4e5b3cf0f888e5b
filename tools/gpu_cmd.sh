timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "f32" 2>&1 | tail -2
python tools/stream_sweep.py --sizes 17,20,24,25,28,32,33,36,40,44,48,52,56,60,64 --dtypes f32 --repeats 1,100 --gb 1 --steps 3 > gpurun_out/f32blk.jsonl 2>&1; echo rc=$?
