# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -v "^\.\+ *\[" | tail -3
python tools/stream_sweep.py --sizes 20,24,28,32,36,40,44,48,52,56,60,64 --dtypes f32 --repeats 1,100 --gb 0.5 --steps 3 > gpurun_out/f32vec.jsonl 2>&1; echo rc=$?
