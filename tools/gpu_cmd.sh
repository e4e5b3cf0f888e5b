# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+ *\[" | tail -3
python tools/stream_sweep.py --sizes 21,22,23,24,36,37,38,39,40 --dtypes f32 --repeats 1,100 --gb 1 --steps 3 > gpurun_out/f32ovr2.jsonl 2>&1; echo rc=$?
