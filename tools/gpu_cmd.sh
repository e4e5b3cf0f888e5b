timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -v "^\.\+ *\[" | tail -4
python tools/stream_sweep.py --sizes 12,13,14,15,16 --dtypes f32 --repeats 1,10,100 --gb 1 --steps 3 > gpurun_out/f32p_inpl.jsonl 2>&1; echo rc=$?
