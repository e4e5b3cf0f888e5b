timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+ *\[" | tail -4
python tools/stream_sweep.py --sizes 49,51,53,55,57,59,61,63 --dtypes f32 --repeats 1,2,4 --gb 0.5 --steps 3 > gpurun_out/f32odd.jsonl 2>&1; echo rc=$?
