timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -v "^\.\+ *\[" | tail -15
python tools/stream_sweep.py --sizes 8 --dtypes f64 --repeats 1,2,3,4,8,16,100 --gb 2 --steps 3 > gpurun_out/tpm2.jsonl 2>&1; echo rc=$?
