timeout 900 python -m pytest tests/test_gpu_stream.py -q -x 2>&1 | tail -2
timeout 900 python tools/sweep.py --only c4 --out gpurun_out/c4b.jsonl > /dev/null 2>&1; echo rc=$?
