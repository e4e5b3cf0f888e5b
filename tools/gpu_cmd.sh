timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/matmul_bench.py --out gpurun_out/matmul_r01.jsonl > gpurun_out/matmul.log 2>&1; tail -12 gpurun_out/matmul.log | cut -c1-700
