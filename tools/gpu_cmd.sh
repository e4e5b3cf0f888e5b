set -x
timeout 900 python -m pytest tests/test_gpu_matmul.py -x -q 2>&1 | tail -15
timeout 600 python tools/matmul_bench.py --out gpurun_out/matmul.jsonl > gpurun_out/matmul.log 2>&1; echo rc=$?; grep HBM gpurun_out/matmul.jsonl
