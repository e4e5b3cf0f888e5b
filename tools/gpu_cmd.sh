timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
./tools/microbench/lds_patterns > gpurun_out/lds_patterns.json 2>&1; cat gpurun_out/lds_patterns.json
python bench.py --steps 20 > gpurun_out/bench2.log 2> gpurun_out/bench2.err; tail -2 gpurun_out/bench2.err; cat gpurun_out/bench2.log
