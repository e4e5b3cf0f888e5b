./tools/microbench/lds_patterns > gpurun_out/lds_patterns.json 2>&1; cat gpurun_out/lds_patterns.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -c 1 -o gpurun_out/prof_tpm4 python bench.py --n 4 --dtype f64 --batch 4194304 --steps 1 --warmup 1 --no-generic --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -c 1 -o gpurun_out/prof_dmma8 python bench.py --n 8 --dtype f64 --batch 1048576 --steps 1 --warmup 1 --no-generic --no-e2e --no-cpu > /dev/null 2>&1
ls gpurun_out
