timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 1200 python tools/sweep.py --out gpurun_out/sweep_r01d.jsonl > gpurun_out/sweep_d.log 2>&1; wc -l gpurun_out/sweep_r01d.jsonl
python bench.py > gpurun_out/bench4.log 2> gpurun_out/bench4.err; tail -c 1500 gpurun_out/bench4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2b.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 -o gpurun_out/prof_c2b python bench.py --steps 2 --warmup 3 --no-generic --no-e2e --no-cpu > /dev/null 2>&1
ls gpurun_out/*c2b*
