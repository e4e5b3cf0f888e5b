timeout 1800 python tools/sweep.py --out gpurun_out/sweep_v2.jsonl > gpurun_out/sweep_v2.log 2>&1; echo sweep rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update_stream -s 3 -c 1 -o gpurun_out/prof_stream32 python bench.py --n 32 --repeat 1 --batch 1000000 --steps 2 --warmup 3 --no-generic --no-e2e --no-cpu > gpurun_out/prof_stream32.log 2>&1; echo ncu rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_stream32.csv python bench.py --n 32 --repeat 1 --batch 1000000 --steps 4 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2 rc=$?
timeout 600 python bench.py --n 32 --repeat 1 --batch 1000000 --no-cpu > gpurun_out/bench_stream32.json 2>&1
