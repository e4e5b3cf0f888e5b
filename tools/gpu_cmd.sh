timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+ *\[" | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python tools/sweep.py --out gpurun_out/sweep_v4.jsonl > gpurun_out/sweep_v4.log 2>&1; echo sweep rc=$?
timeout 600 python bench.py > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2_v4.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_v4.json 2>&1; echo ref rc=$?
