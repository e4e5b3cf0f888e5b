# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02f
O=gpurun_out/r02f
timeout 2700 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
ALLN=$(seq -s, 2 64)
timeout 1200 python tools/stream_sweep.py --sizes $ALLN --dtypes f64,f32 --repeats 1,100 --gb 0.5 --steps 5 --out $O/all_n.jsonl > /dev/null 2> $O/all_n.err
timeout 1500 python tools/sweep.py --out $O/sweep_c1c3c4.jsonl > /dev/null 2> $O/sweep.err
mkdir -p /tmp/ncu
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_update|jm_generic" -o /tmp/ncu/kinds python tools/ncu_configs.py $(python tools/ncu_kinds.py) > $O/ncu_kinds.log 2>&1
python tools/ncu_summary.py /tmp/ncu/kinds.ncu-rep --algo $(python tools/ncu_kinds.py --algo) --json > $O/ncu_kinds.jsonl 2> $O/ncu_kinds_sum.err
ncu -i /tmp/ncu/kinds.ncu-rep --page raw --csv 2>/dev/null | gzip -c > $O/ncu_kinds_raw.csv.gz
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 1200 python tools/work_check.py --out $O/work_check.jsonl > /dev/null 2> $O/work_check.err
du -sh $O; tail -3 $O/gputest.txt; tail -2 $O/smoke.txt; head -c 400 $O/bench_c2.json; echo; head -c 300 $O/bench_reference.json; tail -2 $O/work_check.err
