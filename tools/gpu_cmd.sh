# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# r02 final measurement pass: GPU suite, smoke, bench (+ launch list), reference arm, all-n sweep, C1/C3/C4 sweep, mass F7
O=gpurun_out/s9; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1; tail -3 $O/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 400 $O/bench_c2.json
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_launches_c2.csv python bench.py --steps 2 --warmup 3 > $O/ncu_bench.log 2>&1
timeout 1800 python tools/stream_sweep.py --sizes 2..64 --dtypes f64,f32 --repeats 1,100 --gb 0.5 --out $O/all_n.jsonl > /dev/null 2> $O/all_n.err
timeout 1200 python tools/sweep.py --out $O/sweep_c1c3c4.jsonl > /dev/null 2> $O/sweep.err
timeout 300 python tools/mass_bench.py --out $O/mass_f7.jsonl > /dev/null 2> $O/mass_f7.err
echo done
