# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# final check of the final build: GPU suite, smoke, mass (all pairs + Fig. 7 analog), C2 bench
O=gpurun_out/s16; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1; tail -3 $O/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 600 python tools/mass_bench.py --pairs all --elements 2097152 --out $O/mass_all.jsonl > /dev/null 2> $O/mass_all.err
timeout 300 python tools/mass_bench.py --out $O/mass_f7.jsonl > /dev/null 2> $O/mass_f7.err
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json
