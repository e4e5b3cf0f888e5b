# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# tensor-core FP32 kind with the non-finite fallback: GPU suite, smoke, cost of the check (A/B), C3 FP32 sweep, all-n FP32 rows
O=gpurun_out/s25; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1; tail -2 $O/gputest.txt; grep -E "^FAILED" $O/gputest.txt | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -3 $O/smoke.txt
timeout 900 python tools/ab.py --variant unsafe="JM_F32TC_SAFE=0" --variant safe= --sizes 16,32,64 --dtypes f32 --repeats 100,8 --out $O/ab_safe.jsonl > $O/ab_safe.log 2>&1
python tools/ab.py --table $O/ab_safe.jsonl
timeout 900 python tools/sweep.py --only c3 --dtypes f32 --out $O/sweep_c3_f32.jsonl > $O/sweep_c3.log 2>&1
timeout 1200 python tools/stream_sweep.py --sizes 2..64 --dtypes f32 --repeats 1,100 --gb 0.5 --out $O/all_n_f32.jsonl > /dev/null 2> $O/all_n.err
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 200 $O/bench_c2.json
