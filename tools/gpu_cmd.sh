# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# FP32 n = 49..57 register caps at R = 100, then the full GPU suite, smoke and the C2 bench on the default build
O=gpurun_out/s18; mkdir -p $O
timeout 1200 python tools/ab.py --variant cap144="JM_F32T_MAXREG=144" --variant cap200="JM_F32T_MAXREG=200" \
  --variant base= --sizes 49..57 --dtypes f32 --repeats 100 --out $O/ab_cap.jsonl > $O/ab_cap.log 2>&1
python tools/ab.py --table $O/ab_cap.jsonl
timeout 2400 python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1; tail -3 $O/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 400 $O/bench_c2.json
