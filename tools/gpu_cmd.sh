# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# FP32 n = 16, 32 on the tensor cores by default: GPU suite, smoke, resident/streaming crossover, ncu of the kind
O=gpurun_out/s22; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1; tail -3 $O/gputest.txt; grep -E "^FAILED" $O/gputest.txt | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; grep -E "f32|Error" $O/smoke.txt
timeout 600 python tools/stream_sweep.py --sizes 16,32 --dtypes f32 --repeats 1,2,3,4,6,8,100 --out $O/xover.jsonl > /dev/null 2> $O/xover.err
python - <<'PY'
import json
for l in open('gpurun_out/s22/xover.jsonl'):
    d=json.loads(l); print(d['n'], d['repeat'], {k:(d[k].get('frac_pipe'), d[k].get('frac_hbm'), d[k].get('ms')) for k in ('resident','streaming','auto') if k in d})
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -o $O/prof_f32tc \
  python tools/ncu_configs.py 16:f32:262144:100:resident 32:f32:65536:100:resident > $O/ncu.log 2>&1; tail -1 $O/ncu.log
ncu -i $O/prof_f32tc.ncu-rep --page raw --csv > $O/prof_f32tc_raw.csv 2>/dev/null
