# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# tensor-core FP32 kind for n not a multiple of 8 (zero-padded to 8*ceil(n/8)): error, parity, A/B; default-build GPU suite
O=gpurun_out/s29; mkdir -p $O
JM_BUILD_DEFINES="JM_F32TC_ODD=33" python -c "import paper_1904_08555_b200._build as b; b.build(force=True)" > $O/build_odd.log 2>&1
timeout 600 python tools/tc_err.py 35,47,57,63 2>&1 | tee $O/tc_err_odd.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "f32 and (33 or 35 or 38 or 41 or 44 or 47 or 50 or 53 or 57 or 60 or 63)" > $O/parity_odd.txt 2>&1; tail -2 $O/parity_odd.txt; grep -E "^FAILED" $O/parity_odd.txt | head -3
timeout 1500 python tools/ab.py --variant odd="JM_F32TC_ODD=33" --variant base= \
  --sizes 35,38,41,44,47,50,53,57,60,63 --dtypes f32 --repeats 100,8 --out $O/ab_odd.jsonl > $O/ab_odd.log 2>&1
python - <<'PY'
import json
rows={}
for l in open('gpurun_out/s29/ab_odd.jsonl'):
    d=json.loads(l); rows.setdefault((d['n'],d['repeat']),{})[d['ab']]=(d['resident']['frac_pipe'], d['auto']['frac_pipe'])
for k in sorted(rows): print(k, rows[k])
PY
timeout 2000 python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1; tail -2 $O/gputest.txt; grep -E "^FAILED" $O/gputest.txt | head
