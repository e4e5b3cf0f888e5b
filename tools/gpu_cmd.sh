# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# tensor-core FP32 kind at n = 24, 40, 48, 56 (padded last m-tile where n % 16 == 8): error, parity, A/B
O=gpurun_out/s27; mkdir -p $O
JM_BUILD_DEFINES="JM_F32TC_ALL=1" python -c "import paper_1904_08555_b200._build as b; b.build(force=True)" > $O/build_all.log 2>&1
timeout 600 python tools/tc_err.py 24,40,56 2>&1 | tee $O/tc_err_pad.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "f32 and (24 or 40 or 48 or 56)" > $O/parity_pad.txt 2>&1; tail -2 $O/parity_pad.txt; grep -E "^FAILED" $O/parity_pad.txt | head -5
timeout 1500 python tools/ab.py --variant all="JM_F32TC_ALL=1" --variant all_mtw3="JM_F32TC_ALL=1 JM_F32TC_MTW=3" --variant base= \
  --sizes 24,40,48,56 --dtypes f32 --repeats 100,8 --out $O/ab_pad.jsonl > $O/ab_pad.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/s27/ab_pad.jsonl'):
    d=json.loads(l); print(d['ab'], d['n'], d['repeat'], {k:(d[k].get('frac_pipe'),) for k in ('resident','streaming','auto') if k in d})
PY
