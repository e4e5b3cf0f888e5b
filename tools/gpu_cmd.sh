# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# tensor-core FP32 kind for n = 48, 64 (warps split the rows) and the warps-per-matrix choice; error, parity, A/B, crossover
O=gpurun_out/s23; mkdir -p $O
JM_BUILD_DEFINES="JM_F32TC_MAXN=64" python -c "import paper_1904_08555_b200._build as b; b.build(force=True)" > $O/build64.log 2>&1
timeout 600 python tools/tc_err.py 48,64 2>&1 | tee $O/tc_err_48_64.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "f32 and (48 or 64)" > $O/parity64.txt 2>&1; tail -2 $O/parity64.txt
timeout 900 python tools/stream_sweep.py --sizes 48,64 --dtypes f32 --repeats 1,2,3,4,6,8,100 --out $O/xover64.jsonl > /dev/null 2> $O/xover64.err
timeout 1500 python tools/ab.py --variant mtw1="JM_F32TC_MAXN=64 JM_F32TC_MTW=1" --variant mtw2="JM_F32TC_MAXN=64 JM_F32TC_MTW=2" \
  --variant ffma="JM_F32TC_MAXN=32" --variant tc64="JM_F32TC_MAXN=64" --sizes 32,48,64 --dtypes f32 --repeats 100,8 --out $O/ab64.jsonl > $O/ab64.log 2>&1
python - <<'PY'
import json
for f in ('xover64', 'ab64'):
    for l in open(f'gpurun_out/s23/{f}.jsonl'):
        d=json.loads(l); print(f, d.get('ab',''), d['n'], d['repeat'], {k:(d[k].get('frac_pipe'), d[k].get('frac_hbm')) for k in ('resident','streaming','auto') if k in d})
PY
