for G in 2 4; do
JM_BUILD_DEFINES="JM_F64_ROWS_MAX=15 JM_F64P_G=$G" python -m paper_1904_08555_b200._build --force > /dev/null 2>&1; echo build rc=$?
python tools/stream_sweep.py --sizes 11,12,13,15 --dtypes f64 --repeats 1,100 --gb 1 --steps 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('G=$G', d['n'], d['repeat'], 'pipe %.3f hbm %.2f'%(d['resident']['frac_pipe'], d['resident']['frac_hbm']), d['kernels']['0'])
"
done
