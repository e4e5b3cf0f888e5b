# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
for R in 1 2 3; do
  JM_BUILD_DEFINES="JM_TPMS_ROWS=$R" python -m paper_1904_08555_b200._build --force > /dev/null 2>&1
  python tools/stream_sweep.py --sizes 9,10 --dtypes f64 --repeats 100 --gb 0.5 --steps 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('rows=$R', d['dtype'], d['n'], round(d['resident']['frac_pipe'],3))
"
  python tools/stream_sweep.py --sizes 12,13,14 --dtypes f32 --repeats 100 --gb 0.5 --steps 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('rows=$R', d['dtype'], d['n'], round(d['resident']['frac_pipe'],3))
"
done
