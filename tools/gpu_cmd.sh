for shape in "6 8" "4 8" "5 12" "9 8" "3 12" "6 4"; do
  set -- $shape
  JM_BUILD_DEFINES="JM_F32_TILE_RA=$1 JM_F32_TILE_CB=$2" python -m paper_1904_08555_b200._build --force > /dev/null 2>&1
  python tools/stream_sweep.py --sizes 17,18,20,21,25,26 --dtypes f32 --repeats 100 --gb 0.5 --steps 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('ra=$1 cb=$2', d['n'], round(d['resident']['frac_pipe'],3), d['kernels']['0']['regs'], d['kernels']['0']['local'])
"
done
