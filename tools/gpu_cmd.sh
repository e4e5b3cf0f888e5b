# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
SIZES=$(seq -s, 26 64)
python tools/stream_sweep.py --sizes $SIZES --dtypes f32 --repeats 100 --gb 0.25 --steps 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('default', d['n'], round(d['resident']['frac_pipe'],3), d['kernels']['0']['regs'], d['kernels']['0']['local'])
"
for shape in "7 12" "7 20" "6 24" "4 32" "8 8" "8 20" "3 16" "6 28"; do
  set -- $shape
  JM_BUILD_DEFINES="JM_F32_TILE_RA=$1 JM_F32_TILE_CB=$2" python -m paper_1904_08555_b200._build --force > /dev/null 2>&1
  python tools/stream_sweep.py --sizes $SIZES --dtypes f32 --repeats 100 --gb 0.25 --steps 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('ra=$1 cb=$2', d['n'], round(d['resident']['frac_pipe'],3), d['kernels']['0']['regs'], d['kernels']['0']['local'])
"
done
