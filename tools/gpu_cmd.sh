# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
for C in 8192 4096; do
  JM_BUILD_DEFINES="JM_RING_CHUNK=$C" python -m paper_1904_08555_b200._build --force > /dev/null 2>&1
  python tools/stream_sweep.py --sizes 12,16,20,24,28 --dtypes f64 --repeats 1,2 --gb 0.5 --steps 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('chunk=$C', d['dtype'], d['n'], d['repeat'], round(d['streaming']['frac_hbm'],3), d['kernels']['1']['smem'])
"
  python tools/stream_sweep.py --sizes 17,20,24,32 --dtypes f32 --repeats 1,2 --gb 0.5 --steps 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('chunk=$C', d['dtype'], d['n'], d['repeat'], round(d['streaming']['frac_hbm'],3), d['kernels']['1']['smem'])
"
done
