timeout 900 python -m pytest tests/test_gpu_mass.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python tools/mass_bench.py --out gpurun_out/mass_r01.jsonl > /dev/null 2>&1; python -c "
import json
for l in open('gpurun_out/mass_r01.jsonl'):
    d=json.loads(l); s,g=d['specialized'],d['generic']
    print(d['dofs'], d['quads'], d['elements'], 'spec ms', round(s['ms'],4), 'hbm', round(s['frac_hbm'],3), 'gen ms', round(g['ms'],4), 'x', round(d['specialized_speedup'],2))"
