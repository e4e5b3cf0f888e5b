timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --only c3 --sizes 32,40,48,64 --dtypes f64 --out gpurun_out/sweep_mb1.jsonl > /dev/null 2>&1; python -c "
import json
for l in open('gpurun_out/sweep_mb1.jsonl'):
    d=json.loads(l)
    s=d['specialized']; g=d['generic']; print(d['n'], d['dtype'], d['repeat'], d['tile'], d['regs'], round(s['ms'],2), round(s['tflops'],1), 'pipe', round(s['frac_pipe'],3), 'hbm', round(s['frac_hbm'],3), 'x', round(d['speedup'],2))"
