timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "f64" > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --only c3 --sizes 24,25,28,32 --dtypes f64 --out gpurun_out/sweep_w1.jsonl > /dev/null 2>&1; python -c "
import json
for l in open('gpurun_out/sweep_w1.jsonl'):
    d=json.loads(l)
    s=d['specialized']; print(d['n'], d['dtype'], d['repeat'], d['tile'], d['regs'], d['smem'], round(s['ms'],2), round(s['tflops'],2), 'pipe', round(s['frac_pipe'],3), 'hbm', round(s['frac_hbm'],3))"
