timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --only c3 --sizes 8,13,16,24,32,40,48,56,64 --dtypes f64 --repeats 100 --out gpurun_out/sweep_addr.jsonl > /dev/null 2>&1; python -c "
import json
for l in open('gpurun_out/sweep_addr.jsonl'):
    d=json.loads(l)
    s=d['specialized']; print(d['n'], d['dtype'], d['repeat'], d['tile'], d['regs'], d['smem'], round(s['ms'],2), round(s['tflops'],2), 'pipe', round(s['frac_pipe'],3))"
python bench.py --steps 30 --no-e2e --no-cpu --no-generic | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['kernel'])"
