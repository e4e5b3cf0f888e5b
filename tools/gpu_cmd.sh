./tools/microbench/peaks | grep -E "dmma|dfma"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "f64" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --only c3 --sizes 8,16,24,32,40,48,64 --dtypes f64 --repeats 100 --out gpurun_out/sweep_dmmac.jsonl > /dev/null 2>&1; python -c "
import json
for l in open('gpurun_out/sweep_dmmac.jsonl'):
    d=json.loads(l)
    s=d['specialized']; print(d['n'], d['dtype'], d['repeat'], d['tile'], d['regs'], round(s['ms'],2), round(s['tflops'],2), 'pipe', round(s['frac_pipe'],3))"
python bench.py --steps 30 --no-e2e --no-cpu --no-generic | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['kernel'])"
