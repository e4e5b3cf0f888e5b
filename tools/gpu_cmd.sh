timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "f32 or run_many" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep.py --only c3 --sizes 9,12,16 --dtypes f32 --out gpurun_out/sweep_f32p2.jsonl > /dev/null 2>&1; python -c "
import json
for l in open('gpurun_out/sweep_f32p2.jsonl'):
    d=json.loads(l); s=d['specialized']; print(d['n'], d['repeat'], d['regs'], round(s['ms'],2), round(s['tflops'],1), round(s['frac_pipe'],3), round(s['frac_hbm'],3))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -c 1 -o gpurun_out/prof_f32p16b python bench.py --n 16 --dtype f32 --batch 262144 --steps 1 --warmup 1 --no-generic --no-e2e --no-cpu > /dev/null 2>&1
