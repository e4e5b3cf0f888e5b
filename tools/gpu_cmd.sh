timeout 600 python tools/matmul_bench.py --out gpurun_out/matmul_r01.jsonl > gpurun_out/matmul.log 2>&1; python -c "
import json
for l in open('gpurun_out/matmul_r01.jsonl'):
    d=json.loads(l)
    if d['config']=='HBM': print('HBM', d['n'], {k: round(v['frac_hbm'],3) for k,v in d.items() if isinstance(v, dict)}); continue
    s,g=d['specialized'],d['generic']; print(d['n'], d['batch'], 'spec us', round(s['us_per_call'],2), 'graph us', round(s['graph_us_per_call'],2), 'gen us', round(g['us_per_call'],2), 'graph', round(g['graph_us_per_call'],2), 'x', round(d['specialized_speedup'],2), round(d['specialized_speedup_graph'],2), 'lookup ns', round(d['lookup_hit_ns'],1))"
