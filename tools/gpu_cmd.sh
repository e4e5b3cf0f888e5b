# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
for mb in 16 32 64 128 256; do
  JIT_MAT_HOST_CHUNK_MB=$mb timeout 600 python bench.py --no-cpu --no-generic --steps 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunk_mb=$mb', d['e2e']['value'], d['e2e']['ms_per_step'])"
done
