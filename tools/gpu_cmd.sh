# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
S=11,12,13,14,17,18,19,20,21,25,26,27,28,33,34,35,36,41,42,43,44,49,50,51,52,57,58,59,60
rm -f gpurun_out/r02/ab_dmma.jsonl
timeout 1500 python tools/ab.py --sizes $S --dtypes f64 --repeats 1,100 --out gpurun_out/r02/ab_dmma.jsonl \
  --variant old="JM_DMMA_KCOMPACT=0 JM_DMMA_BORDER_MAX=2" \
  --variant cmp_b2="JM_DMMA_BORDER_MAX=2" \
  --variant b4_nocmp="JM_DMMA_KCOMPACT=0" \
  --variant bmin8="JM_DMMA_BORDER_MIN=8" \
  --variant f64t="JM_F64T_ON=1" \
  --variant new= 2> gpurun_out/r02/ab_dmma.err
python tools/ab.py --table gpurun_out/r02/ab_dmma.jsonl > gpurun_out/r02/ab_dmma.md
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02/gputest_full2.txt
cat gpurun_out/r02/ab_dmma.md gpurun_out/r02/gputest_full2.txt
