# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# tensor-core FP32 kind with the expansion check (exact FP32 path when max|m| > 1/(2cn)): paper-init error, GPU suite, smoke, perf
O=gpurun_out/s34; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/tc_diag_paper.py 2>&1 | tee $O/diag_paper.txt
timeout 2000 python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1; tail -2 $O/gputest.txt; grep -E "^FAILED" $O/gputest.txt | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python tools/stream_sweep.py --sizes 32,40,47,48,56,63,64 --dtypes f32 --repeats 100 --out $O/tc_check.jsonl > /dev/null 2> $O/tc_check.err
python - <<'PY'
import json
for l in open('gpurun_out/s34/tc_check.jsonl'):
    d=json.loads(l); print(d['n'], d['repeat'], d['auto']['frac_pipe'])
PY
