timeout 1800 python tools/work_check.py --out gpurun_out/work_check2.jsonl > gpurun_out/work_check2.log 2>&1; echo rc=$?
