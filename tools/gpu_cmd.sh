timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "f32 or F32" 2>&1 | tail -4
timeout 900 python tools/sweep.py --only c3 --sizes 17,20,24,25,28,32,33,36,40,41,44,48,49,52,56,57,60,63,64 --dtypes f32 --repeats 1,100 --out gpurun_out/sweep_f32v4.jsonl > gpurun_out/sweep_f32v4.log 2>&1; echo rc=$?
python tools/make_report.py gpurun_out/sweep_f32v4.jsonl | grep "^| [0-9]"
