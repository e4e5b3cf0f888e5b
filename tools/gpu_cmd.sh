# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -x -q -k "f32 or overflow" 2>&1 | tail -5 > gpurun_out/r02/f32t_tests_c.txt
rm -f gpurun_out/r02/f32_search_hard.jsonl
timeout 2400 python tools/f32_search.py --run tools/f32_candidates_hard.json --out gpurun_out/r02/f32_search_hard.jsonl 2> gpurun_out/r02/f32_search_hard.err
python tools/f32_search.py --pick gpurun_out/r02/f32_search_hard.jsonl > gpurun_out/r02/f32_search_hard_pick.txt
cat gpurun_out/r02/f32t_tests_c.txt gpurun_out/r02/f32_search_hard_pick.txt
