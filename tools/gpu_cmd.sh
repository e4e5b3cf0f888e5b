# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02/gputest_full_a.txt
timeout 900 python tools/stream_sweep.py --sizes 16,17,20,24,28,32,40,48,56,64 --dtypes f32 --repeats 1,2,4,8,16 --gb 0.5 --steps 5 > gpurun_out/r02/f32t_lowr.jsonl 2>gpurun_out/r02/f32t_lowr.err
rm -f gpurun_out/r02/f64_search.jsonl
timeout 2400 python tools/f32_search.py --dtype f64 --baseline --run tools/f64_candidates.json --out gpurun_out/r02/f64_search.jsonl 2> gpurun_out/r02/f64_search.err
python tools/f32_search.py --pick gpurun_out/r02/f64_search.jsonl --margin 0.02 > gpurun_out/r02/f64_search_pick.txt
cat gpurun_out/r02/gputest_full_a.txt gpurun_out/r02/f64_search_pick.txt
