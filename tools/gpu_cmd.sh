# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 1500 python tools/stream_sweep.py --sizes $(seq -s, 17 64) --dtypes f32 --repeats 24,100 --gb 0.5 --steps 3 > $O/f32_xover3.jsonl 2> $O/f32_xover3.err
rm -f $O/f64_n17.jsonl
timeout 900 python tools/f32_search.py --dtype f64 --run tools/f64_candidates_n17.json --out $O/f64_n17.jsonl 2> $O/f64_n17.err
python tools/f32_search.py --pick $O/f64_n17.jsonl > $O/f64_n17_pick.txt
cat $O/f64_n17_pick.txt
