# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 2700 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/gputest_full8.txt
ALLN=$(seq -s, 2 64)
rm -f $O/all_n8.jsonl $O/f32_wpc.jsonl
timeout 1200 python tools/stream_sweep.py --sizes $ALLN --dtypes f64,f32 --repeats 1,100 --gb 0.5 --steps 5 --out $O/all_n8.jsonl > /dev/null 2> $O/all_n8.err
timeout 2400 python tools/f32_search.py --run tools/f32_candidates_wpc.json --out $O/f32_wpc.jsonl 2> $O/f32_wpc.err
python tools/f32_search.py --pick $O/f32_wpc.jsonl > $O/f32_wpc_pick.txt
tail -3 $O/gputest_full8.txt; cat $O/f32_wpc_pick.txt
