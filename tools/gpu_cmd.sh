# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 2700 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/gputest_full5.txt
rm -f $O/ab_rows.jsonl $O/f32s_search.jsonl
timeout 900 python tools/ab.py --sizes 16,20,24,28,32,36,40,44,48,56,64 --dtypes f32 --repeats 1,2,4 --out $O/ab_rows.jsonl \
  --variant norows="JM_F32T_RING_ROWS=0" --variant rows= 2> $O/ab_rows.err
python tools/ab.py --table $O/ab_rows.jsonl > $O/ab_rows.md
timeout 1800 python tools/f32_search.py --stream --baseline --run tools/f32s_candidates.json --out $O/f32s_search.jsonl 2> $O/f32s_search.err
python tools/f32_search.py --pick $O/f32s_search.jsonl --margin 0.01 > $O/f32s_search_pick.txt
tail -3 $O/gputest_full5.txt; cat $O/ab_rows.md $O/f32s_search_pick.txt
