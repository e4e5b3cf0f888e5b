# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
rm -f $O/ab_rt.jsonl $O/f32s_search_v2.jsonl
timeout 900 python tools/ab.py --sizes 33..56 --dtypes f64 --repeats 1,2 --out $O/ab_rt.jsonl \
  --variant rt2="JM_DMMA_RT_LARGE=2" --variant rt3="JM_DMMA_RT_LARGE=3" --variant base= 2> $O/ab_rt.err
python tools/ab.py --table $O/ab_rt.jsonl > $O/ab_rt.md
timeout 2700 python tools/f32_search.py --stream --baseline --run tools/f32s_candidates_v2.json --out $O/f32s_search_v2.jsonl 2> $O/f32s_search_v2.err
python tools/f32_search.py --pick $O/f32s_search_v2.jsonl --margin 0.01 > $O/f32s_search_v2_pick.txt
cat $O/ab_rt.md $O/f32s_search_v2_pick.txt
