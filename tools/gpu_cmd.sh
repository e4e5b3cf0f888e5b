# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 2700 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/gputest_full7.txt
rm -f $O/ab_pvec.jsonl $O/ab_skew.jsonl $O/f32_xover.jsonl
timeout 1500 python tools/ab.py --sizes 17..64 --dtypes f32 --repeats 1,100 --out $O/ab_pvec.jsonl \
  --variant nopvec="JM_F32T_PVEC=0" --variant pvec= 2> $O/ab_pvec.err
python tools/ab.py --table $O/ab_pvec.jsonl > $O/ab_pvec.md
timeout 600 python tools/ab.py --sizes 12..16 --dtypes f32 --repeats 1,100 --out $O/ab_skew.jsonl \
  --variant noskew="JM_F32P_PAIR_SKEW=0" --variant skew= 2> $O/ab_skew.err
python tools/ab.py --table $O/ab_skew.jsonl > $O/ab_skew.md
timeout 900 python tools/stream_sweep.py --sizes 17,20,24,28,32,33,40,48,56,64 --dtypes f32 --repeats 2,3,4,6,8 --gb 0.5 > $O/f32_xover.jsonl 2> $O/f32_xover.err
tail -3 $O/gputest_full7.txt; cat $O/ab_skew.md; head -52 $O/ab_pvec.md
