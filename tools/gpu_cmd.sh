# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q -x -k "f32" 2>&1 | tail -4 > $O/gputest_f32.txt
rm -f $O/f32s_search_v3.jsonl $O/f64_regcap.jsonl
timeout 2400 python tools/f32_search.py --stream --baseline --run tools/f32s_candidates_v3.json --out $O/f32s_search_v3.jsonl 2> $O/f32s_search_v3.err
python tools/f32_search.py --pick $O/f32s_search_v3.jsonl --margin 0.01 > $O/f32s_search_v3_pick.txt
timeout 1200 python tools/f32_search.py --dtype f64 --run tools/f64_candidates_regcap.json --out $O/f64_regcap.jsonl 2> $O/f64_regcap.err
python tools/f32_search.py --pick $O/f64_regcap.jsonl > $O/f64_regcap_pick.txt
cat $O/gputest_f32.txt $O/f32s_search_v3_pick.txt $O/f64_regcap_pick.txt
