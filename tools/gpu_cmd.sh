# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q -x -k "f32" 2>&1 | tail -4 > $O/gputest_f32b.txt
timeout 600 python tools/stream_sweep.py --sizes 16 --dtypes f32 --repeats 1,2,4,8,12,24,100 --gb 0.5 > $O/f32_n16_xover.jsonl 2> /dev/null
rm -f $O/f32_n16_res.jsonl
export JM_BUILD_DEFINES="JM_F32P_MAX=15"
timeout 1200 python tools/f32_search.py --run tools/f32_candidates_n16.json --out $O/f32_n16_res.jsonl 2> $O/f32_n16_res.err
python tools/f32_search.py --pick $O/f32_n16_res.jsonl > $O/f32_n16_res_pick.txt
cat $O/gputest_f32b.txt $O/f32_n16_res_pick.txt
