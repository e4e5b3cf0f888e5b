# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 2700 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/gputest_full11.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke11.txt 2>&1
rm -f $O/f32_n12_15.jsonl
export JM_BUILD_DEFINES="JM_F32P_MAX=11 JM_F32_TPMS_MAX=11"
timeout 1500 python tools/f32_search.py --run tools/f32_candidates_n12_15.json --out $O/f32_n12_15.jsonl 2> $O/f32_n12_15.err
python tools/f32_search.py --pick $O/f32_n12_15.jsonl > $O/f32_n12_15_pick.txt
tail -3 $O/gputest_full11.txt; tail -3 $O/smoke11.txt; cat $O/f32_n12_15_pick.txt
