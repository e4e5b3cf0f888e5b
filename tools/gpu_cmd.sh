# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
O=gpurun_out/s8; mkdir -p $O
PLAN=paper_1904_08555_b200/csrc/kernels/jm_plan.h
cp $PLAN $O/jm_plan.h.orig
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 3000 python tools/f32_search.py --run tools/f32_candidates_nb2.json --out $O/f32_nb2.jsonl 2> $O/f32_nb2.err
python tools/f32_search.py --pick $O/f32_nb2.jsonl > $O/f32_nb2_pick.txt
cp $O/jm_plan.h.orig $PLAN
cat $O/f32_nb2_pick.txt
