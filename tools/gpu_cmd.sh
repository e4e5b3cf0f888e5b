# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
O=gpurun_out/s14; mkdir -p $O
PLAN=paper_1904_08555_b200/csrc/kernels/jm_plan.h
cp $PLAN $O/jm_plan.h.orig
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_mass.py tests/test_gpu_guard.py -x -q > $O/test.txt 2>&1; tail -2 $O/test.txt
timeout 900 python tools/ab.py --tool mass_bench --variant sync="JM_MASS_PF=0" --variant pf= --out $O/mass_pf.jsonl 2> $O/mass_pf.err
python tools/mass_report.py $O/mass_pf.jsonl --pick sync,pf > $O/mass_pf.md; cat $O/mass_pf.md | tail -4
timeout 2400 python tools/f32_search.py --stream --run tools/f32s_candidates_nb.json --out $O/f32s_nb.jsonl 2> $O/f32s_nb.err
python tools/f32_search.py --pick $O/f32s_nb.jsonl > $O/f32s_nb_pick.txt
cp $O/jm_plan.h.orig $PLAN
