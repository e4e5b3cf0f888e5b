# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
O=gpurun_out/s6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -x -q > $O/test.txt 2>&1; tail -2 $O/test.txt
timeout 1200 python tools/ab.py --variant off="JM_F32T_PSHIFT=0" --variant pshift= --sizes 17,19,21,23,25,27,29,31,33,35,37,39,41,43,45,47,49,51,53,55,57,59,61,63 --dtypes f32 --repeats 1,2 --out $O/ab_pshift.jsonl 2> $O/ab.err
python tools/ab.py --table $O/ab_pshift.jsonl > $O/ab_pshift.md; cat $O/ab_pshift.md
