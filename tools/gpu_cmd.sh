# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
O=gpurun_out/s10; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -x -q > $O/test.txt 2>&1; tail -2 $O/test.txt
timeout 1500 python tools/ab.py --variant off="JM_RING_SHIFT=0" --variant shift= --sizes 33,35,37,39,41,43,45,47,49,51,53,55,57,59,61,63 --dtypes f64 --repeats 1,2,8 --out $O/ab_ringshift.jsonl 2> $O/ab.err
python tools/ab.py --table $O/ab_ringshift.jsonl > $O/ab_ringshift.md; cat $O/ab_ringshift.md
