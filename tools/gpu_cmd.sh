# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
O=gpurun_out/s12; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_guard.py -x -q > $O/test.txt 2>&1; tail -2 $O/test.txt
timeout 1500 python tools/ab.py --variant two="JM_DMMA_STREAM_1BUF=0" --variant one= --sizes 33..64 --dtypes f64 --repeats 1,2,4 --out $O/ab_1buf.jsonl 2> $O/ab.err
python tools/ab.py --table $O/ab_1buf.jsonl > $O/ab_1buf.md; cat $O/ab_1buf.md
