# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
O=gpurun_out/s15; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -x -q -k "f32 or float" > $O/test.txt 2>&1; tail -2 $O/test.txt
timeout 900 python tools/ab.py --tool mass_bench --variant thread_pf="JM_MASS_DMMA=-1" --variant dmma="JM_MASS_DMMA=1" --variant default= --out $O/mass_tab.jsonl 2> $O/mass_tab.err
python tools/mass_report.py $O/mass_tab.jsonl --pick thread_pf,dmma > $O/mass_tab.md; tail -4 $O/mass_tab.md
timeout 1500 python tools/stream_sweep.py --sizes 2..64 --dtypes f32 --repeats 1,100 --gb 0.5 --out $O/all_n_f32.jsonl > /dev/null 2> $O/all_n.err
echo done
