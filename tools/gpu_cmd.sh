# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# final numbers of the committed build: FP32 all-n sweep, C3 FP32, ncu of the tensor-core kinds, C2 bench
O=gpurun_out/s35; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python tools/stream_sweep.py --sizes 2..64 --dtypes f32 --repeats 1,100 --gb 0.5 --out $O/all_n_f32.jsonl > /dev/null 2> $O/all_n.err
timeout 900 python tools/sweep.py --only c3 --dtypes f32 --out $O/sweep_c3_f32.jsonl > $O/sweep_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -o $O/prof_f32tc_final \
  python tools/ncu_configs.py 32:f32:65536:100:resident 47:f32:40000:100:resident 48:f32:40000:100:resident 64:f32:30517:100:resident > $O/ncu.log 2>&1; tail -1 $O/ncu.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 150 $O/bench_c2.json
