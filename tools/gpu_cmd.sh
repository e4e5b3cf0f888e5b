# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
O=gpurun_out/s11; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python tools/stream_sweep.py --sizes 2..64 --dtypes f64 --repeats 1,100 --gb 0.5 --out $O/all_n_f64.jsonl > /dev/null 2> $O/all_n.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -o $O/late_kinds python tools/ncu_configs.py 49:f64:26030:1:streaming 39:f64:41091:1:streaming 63:f32:31494:1:streaming > $O/ncu_late.log 2>&1
ncu -i $O/late_kinds.ncu-rep --page raw --csv > $O/late_kinds_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/late_kinds.ncu-rep --algo 49,f64,26030,1 39,f64,41091,1 63,f32,31494,1 > $O/late_kinds.md 2> $O/late_kinds.err
cat $O/late_kinds.md
