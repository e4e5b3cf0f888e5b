# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
O=gpurun_out/s5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/mass_bench.py --out $O/mass_f7.jsonl > /dev/null 2> $O/mass_f7.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mass -o $O/mass python tools/mass_ncu.py 8:8 8:4 6:6 4:4 > $O/mass_ncu.log 2>&1
ncu -i $O/mass.ncu-rep --page raw --csv > $O/mass_raw.csv 2>/dev/null
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py > $O/san_$t.txt 2>&1; echo "$t rc=$?" >> $O/san_summary.txt
  tail -3 $O/san_$t.txt >> $O/san_summary.txt
done
cat $O/san_summary.txt
