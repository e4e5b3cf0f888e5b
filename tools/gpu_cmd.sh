# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02 gpurun_out/r02/san
O=gpurun_out/r02
timeout 2700 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/gputest_full10.txt
rm -f $O/all_n10.jsonl
timeout 1200 python tools/stream_sweep.py --sizes $(seq -s, 2 64) --dtypes f64,f32 --repeats 1,100 --gb 0.5 --steps 5 --out $O/all_n10.jsonl > /dev/null 2> $O/all_n10.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/san/$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/san/summary.txt
  tail -3 $O/san/$tool.txt >> $O/san/summary.txt
done
tail -3 $O/gputest_full10.txt; cat $O/san/summary.txt
