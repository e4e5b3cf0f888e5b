for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1; echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|sanitize_run:" gpurun_out/sanitize_$t.log | tail -4
done
