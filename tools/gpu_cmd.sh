mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1800 compute-sanitizer --tool $tool python tools/sanitize_run.py > gpurun_out/san/$tool.txt 2>&1; echo $tool rc=$?; tail -1 gpurun_out/san/$tool.txt
done
