# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 -o gpurun_out/prof_c2_final python bench.py --steps 2 --warmup 3 --no-generic --no-e2e --no-cpu > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2_final.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo rc=$?
