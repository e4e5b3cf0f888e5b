python tools/stream_sweep.py --sizes 9,12,13,16,20,24 --dtypes f64 --repeats 1,2,3,4 --gb 2 --steps 3 > gpurun_out/lowr_s2.jsonl 2>&1
JM_BUILD_DEFINES="JM_RING_S=3" python -m paper_1904_08555_b200._build --force > /dev/null 2>&1; echo build rc=$?
python tools/stream_sweep.py --sizes 9,12,13,16,20,24 --dtypes f64 --repeats 1,2,3,4 --gb 2 --steps 3 > gpurun_out/lowr_s3.jsonl 2>&1
JM_BUILD_DEFINES="JM_RING_CHUNK=16384" python -m paper_1904_08555_b200._build --force > /dev/null 2>&1; echo build rc=$?
python tools/stream_sweep.py --sizes 9,12,13,16,20,24 --dtypes f64 --repeats 1,2,3,4 --gb 2 --steps 3 > gpurun_out/lowr_c16.jsonl 2>&1
