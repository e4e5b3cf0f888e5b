# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
mkdir -p gpurun_out/r02
rm -f gpurun_out/r02/ab_ws40.jsonl gpurun_out/r02/f64_wide.jsonl gpurun_out/r02/f32_wide.jsonl
timeout 900 python tools/ab.py --sizes 33..40 --dtypes f64 --repeats 1,2,4 --out gpurun_out/r02/ab_ws40.jsonl \
  --variant ws40="JM_DMMA_WARP_MAX_STREAM=40" --variant ws40slot="JM_DMMA_WARP_MAX_STREAM=40 JM_DMMA_RING_SLOT=2" \
  --variant base= 2> gpurun_out/r02/ab_ws40.err
python tools/ab.py --table gpurun_out/r02/ab_ws40.jsonl > gpurun_out/r02/ab_ws40.md
timeout 1200 python tools/f32_search.py --dtype f64 --baseline --run tools/f64_candidates_wide.json --out gpurun_out/r02/f64_wide.jsonl 2> gpurun_out/r02/f64_wide.err
python tools/f32_search.py --pick gpurun_out/r02/f64_wide.jsonl > gpurun_out/r02/f64_wide_pick.txt
timeout 1800 python tools/f32_search.py --run tools/f32_candidates_wide.json --out gpurun_out/r02/f32_wide.jsonl 2> gpurun_out/r02/f32_wide.err
python tools/f32_search.py --pick gpurun_out/r02/f32_wide.jsonl > gpurun_out/r02/f32_wide_pick.txt
cat gpurun_out/r02/ab_ws40.md gpurun_out/r02/f64_wide_pick.txt gpurun_out/r02/f32_wide_pick.txt
