# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
set -x
mkdir -p gpurun_out/ncu_r02
CFG_A="2:f64:16777216:1:auto 4:f64:4194304:1:auto 4:f64:4194304:100:auto 4:f32:4194304:1:auto 10:f64:1048576:100:auto 16:f64:1048576:100:auto 17:f64:524288:100:auto 32:f64:131072:100:auto 48:f64:32768:100:auto 64:f64:16384:100:auto 32:f64:65536:1:auto 48:f64:32768:1:auto 64:f64:16384:1:auto"
CFG_B="13:f32:1048576:100:auto 16:f32:1048576:100:auto 16:f32:524288:1:auto 17:f32:524288:100:auto 24:f32:262144:100:auto 32:f32:131072:100:auto 48:f32:65536:100:auto 64:f32:32768:100:auto 17:f32:524288:1:auto 24:f32:262144:1:auto 32:f32:131072:1:auto 48:f32:65536:1:auto 64:f32:32768:1:auto"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -o gpurun_out/ncu_r02/base_a python tools/ncu_configs.py $CFG_A > gpurun_out/ncu_r02/base_a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -o gpurun_out/ncu_r02/base_b python tools/ncu_configs.py $CFG_B > gpurun_out/ncu_r02/base_b.log 2>&1
tail -3 gpurun_out/ncu_r02/base_a.log gpurun_out/ncu_r02/base_b.log
