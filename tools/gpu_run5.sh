# fixed-point coarse on the tensor cores: parity tests, timing (C4, C2), ncu of the new kernels
set -x
timeout 1200 python -m pytest tests/test_gpu_fx16.py -x -q -k "not full_size" > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
timeout 600 python tools/time_fx.py --configs c2,c4 --reps 3 > gpurun_out/tfx.log 2>&1; cat gpurun_out/tfx.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"fx_coarse_tc_kernel|fx_merge_tc" -c 2 -o gpurun_out/ncu_fx_v1 python tools/prof_fx.py --config c4 > gpurun_out/ncu_fx_v1.log 2>&1; tail -2 gpurun_out/ncu_fx_v1.log
