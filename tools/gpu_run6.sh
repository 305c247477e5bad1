# fixed-point list-major scan: parity tests, timing (C2, C4), ncu of lm_fx_kernel
set -x
timeout 1200 python -m pytest tests/test_gpu_fx16.py -x -q -k "not full_size" > gpurun_out/t6.log 2>&1; tail -3 gpurun_out/t6.log
timeout 600 python tools/time_fx.py --configs c2,c4 --reps 3 > gpurun_out/tfx6.log 2>&1; cat gpurun_out/tfx6.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_fx_kernel|lm_select" -c 2 -o gpurun_out/ncu_fxlm_v1 python tools/prof_fx.py --config c4 > gpurun_out/ncu_fxlm_v1.log 2>&1; tail -2 gpurun_out/ncu_fxlm_v1.log
./tools/tc_bench_n > gpurun_out/tc_bench_n.log 2>&1; cat gpurun_out/tc_bench_n.log
