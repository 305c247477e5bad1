# coarse merge restructure check + a kept C4 capture for per-line analysis
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse or small_configs" > gpurun_out/t17.log 2>&1; tail -2 gpurun_out/t17.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_kernel|lm_select_warp|merge_kernel" -c 3 -o gpurun_out/c4_lines python tools/prof_query.py --config c4 --reps 1 > gpurun_out/c4_lines.log 2>&1
ls -la gpurun_out/
