# profile batch: C4 main kernel (NT 64) and C3 coarse kernel + merge
set -x
timeout 300 python tools/prof_query.py --config c4 --reps 1 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_kernel|lm_scan_items|pair_scatter" -c 3 -o gpurun_out/ncu_c4_v9 python tools/prof_query.py --config c4 --reps 1 > gpurun_out/ncu_c4_v9.log 2>&1
timeout 300 python tools/prof_query.py --config c3 --reps 1 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"coarse_tc_kernel|merge_kernel|lm_select" -c 3 -o gpurun_out/ncu_c3_v9 python tools/prof_query.py --config c3 --reps 1 > gpurun_out/ncu_c3_v9.log 2>&1
ls -la gpurun_out/*v9*
