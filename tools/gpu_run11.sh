# hot spots of lm_kernel and the Step-5 warp kernel at C4, the C1 kernels (after cc0712d); summarised on the box
set -x
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_kernel|lm_select_warp|merge_kernel|lm_scan_items|pair_scatter" -c 5 -o /tmp/lm_c4 python tools/prof_query.py --config c4 --reps 1 > gpurun_out/lm_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 12 -o /tmp/lm_c1 python tools/prof_query.py --config c1 --reps 1 > gpurun_out/lm_c1.log 2>&1
for k in lm_kernel lm_select_warp merge_kernel lm_scan_items pair_scatter; do python tools/ncu_hot.py /tmp/lm_c4.ncu-rep $k 60 > gpurun_out/hot_c4_$k.txt 2>&1; done
python tools/ncu_summary.py rep /tmp/lm_c4.ncu-rep > gpurun_out/sum_c4.md 2>&1
python tools/ncu_summary.py rep /tmp/lm_c1.ncu-rep > gpurun_out/sum_c1.md 2>&1
cp /tmp/lm_c4.ncu-rep gpurun_out/ 
ls -la gpurun_out
