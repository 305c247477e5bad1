# Step-5 hot spots at C3 (CTA kernel) and C4 (warp kernel), plus the per-kernel times of C1-C4 at HEAD.
set -x
for c in c1 c2 c3 c4; do timeout 300 python tools/time_query.py --config $c --algos 3 2>&1 | tail -2; done
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_select_fast|lm_select_warp|merge_kernel" -c 3 -o gpurun_out/sel_c3 python tools/prof_query.py --config c3 --reps 1 > gpurun_out/sel_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_select_warp|merge_kernel" -c 2 -o gpurun_out/sel_c4 python tools/prof_query.py --config c4 --reps 1 > gpurun_out/sel_c4.log 2>&1
ls -la gpurun_out
