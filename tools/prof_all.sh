# Round profiling batch (run under gpurun from the repo root): bench lines C1-C4 (int8) and C4 fx16,
# the C4 launch list (int8 and fx16), and one ncu --set full capture per config of the query kernels.
set -x
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_r02_$c.json 2> gpurun_out/bench_r02_$c.err
done
timeout 900 python bench.py --config c4 --precision fx16 --steps 5 --warmup 3 > gpurun_out/bench_r02_fx16_c4.json 2> gpurun_out/bench_r02_fx16_c4.err
timeout 300 python tools/prof_query.py --config c4 --reps 2 > gpurun_out/pq_c4.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r02_c4.csv python tools/prof_query.py --config c4 --reps 2 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r02_fx16_c4.csv python tools/prof_fx.py --config c4 > gpurun_out/ncu_launch_fx.log 2>&1
for c in c1 c2 c3 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_kernel|lm_select|coarse_tc_kernel|merge_kernel" -c 5 -o gpurun_out/ncu_r02_$c python tools/prof_query.py --config $c --reps 1 > gpurun_out/ncu_r02_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"fx_coarse_tc_kernel|fx_merge_tc|scan_fx" -c 3 -o gpurun_out/ncu_r02_fx16_c4 python tools/prof_fx.py --config c4 > gpurun_out/ncu_r02_fx16_c4.log 2>&1
ls -la gpurun_out/*r02*
