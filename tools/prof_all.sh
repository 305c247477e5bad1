# Round profiling batch (run under gpurun from the repo root): bench lines C1-C4 (int8) and C4 fx16,
# the C4 launch lists (int8, fx16), one ncu --set full capture per config summarised ON THE BOX
# (reports are deleted afterwards: gpurun_out must stay under 64 MiB), the DRAM traffic of the
# dominant kernels, and the tcgen05 issue microbenchmark.
set -x
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_r02_$c.json 2> gpurun_out/bench_r02_$c.err
done
timeout 900 python bench.py --config c4 --precision fx16 --steps 5 --warmup 3 > gpurun_out/bench_r02_fx16_c4.json 2> gpurun_out/bench_r02_fx16_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r02_c4.csv python tools/prof_query.py --config c4 --reps 2 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r02_fx16_c4.csv python tools/prof_fx.py --config c4 > gpurun_out/ncu_launch_fx.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_r02_c4.csv > gpurun_out/launches_r02_c4.md
python tools/ncu_summary.py launches gpurun_out/launches_r02_fx16_c4.csv > gpurun_out/launches_r02_fx16_c4.md
for c in c1 c2 c3 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_kernel|lm_select|coarse_tc_kernel|merge_kernel" -c 5 -o gpurun_out/ncu_r02_$c python tools/prof_query.py --config $c --reps 1 > gpurun_out/ncu_r02_$c.log 2>&1
  python tools/ncu_summary.py rep gpurun_out/ncu_r02_$c.ncu-rep > gpurun_out/ncu_r02_$c.md
  python tools/ncu_traffic.py gpurun_out/ncu_r02_$c.ncu-rep lm_kernel >> gpurun_out/traffic.txt
done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"fx_coarse_tc_kernel|fx_merge_tc|lm_fx_kernel|lm_select" -c 4 -o gpurun_out/ncu_r02_fx16_c4 python tools/prof_fx.py --config c4 > gpurun_out/ncu_r02_fx16_c4.log 2>&1
python tools/ncu_summary.py rep gpurun_out/ncu_r02_fx16_c4.ncu-rep > gpurun_out/ncu_r02_fx16_c4.md
python tools/ncu_traffic.py gpurun_out/ncu_r02_fx16_c4.ncu-rep lm_fx_kernel >> gpurun_out/traffic.txt
./tools/tc_bench_n > gpurun_out/tc_bench_n.log 2>&1
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/
