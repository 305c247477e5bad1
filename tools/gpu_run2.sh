# quick iteration batch: targeted parity tests, per-step timing of C1-C4, C4 launch list + ncu of the
# Step 2 / Step 5 kernels
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse or lm or small_configs or edge or ragged" > gpurun_out/t2.log 2>&1; tail -3 gpurun_out/t2.log
for c in c1 c2 c3 c4; do timeout 300 python tools/time_query.py --config $c --algos 3 --opts LM_DECODE=1 > gpurun_out/tq_$c.log 2>&1; cat gpurun_out/tq_$c.log; done
timeout 300 python tools/prof_query.py --config c4 --reps 2 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c4_v12.csv python tools/prof_query.py --config c4 --reps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_kernel|merge_kernel|lm_scan_items" -c 3 -o gpurun_out/ncu_c4_v12 python tools/prof_query.py --config c4 --reps 1 > gpurun_out/ncu_c4_v12.log 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/bench_c4_v12.json 2> gpurun_out/bench_c4_v12.err; cat gpurun_out/bench_c4_v12.json
timeout 300 python tools/time_query.py --config c3 --algos 3 > gpurun_out/tq_c3b.log 2>&1; cat gpurun_out/tq_c3b.log
