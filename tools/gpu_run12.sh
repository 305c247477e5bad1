# complete-block coarse path (KB >= nprobe), batched / smem-aggregated pair scatter: parity, full-size C1/C2, timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t12.log 2>&1; tail -3 gpurun_out/t12.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1 or c2" > gpurun_out/t12f.log 2>&1; tail -3 gpurun_out/t12f.log
for c in c1 c2 c3 c4; do timeout 300 python tools/time_query.py --config $c --algos 3 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c1.csv python tools/prof_query.py --config c1 --reps 2 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c1.csv
