# coalesced items kernel: parity (list-major + fixed point), timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fx16.py -x -q -k "lm or small_configs or fx_end_to_end or fx_list_major or edge" > gpurun_out/t14.log 2>&1; tail -2 gpurun_out/t14.log
for c in c1 c2 c3 c4; do timeout 300 python tools/time_query.py --config $c --algos 3 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c4.csv python tools/prof_query.py --config c4 --reps 2 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c4.csv
