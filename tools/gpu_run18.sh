# dynamic item scheduling in lm_kernel: parity, timing (dynamic vs static), per-CTA finish times
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lm or small_configs or edge or ragged" > gpurun_out/t18.log 2>&1; tail -2 gpurun_out/t18.log
for c in c1 c2 c3 c4; do timeout 300 python tools/time_query.py --config $c --algos 3 --reps 9 --opts LM_STATIC=1 2>&1 | tail -2; done
for c in c4 c2 c3 c1; do V3DB_LIB=$PWD/exp/libv3db_times.so timeout 200 python tools/lm_times.py --config $c 2>&1 | tail -1; done
