# Step-5 candidate loads in flight (kSwH) and the flagged-query list: parity, then per-kernel times
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fx16.py -x -q -k "not full_size" > gpurun_out/t10.log 2>&1; tail -3 gpurun_out/t10.log
for lib in "" $PWD/exp/libv3db_fast8.so $PWD/exp/libv3db_h8.so; do
  for c in c1 c2 c3 c4; do V3DB_LIB=$lib timeout 300 python tools/time_query.py --config $c --algos 3 2>&1 | tail -1; done
done
