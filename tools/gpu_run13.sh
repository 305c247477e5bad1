# merge occupancy (launch bounds 6 / 8 per SM) vs default; parity of d2f94f6's untested bits
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse or lm_select or small_configs or lm_topk" > gpurun_out/t13.log 2>&1; tail -2 gpurun_out/t13.log
for lib in "" $PWD/exp/libv3db_m6.so $PWD/exp/libv3db_m8.so; do
  for c in c2 c3 c4; do V3DB_LIB=$lib timeout 300 python tools/time_query.py --config $c --algos 3 2>&1 | tail -1; done
done
