set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse or small_configs or edge" > gpurun_out/t8.log 2>&1; tail -2 gpurun_out/t8.log
for c in c3 c4 c2; do timeout 200 python tools/time_query.py --config $c --algos 3 --opts COARSE_KEYS=2,COARSE_KEYS=4 2>&1 | tail -3; done
