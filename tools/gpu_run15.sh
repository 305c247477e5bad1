# cooperative items kernel; fixed-point merge staged through cp.async: parity, timing
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fx16.py -x -q -k "not full_size" > gpurun_out/t15.log 2>&1; tail -2 gpurun_out/t15.log
for c in c1 c2 c3 c4; do timeout 300 python tools/time_query.py --config c$(echo $c | tr -d c) --algos 3 2>&1 | tail -1; done
timeout 600 python tools/time_fx.py --configs c1,c2,c4 2>&1 | tail -4
timeout 300 python tools/time_fx_coarse.py --config c4 2>&1 | tail -3
