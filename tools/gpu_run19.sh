# item ring in the fixed-point list-major kernel: parity, timing (dynamic vs static)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fx16.py -x -q -k "not full_size" > gpurun_out/t19.log 2>&1; tail -2 gpurun_out/t19.log
timeout 600 python tools/time_fx.py --configs c2,c4 2>&1 | tail -2
timeout 600 python tools/time_fx.py --configs c2,c4 --opts LM_STATIC=1 2>&1 | tail -2
