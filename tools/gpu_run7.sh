set -x
timeout 1200 python -m pytest tests/test_gpu_fx16.py -x -q -k "not full_size" > gpurun_out/t7.log 2>&1; tail -3 gpurun_out/t7.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lm or coarse or small_configs" > gpurun_out/t7b.log 2>&1; tail -3 gpurun_out/t7b.log
timeout 200 python tools/time_query.py --config c4 --algos 3 --opts LM_NT=128,LM_NT=256 > gpurun_out/tq7.log 2>&1; cat gpurun_out/tq7.log
timeout 600 python tools/time_fx.py --configs c4 --reps 3 > gpurun_out/tfx7.log 2>&1; cat gpurun_out/tfx7.log
