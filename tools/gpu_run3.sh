# option sweep on the list-major scan (C4, C2)
set -x
for c in c4 c2; do timeout 300 python tools/time_query.py --config $c --algos 3 --opts LM_NT=64,LM_NT=128,LM_NT=256 > gpurun_out/tq3_$c.log 2>&1; cat gpurun_out/tq3_$c.log; done
