# HEAD validation (run under gpurun from the repo root): the whole GPU suite, smoke, then the round's profiling batch (tools/prof_all.sh)
set -x
mkdir -p gpurun_out
(time timeout 3000 python -m pytest tests -m gpu -x -q) > gpurun_out/t16.log 2>&1; tail -3 gpurun_out/t16.log
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_bench_n tools/tc_bench_n.cu -lcuda > /dev/null 2>&1
bash tools/prof_all.sh > gpurun_out/prof_all.log 2>&1
tail -5 gpurun_out/prof_all.log
cat gpurun_out/bench_r02_c4.json
