# Per-source-line warp-stall summary of the C4 query kernels (run under gpurun from the repo root):
# one ncu --set full capture with source, summarised on the box by tools/ncu_lines.py.
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"lm_kernel|lm_select_warp|merge_kernel|coarse_tc_kernel" -c 4 -o gpurun_out/c4_lines python tools/prof_query.py --config c4 --reps 1 > gpurun_out/c4_lines.log 2>&1
for k in lm_kernel lm_select_warp merge_kernel coarse_tc_kernel; do
  echo "## $k" >> gpurun_out/ncu_r02_c4_lines.txt
  python tools/ncu_lines.py gpurun_out/c4_lines.ncu-rep $k 25 | cut -c1-200 >> gpurun_out/ncu_r02_c4_lines.txt
done
rm -f gpurun_out/c4_lines.ncu-rep
