#!/bin/bash
# Scan time vs stage geometry (experiments; V3DB_SEG / V3DB_NS force the pipeline shape).
cfg=${1:-c4}
for sn in "16 4" "15 4" "12 5" "8 8" "10 6" "8 6" "4 12" "16 3"; do
  set -- $sn
  envs="$envs,V3DB_SEG=$1:V3DB_NS=$2"
done
python tools/time_query.py --config $cfg --algos 2 --envs "${envs#,}"
