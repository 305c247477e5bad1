#!/bin/bash
# Experiment library: the sources named by SRCS (default scan_lm.cu) recompiled with extra -D flags,
# linked with the release objects.
#   [SRCS="coarse_tc scan_lm"] tools/exp_build.sh NAME -DFOO=1 ...  ->  exp/libv3db_NAME.so
#   (load with V3DB_LIB=$PWD/exp/libv3db_NAME.so)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
python -m paper_2603_03065_b200.build >/dev/null
mkdir -p exp/obj_$name
B=paper_2603_03065_b200
SRCS=${SRCS:-scan_lm}
cp $B/build/*.o exp/obj_$name/
for f in $SRCS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O3 "$@" -Iinclude -c $B/csrc/$f.cu -o exp/obj_$name/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/libv3db_$name.so exp/obj_$name/*.o
rm -rf exp/obj_$name
echo exp/libv3db_$name.so
