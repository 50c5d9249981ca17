#!/bin/bash
# on the GPU box: alternate bench runs of the default library and tmp_libs/*.so (same box, back to back)
# tools/ab_run.sh TAG CONFIG ROUNDS lib1 lib2 ...
TAG=$1; C=$2; R=$3; shift 3
mkdir -p gpurun_out
for r in $(seq 1 $R); do
  for L in default "$@"; do
    if [ "$L" = default ]; then unset CHK_LIB_PATH; else export CHK_LIB_PATH=$PWD/tmp_libs/$L.so; fi
    timeout 600 python bench.py --config $C --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/${TAG}_${L}_$r.json 2>/dev/null
  done
done
unset CHK_LIB_PATH
