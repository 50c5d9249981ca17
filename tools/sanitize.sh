#!/bin/bash
# compute-sanitizer over reduced solves of every grid-size path (run on the GPU box):
#   gpurun -- 'bash tools/sanitize.sh TAG'
TAG=${1:-r2}
mkdir -p gpurun_out
CS=compute-sanitizer
run() {  # tool, label, timeout, args...
  local tool=$1 label=$2 to=$3; shift 3
  timeout $to $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/run_solve.py "$@" \
    > gpurun_out/${TAG}_san_${tool}_${label}.log 2>&1
  echo "$tool $label rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${TAG}_san_${tool}_${label}.log | tail -1)" >> gpurun_out/${TAG}_sanitize.txt
}
: > gpurun_out/${TAG}_sanitize.txt
for tool in memcheck synccheck racecheck; do
  run $tool c1 900 --config 1 --batch 2
  run $tool c2 900 --config 2 --batch 8
  run $tool c3pair 1500 --config 3 --batch 32
  run $tool c4 1500 --config 4 --batch 2
  run $tool c5 1500 --config 5 --batch 1
done
run memcheck c2fourier 600 --config 2 --batch 4 --kind fourier
cat gpurun_out/${TAG}_sanitize.txt
