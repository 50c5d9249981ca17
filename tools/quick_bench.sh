#!/bin/bash
# quick A/B on the GPU box: parity subset + bench lines for the given configs
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -q -p no:cacheprovider -x > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_bench$c.json 2> gpurun_out/${TAG}_bench$c.err
done
