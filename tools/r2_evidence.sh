#!/bin/bash
# Round-2 evidence pass on the GPU box:
#   gpurun --timeout 3000 -- 'bash tools/r2_evidence.sh r2e'
# smoke, the full -m gpu suite, bench lines for configs 3/4/5, the config-3 launch
# list (ncu --metrics gpu__time_duration.sum) and ncu --set full summaries.
TAG=${1:-r2e}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench3.json 2> gpurun_out/${TAG}_bench3.err
for c in 4 5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench$c.json 2> gpurun_out/${TAG}_bench$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/${TAG}_launches_config3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 1500 bash tools/ncu_round.sh ${TAG} "3 4 5" > gpurun_out/${TAG}_ncu_round.log 2>&1
du -sh gpurun_out
