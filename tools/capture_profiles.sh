#!/bin/bash
# Round-end evidence for profiles/ (run on the GPU box: gpurun -- 'bash tools/capture_profiles.sh TAG').
# Bench lines, the config-3 launch list and ncu --set full summaries (the .ncu-rep stays in /tmp).
TAG=${1:-r1d}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_default.json 2> gpurun_out/${TAG}_default.err
python bench.py --config 5 --no-cpu-baseline > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/${TAG}_launches_config3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mid_column|pair_plane" -s 12 -c 2 -o /tmp/${TAG}_config3 \
  python tools/run_solve.py --config 3 --batch 256 > gpurun_out/${TAG}_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/${TAG}_config3.ncu-rep 268435456 > gpurun_out/${TAG}_ncu_config3.txt 2>&1
python tools/ncu_lines.py /tmp/${TAG}_config3.ncu-rep pair_plane > gpurun_out/${TAG}_lines_pair.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mid_column|fwd_plane|inv_plane" -s 6 -c 3 -o /tmp/${TAG}_config5 \
  python tools/run_solve.py --config 5 --batch 1 > gpurun_out/${TAG}_ncu_full5.log 2>&1
python tools/ncu_summary.py /tmp/${TAG}_config5.ncu-rep 134217728 > gpurun_out/${TAG}_ncu_config5.txt 2>&1
