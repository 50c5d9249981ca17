mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r1d_launches_config3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1d_ncu_launch.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"mid_column|pair_plane" -s 12 -c 2 -o gpurun_out/r1d_config3 python tools/run_solve.py --config 3 --batch 256 > gpurun_out/r1d_ncu_full.log 2>&1
echo full rc=$?
ncu --set full --clock-control none --import-source on -k regex:"mid_column|fwd_plane|inv_plane" -s 6 -c 3 -o gpurun_out/r1d_config5 python tools/run_solve.py --config 5 --batch 1 > gpurun_out/r1d_ncu_full5.log 2>&1
echo full5 rc=$?
ls -la gpurun_out
