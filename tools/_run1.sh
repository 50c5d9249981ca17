mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/r1d_default.json 2> gpurun_out/r1d_default.err; tail -c 600 gpurun_out/r1d_default.json
python bench.py --config 5 --no-cpu-baseline > gpurun_out/r1d_c5.json 2> gpurun_out/r1d_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r1d_launches_config3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1d_ncu_launch.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"mid_column|pair_plane" -s 12 -c 2 -o /tmp/r1d_config3 python tools/run_solve.py --config 3 --batch 256 > gpurun_out/r1d_ncu_full.log 2>&1
echo full rc=$?
python tools/ncu_summary.py /tmp/r1d_config3.ncu-rep 268435456 > gpurun_out/r1d_ncu_config3.txt 2>&1
python tools/ncu_lines.py /tmp/r1d_config3.ncu-rep pair_plane > gpurun_out/r1d_lines_pair.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mid_column|fwd_plane|inv_plane" -s 6 -c 3 -o /tmp/r1d_config5 python tools/run_solve.py --config 5 --batch 1 > gpurun_out/r1d_ncu_full5.log 2>&1
echo full5 rc=$?
python tools/ncu_summary.py /tmp/r1d_config5.ncu-rep 134217728 > gpurun_out/r1d_ncu_config5.txt 2>&1
du -sh gpurun_out
