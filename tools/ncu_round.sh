#!/bin/bash
# ncu --set full captures of the steady-state kernels (run on the GPU box).  The
# reports stay in /tmp; their raw metric pages, per-kernel source pages and
# summaries come back in gpurun_out/ (the 64 MiB pull limit).
TAG=${1:-r2}
CFGS=${2:-"3 4 5"}
mkdir -p gpurun_out
for c in $CFGS; do
  case $c in
    3) K='mid_column|pair_plane'; S=12; N=2; B=256; DOF=268435456 ;;
    4) K='mid_column|fwd_plane|inv_plane'; S=9; N=3; B=16; DOF=268435456 ;;
    5) K='mid_column|fwd_plane|inv_plane'; S=9; N=3; B=1; DOF=134217728 ;;
    2) K='mid_column|fwd_plane|inv_plane'; S=9; N=3; B=64; DOF=16777216 ;;
  esac
  R=/tmp/${TAG}_config$c
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $N -o $R -f \
    python tools/run_solve.py --config $c --batch $B > gpurun_out/${TAG}_ncu$c.log 2>&1
  ncu -i $R.ncu-rep --page raw --csv > gpurun_out/${TAG}_config${c}_raw.csv 2>&1
  python tools/ncu_summary.py $R.ncu-rep $DOF > gpurun_out/${TAG}_config${c}_summary.jsonl 2>&1
  for k in $(echo $K | tr '|' ' '); do
    ncu -i $R.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:$k --launch-count 1 \
      > /tmp/${TAG}_src_${c}_$k.csv 2>&1
    python tools/ncu_lines.py $R.ncu-rep $k 40 > gpurun_out/${TAG}_config${c}_lines_$k.txt 2>&1
    gzip -c /tmp/${TAG}_src_${c}_$k.csv > gpurun_out/${TAG}_config${c}_src_$k.csv.gz
  done
done
du -sh gpurun_out
