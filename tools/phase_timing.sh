# Per-phase timing experiment of fwd_plane (CHK_DEBUG_FLAGS: 4 = debug mode, +1 = skip the
# transform phase of fwd_plane).  Numbers are per-launch averages (us); not a bench result.
for f in 4 5; do CHK_DEBUG_FLAGS=$f python bench.py --steps 1 --warmup 1 --config 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('flags',$f,{k:v['avg_us'] for k,v in d['kernels'].items()})"; done
