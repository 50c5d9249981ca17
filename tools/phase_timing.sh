# Timing experiments (CHK_DEBUG_FLAGS): 4 = debug mode (no breakdown stop), +1 = fwd_plane
# without its transform phase, +8 = mid pass without phase-B work.  Not bench results.
for f in 4 12; do CHK_DEBUG_FLAGS=$f python bench.py --steps 1 --warmup 1 --config 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('flags',$f,{k:v['avg_us'] for k,v in d['kernels'].items()})"; done
