TAG=${1:-r2}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider -s > gpurun_out/${TAG}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
CHK_PROF_TRACE=gpurun_out/${TAG}_trace3.txt timeout 300 python tools/trace_solve.py --config 3 --batch 256 > gpurun_out/${TAG}_trace3.log 2>&1
