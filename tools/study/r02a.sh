cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r02a_pt.log 2>&1; tail -5 gpurun_out/r02a_pt.log
NOTEST=1 CASES="cfg2 cfg4" bash profiles/quick.sh
timeout -s KILL 900 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; tail -c 3000 gpurun_out/r02a_bench.json
