cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -q -m gpu 2>&1 | tail -5
NOTEST=1 CASES="cfg2 cfg4" bash profiles/quick.sh
