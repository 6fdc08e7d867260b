cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x -s -k "3d or cfg4 or parity or full_configs" 2>&1 | grep -E "cfg4|q=11|3d|passed|failed|Error|assert" | tail -30
NOTEST=1 CASES="cfg4" bash profiles/quick.sh
