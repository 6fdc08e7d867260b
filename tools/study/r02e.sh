cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_loopback.py -q -x -s 2>&1 | grep -E "ranks|passed|failed|Error|assert" | tail -20
timeout -s KILL 1500 python -m pytest tests -q -m gpu 2>&1 | tail -5
