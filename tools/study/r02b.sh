cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -q -m gpu -k "glibm or parity or full_configs or dropin or cache or jv_bench" -x -s > gpurun_out/r02b_pt.log 2>&1; tail -5 gpurun_out/r02b_pt.log
grep -E "GPU-formed|bit-identical|fallbacks [0-9]" gpurun_out/r02b_pt.log | head -40
