cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in 5451776 3936256 1806336 1048576; do tools/mgs_bench_bin $n 30 | tr '\n' ' '; echo; done | tee gpurun_out/mgs_new.txt
timeout -s KILL 1200 python -m pytest tests -q -m gpu -k "full_configs or multi_path or block_jacobi or report" -x -s 2>&1 | grep -E "its|passed|failed|Error" | tail -20
NOTEST=1 CASES="cfg2 cfg4" bash profiles/quick.sh
