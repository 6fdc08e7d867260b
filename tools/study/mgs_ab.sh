cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in ${NS_LIST:-5451776 3936256 1806336}; do
for v in SPLIT WIDE NARROW; do
 case $v in SPLIT) export TPDG_GPU_MGS_SPLIT=1; unset TPDG_GPU_MGS_WIDE;; WIDE) unset TPDG_GPU_MGS_SPLIT; export TPDG_GPU_MGS_WIDE=1;; NARROW) unset TPDG_GPU_MGS_SPLIT TPDG_GPU_MGS_WIDE;; esac
 echo "$v: $(timeout 120 tools/mgs_bench_bin $n 30 | tr '\n' ' ')"
done; done 2>&1 | tee gpurun_out/mgs_ab.txt
