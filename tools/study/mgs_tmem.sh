cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in 5451776; do for v in tr0 tr4 tr8 tr16 tr0; do
echo "$v n=$n: $(timeout 120 tools/mgs_bench_${v}_bin $n 30 | head -1)"
done; done 2>&1 | tee gpurun_out/mgs_tmem.txt
