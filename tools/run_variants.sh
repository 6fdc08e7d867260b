# GPU: tools/ktime.py for the default build and every study build under _build/var/ -> gpurun_out/var.txt
mkdir -p gpurun_out; : > gpurun_out/var.txt
for p in ${PS:-15}; do
  timeout -s KILL 120 python tools/ktime.py --p $p --save /tmp/base_$p.npy ${KT_ARGS} >> gpurun_out/var.txt 2>&1
  for d in paper_1704_04549_b200/_build/var/*/; do
    n=$(basename $d); [ -n "$VARS" ] && ! echo " $VARS " | grep -q " $n " && continue
    echo -n "$n " >> gpurun_out/var.txt
    TPDG_GPU_LIB=$d/libtpdg_gpu.so timeout -s KILL 120 python tools/ktime.py --p $p --check /tmp/base_$p.npy ${KT_ARGS} >> gpurun_out/var.txt 2>&1
  done
done
cat gpurun_out/var.txt
