#!/bin/bash
# Study builds: libtpdg_gpu.so variants with kron.cu compiled under extra flags, e.g.
#   [SRC=kron_ew] tools/kron_variants.sh a:-DSOME_FLAG=1 b:-DSOME_FLAG=2
# -> paper_1704_04549_b200/_build/var/<name>/libtpdg_gpu.so (select with TPDG_GPU_LIB=...)
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_1704_04549_b200
make -C $P/csrc -j8 >/dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
case "${SRC:-kron}" in kron|kron_ew|kron_fallback|form) FMAD=-fmad=false ;; *) FMAD= ;; esac
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  (d=$P/_build/var/$name; mkdir -p $d
   /usr/local/cuda/bin/nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -I$P/csrc -I$R/include \
     --expt-relaxed-constexpr $FMAD $flags -c $P/csrc/${SRC:-kron}.cu -o $d/${SRC:-kron}.o
   objs=$(ls $P/_build/*.o | grep -v "/${SRC:-kron}.o$")
   /usr/local/cuda/bin/nvcc $ARCH -shared -o $d/libtpdg_gpu.so $d/${SRC:-kron}.o $objs -L/usr/lib/x86_64-linux-gnu -lnccl
   echo built $name) &
done
wait
