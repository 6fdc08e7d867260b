# MGS per-launch cost at the GMRES sizes (see tools/mgs_bench.cu)
set -e
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1704_04549_b200/csrc -Iinclude tools/mgs_bench.cu paper_1704_04549_b200/csrc/blas.cu -o /tmp/mb0
for n in 1048576 1806336 5451776; do for K in 1 25; do /tmp/mb0 $n $K; done; done
