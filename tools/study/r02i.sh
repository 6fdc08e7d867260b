cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/study/ncu_one.sh cfg4 15 kron3d_inv_kernel 5 r02i_kron3d
bash tools/study/ncu_one.sh cfg4 15 jv3d_fast_kernel 5 r02i_jv3d
