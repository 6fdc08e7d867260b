cd $GRAFT_REPO_ROOT
CMD="python bench.py --case cfg4 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"mgs_split|kron3d" -s 40 -c 2 -o gpurun_out/r02_cfg4_mgs_kron $CMD > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
