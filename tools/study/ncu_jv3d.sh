cd $GRAFT_REPO_ROOT
CMD="python bench.py --case cfg4 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile"
export TPDG_JV3D_MINB=${MINB:-3}
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-jv3d_fast}" -s ${SKIP:-20} -c 1 -o gpurun_out/${OUT:-r02_jv3d} $CMD > gpurun_out/ncu_jv3d.log 2>&1
tail -2 gpurun_out/ncu_jv3d.log
