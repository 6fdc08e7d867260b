cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --case cfg4 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile"
$CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
for k in ${KLIST:-mgs_split kron3d jv3d_fast}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 30 -c 1 -o gpurun_out/r02_cfg4_$k $CMD > gpurun_out/ncu_$k.log 2>&1
tail -2 gpurun_out/ncu_$k.log
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg4.csv $CMD > /dev/null 2>&1
ls -la gpurun_out
