# Round-1 evidence run: launch list + ncu --set full captures of the top kernels (cfg2 p=15, cfg4)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-profile"
NCU="ncu --set full --clock-control none --import-source on -c 1 --launch-skip 3"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01f_launches.csv $B > gpurun_out/r01f_ll.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01f_launches_cfg4.csv $B --case cfg4 > gpurun_out/r01f_ll4.log 2>&1
timeout -s KILL 300 $NCU -k regex:kron2d_mma -o gpurun_out/r01f_kron2d $B > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:jv2d_mma -o gpurun_out/r01f_jv2d $B > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:mgs_reg -o gpurun_out/r01f_mgs $B > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:kron3d_mma -o gpurun_out/r01f_kron3d $B --case cfg4 > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:jv3d_sized -o gpurun_out/r01f_jv3d $B --case cfg4 > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:mgs_split -o gpurun_out/r01f_mgs3d $B --case cfg4 > /dev/null 2>&1
TPDG_GPU_FAITHFUL=1 timeout -s KILL 300 python tools/pc_sensitivity.py 2>&1 | tail -1 > gpurun_out/sens_faithful.txt
timeout -s KILL 300 python tools/pc_sensitivity.py 2>&1 | tail -1 > gpurun_out/sens_mma.txt
ls gpurun_out
