mkdir -p gpurun_out
set -x
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-profile"
NCU="ncu --set full --clock-control none --import-source on -c 1 --launch-skip 3"
timeout -s KILL 300 $NCU -k regex:kron2d_sized -o gpurun_out/r01b_kron2d $B > gpurun_out/n1.log 2>&1
timeout -s KILL 300 $NCU -k regex:jv2d_sized -o gpurun_out/r01b_jv2d $B > gpurun_out/n2.log 2>&1
timeout -s KILL 300 $NCU -k regex:mgs_ -o gpurun_out/r01b_mgs $B > gpurun_out/n3.log 2>&1
timeout -s KILL 300 $NCU -k regex:kron3d_sized -o gpurun_out/r01b_kron3d $B --case cfg4 > gpurun_out/n4.log 2>&1
timeout -s KILL 300 $NCU -k regex:jv3d_sized -o gpurun_out/r01b_jv3d $B --case cfg4 > gpurun_out/n5.log 2>&1
ls -la gpurun_out
