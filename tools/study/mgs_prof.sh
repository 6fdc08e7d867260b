# cfg4 MGS evidence after the 512 x 2 change: DRAM per launch, launch list, one full capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --case cfg4 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"mgs_bulk" -s 40 -c 1 --csv $B 2>/dev/null | grep -E "dram__|gpu__time" > gpurun_out/traffic_cfg4_mgs.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_cfg4.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mgs_bulk" -s 40 -c 1 -o gpurun_out/r02_cfg4_mgs_bulk -f $B > /dev/null 2>&1
ls -la gpurun_out | grep -E "mgs|launches"
