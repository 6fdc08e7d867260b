cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
run() {
  CMD="python bench.py --case $1 --p $2 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile"
  timeout 900 ncu --metrics $M --clock-control none -k regex:"$3" -s $4 -c $5 --csv $CMD 2>/dev/null | grep -E "dram__|gpu__time" > gpurun_out/traffic_$6.csv
  echo "$6 $(wc -l < gpurun_out/traffic_$6.csv)"
}
run cfg4 15 "kron3d_inv|jv3d_fast" 20 2 cfg4_pcjv
run cfg4 15 "mgs_bulk" 40 1 cfg4_mgs
