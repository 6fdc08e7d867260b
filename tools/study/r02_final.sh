# Round-2 final evidence (run under gpurun): plain bench first, then DRAM traffic per kernel, launch lists and
# one full capture per cfg4 kernel. Outputs in gpurun_out/ (copied to profiles/ by hand).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
B="--steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile"
python bench.py --case cfg4 $B > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
run() {  # case p regex skip count tag
  timeout 900 ncu --metrics $M --clock-control none -k regex:"$3" -s $4 -c $5 --csv python bench.py --case $1 --p $2 $B 2>/dev/null | grep -E "dram__|gpu__time" > gpurun_out/traffic_$6.csv
  echo "$6 $(wc -l < gpurun_out/traffic_$6.csv)"
}
run cfg4 15 "kron3d_inv_kernel|jv3d_fast" 20 2 cfg4_pcjv
run cfg4 15 "mgs_stream" 40 1 cfg4_mgs
run cfg2 15 "kron2d_ew|jv2d_mma" 20 2 cfg2p15_pcjv
run cfg2 15 "mgs_stream" 40 1 cfg2p15_mgs
run cfg2 30 "kron2d_ew|fb_panel|jv2d_mma" 30 3 cfg2p30_pcjv
run cfg2 30 "mgs_stream" 40 1 cfg2p30_mgs
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_cfg4.csv python bench.py --case cfg4 $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg2p15.csv python bench.py --case cfg2 --p 15 $B > /dev/null 2>&1
for k in mgs_stream kron3d_inv_kernel jv3d_fast; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 40 -c 1 -o gpurun_out/r02f_cfg4_$k -f python bench.py --case cfg4 $B > gpurun_out/ncu_$k.log 2>&1
  tail -1 gpurun_out/ncu_$k.log
done
ls gpurun_out | grep -E "traffic_|r02f_|r02_launches"
