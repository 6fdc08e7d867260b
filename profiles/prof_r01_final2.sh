# Round-1 evidence (second session): bench lines (cfg2 p=15 headline, p sweep, cfg4, reference arm),
# launch lists, and ncu --set full captures of the changed kernels. Writes gpurun_out/r01b_*.
mkdir -p gpurun_out
O=gpurun_out
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > $O/r01b_bench.log 2>&1; tail -1 $O/r01b_bench.log > $O/r01b_bench.json
for p in 4 8 20 30; do
  timeout -s KILL 300 python bench.py --p $p --steps 3 --warmup 3 --no-cpu-baseline > $O/r01b_bench_p$p.log 2>&1
  tail -1 $O/r01b_bench_p$p.log > $O/r01b_bench_p$p.json
done
timeout -s KILL 600 python bench.py --case cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/r01b_bench_cfg4.log 2>&1; tail -1 $O/r01b_bench_cfg4.log > $O/r01b_bench_cfg4.json
TPDG_GPU_KRON=mma timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/r01b_bench_mma.log 2>&1; tail -1 $O/r01b_bench_mma.log > $O/r01b_bench_mma.json
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-profile"
NCU="ncu --set full --clock-control none --import-source on -c 1 --launch-skip 3"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01b_launches.csv $B > $O/r01b_ll.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01b_launches_p30.csv $B --p 30 > $O/r01b_ll30.log 2>&1
timeout -s KILL 300 $NCU -k regex:kron2d_ew -o $O/r01b_kron2d_ew $B > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:fb_apply -o $O/r01b_fb_apply $B --p 30 > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:jv2d_mma -o $O/r01b_jv2d $B > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:mgs_reg -o $O/r01b_mgs $B > /dev/null 2>&1
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/r01b_ref.log 2>&1; tail -1 $O/r01b_ref.log > $O/r01b_bench_reference.json
ls $O/r01b_*
