# Round-1 evidence refresh (after the fused Givens / formation changes): headline bench with CPU
# baseline, cfg4, p sweep, launch list and ncu captures of the fused MGS kernel. gpurun_out/r01c_*.
mkdir -p gpurun_out
O=gpurun_out
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > $O/r01c_bench.log 2>&1; tail -1 $O/r01c_bench.log > $O/r01c_bench.json
for p in 4 8 20 30; do
  timeout -s KILL 300 python bench.py --p $p --steps 3 --warmup 3 --no-cpu-baseline > $O/r01c_bench_p$p.log 2>&1
  tail -1 $O/r01c_bench_p$p.log > $O/r01c_bench_p$p.json
done
timeout -s KILL 600 python bench.py --case cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/r01c_bench_cfg4.log 2>&1; tail -1 $O/r01c_bench_cfg4.log > $O/r01c_bench_cfg4.json
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-profile"
NCU="ncu --set full --clock-control none --import-source on -c 1 --launch-skip 3"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01c_launches.csv $B > $O/r01c_ll.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01c_launches_cfg4.csv $B --case cfg4 > $O/r01c_ll4.log 2>&1
timeout -s KILL 300 $NCU -k regex:mgs_reg -o $O/r01c_mgs $B > /dev/null 2>&1
timeout -s KILL 300 $NCU -k regex:make_factors -o $O/r01c_make_factors $B > /dev/null 2>&1
ls $O/r01c_*
