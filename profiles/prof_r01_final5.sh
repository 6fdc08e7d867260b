# Final round-1 evidence (end of the second session): default bench line, p sweep, cfg4, launch list. r01e_*.
mkdir -p gpurun_out
O=gpurun_out
timeout -s KILL 900 python bench.py > $O/r01e_bench.log 2>&1; tail -1 $O/r01e_bench.log > $O/r01e_bench.json
for p in 4 8 20 30; do
  timeout -s KILL 300 python bench.py --p $p --steps 3 --warmup 3 --no-cpu-baseline > $O/r01e_bench_p$p.log 2>&1
  tail -1 $O/r01e_bench_p$p.log > $O/r01e_bench_p$p.json
done
timeout -s KILL 600 python bench.py --case cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/r01e_bench_cfg4.log 2>&1; tail -1 $O/r01e_bench_cfg4.log > $O/r01e_bench_cfg4.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01e_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-profile > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -c 1 --launch-skip 3 -k regex:jv2d_mma -o $O/r01e_jv2d python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-profile > /dev/null 2>&1
ls $O/r01e_*
