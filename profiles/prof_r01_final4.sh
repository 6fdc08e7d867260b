# Final round-1 evidence: default bench (N=1, as the driver runs it), reference arm, p sweep, cfg4,
# launch list and ncu of the headline's top kernels. gpurun_out/r01d_*.
mkdir -p gpurun_out
O=gpurun_out
timeout -s KILL 900 python bench.py > $O/r01d_bench.log 2>&1; tail -1 $O/r01d_bench.log > $O/r01d_bench.json
timeout -s KILL 900 python bench.py --impl reference > $O/r01d_ref.log 2>&1; tail -1 $O/r01d_ref.log > $O/r01d_bench_reference.json
for p in 4 8 20 30; do
  timeout -s KILL 300 python bench.py --p $p --steps 3 --warmup 3 --no-cpu-baseline > $O/r01d_bench_p$p.log 2>&1
  tail -1 $O/r01d_bench_p$p.log > $O/r01d_bench_p$p.json
done
timeout -s KILL 600 python bench.py --case cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/r01d_bench_cfg4.log 2>&1; tail -1 $O/r01d_bench_cfg4.log > $O/r01d_bench_cfg4.json
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-profile"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01d_launches.csv $B > $O/r01d_ll.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -c 1 --launch-skip 3 -k regex:kron2d_ew -o $O/r01d_kron2d_ew $B > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/r01d_smoke.log 2>&1
ls $O/r01d_*
