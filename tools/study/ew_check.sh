cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m pytest tests/test_gpu_full_pc_parity.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
python bench.py --case cfg2 --p 15 --steps 10 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ew_bench.json 2> gpurun_out/ew_bench.err; tail -c 1500 gpurun_out/ew_bench.json
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"kron2d_ew" -s 20 -c 2 --csv python bench.py --case cfg2 --p 15 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile 2>/dev/null | grep -E "dram__|gpu__time" > gpurun_out/traffic_ew.csv
cat gpurun_out/traffic_ew.csv
