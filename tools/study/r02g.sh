cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 1500 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "ours rc=$?"
timeout -s KILL 1500 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_ref.err; echo "ref rc=$?"
tail -c 600 gpurun_out/r02_bench_reference.json
