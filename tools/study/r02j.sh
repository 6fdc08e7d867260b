cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02j_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02j_gpu_tests.log
timeout -s KILL 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r02j_bench.json'));print(d['value'],d['e2e']['value'],{k:v['avg_us'] for k,v in d['kernels'].items()})"
