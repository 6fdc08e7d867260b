cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m pytest tests/test_gpu_full_configs.py -x -q -k cfg4 2>&1 | tail -2
python bench.py --case cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/cfg4_bench.json 2> gpurun_out/cfg4_bench.err
python - <<'PY'
import json
d = json.loads(open('gpurun_out/cfg4_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()})
PY
