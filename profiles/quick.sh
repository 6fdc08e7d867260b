# quick GPU check: gpu tests + cfg2 / cfg4 kernel times
timeout -s KILL 600 python -m pytest tests -x -q -m gpu > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
for c in cfg2 cfg4 $EXTRA; do
timeout -s KILL 200 python bench.py --case $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],3), d['iterations_per_solve'] if 'iterations_per_solve' in d else d['config'].get('iterations_per_solve'), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, 'form_ms', round(d.get('form_ms',0),1))"
done
