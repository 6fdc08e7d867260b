# quick GPU check: gpu tests + kernel times per case -> gpurun_out/quick.txt
mkdir -p gpurun_out
[ -z "$NOTEST" ] && timeout -s KILL ${TTEST:-900} python -m pytest tests -q -m gpu ${PTARGS} > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log > gpurun_out/quick.txt
for c in ${CASES:-cfg2 cfg4}; do
timeout -s KILL 300 python bench.py --case $c --no-extras --steps 3 --warmup 2 --no-cpu-baseline --no-clocks 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],3), d.get('iterations_per_solve'), {k:(round(v['avg_us'],1), round(v['roofline_frac'],3)) for k,v in d['kernels'].items()}, 'form_ms', round(d.get('form_ms',0),1))" >> gpurun_out/quick.txt 2>&1
done
cat gpurun_out/quick.txt
