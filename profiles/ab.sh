# A/B: kernel times of variant libraries (TPDG_GPU_LIB) on cfg2 / cfg4
for v in $VARIANTS; do
for c in ${CASES:-cfg2 cfg4}; do
TPDG_GPU_LIB=$PWD/paper_1704_04549_b200/_build/var/lib$v.so timeout -s KILL 200 python bench.py --case $c --steps 3 --warmup 2 --no-cpu-baseline --no-clocks 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v$v $c', round(d['value'],3), d['config'].get('iterations_per_solve'), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, 'form_ms', round(d.get('form_ms',0),1))"
done; done
