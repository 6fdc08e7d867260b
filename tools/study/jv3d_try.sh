cd $GRAFT_REPO_ROOT
: > gpurun_out/jv3d_try.txt
for m in ${MINBS:-4 3}; do
echo "== MINB $m" >> gpurun_out/jv3d_try.txt
TPDG_JV3D_MINB=$m timeout 600 python -m pytest -q -m gpu tests/test_gpu_jv_bench_parity.py tests/test_gpu_parity.py -k "cfg4 or 3d or euler3d" 2>&1 | tail -1 >> gpurun_out/jv3d_try.txt
TPDG_JV3D_MINB=$m timeout 300 python bench.py --case cfg4 --no-extras --steps 3 --warmup 2 --no-cpu-baseline --no-clocks 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), d.get('iterations_per_solve'), {k:(round(v['avg_us'],1), round(v['roofline_frac'],3)) for k,v in d['kernels'].items()})" >> gpurun_out/jv3d_try.txt 2>&1
done
cat gpurun_out/jv3d_try.txt
if [ -n "$NCU" ]; then
CMD="python bench.py --case cfg4 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile"
TPDG_JV3D_MINB=$NCU $CMD > gpurun_out/plain.log 2>&1 && TPDG_JV3D_MINB=$NCU ncu --set full --clock-control none --import-source on -k regex:"jv3d_fast" -s 20 -c 1 -o gpurun_out/${OUT:-r02_jv3d_c} $CMD > gpurun_out/ncu_jv3d.log 2>&1
tail -1 gpurun_out/ncu_jv3d.log
fi
