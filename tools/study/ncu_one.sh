# one ncu --set full capture of a bench kernel: tools/study/ncu_one.sh <case> <p> <kernel regex> <skip> <out name>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c 1 -o gpurun_out/$5 -f \
  python bench.py --case $1 --p $2 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-clocks --no-profile > gpurun_out/$5.log 2>&1
ls -la gpurun_out/$5.ncu-rep
