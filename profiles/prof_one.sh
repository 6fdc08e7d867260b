# usage: bash profiles/prof_one.sh <kernel-regex> <out-name> [bench args...]
mkdir -p gpurun_out
K=$1; O=$2; shift 2
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -c 1 --launch-skip 3 -k regex:$K \
  -o gpurun_out/$O python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-clocks --no-profile "$@" > gpurun_out/$O.log 2>&1
tail -3 gpurun_out/$O.log
