#!/bin/bash
# ncu capture of one stand-in kernel (GPU box): tools/study/standin_ncu.sh cfg3 kron2d_sized out_name
set -e
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:$2 -s 2 -c 1 -o gpurun_out/$3 -f \
  python tools/study/standin_time.py $1 > gpurun_out/$3.log 2>&1
