#!/bin/bash
# ncu --set full of the persistent dense PCG (symmetric use, S right-hand sides, n = $1, S = $2)
n=${1:-50000}; S=${2:-4}; tag=${3:-dense}
ncu --set full --import-source on --clock-control none -k regex:pcg_persistent -c 1 \
    -o gpurun_out/ncu_${tag}_S${S} -f python tools/dense_pcg_timing.py $n $S 1 > gpurun_out/ncu_${tag}_S${S}.log 2>&1
echo ncu_rc=$?
