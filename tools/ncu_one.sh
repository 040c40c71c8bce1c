#!/bin/bash
# ncu --set full of one march kernel at late time (C2, 64 samples, t = T):
#   bash tools/ncu_one.sh <kernel-regex> [T] [tag]   -> gpurun_out/one_<tag>.ncu-rep
K=$1; T=${2:-0.002}; TAG=${3:-$1}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"$K" --launch-skip 20 -c 1 \
    -o gpurun_out/one_$TAG -f python bench.py --steps 10 --warmup 3 --t-start $T \
    --no-cpu-baseline --no-postproc --no-e2e --no-roofline > gpurun_out/one_$TAG.log 2>&1
