#!/bin/bash
# Build a compile-time variant of the library beside the default one:
#   tools/build_variant.sh NAME "-DFLAG ..."  -> paper_2605_25282_b200/lib/libvlbm_NAME.so
# (the default build is restored afterwards; use with VLBM_LIB=... / tools/ab_lib.sh)
cd "$(dirname "$0")/.." || exit 1
VLBM_NVCC_EXTRA="$2" python -m paper_2605_25282_b200.build -f > /dev/null || { echo "$1: build failed"; exit 1; }
cp paper_2605_25282_b200/lib/libvlbm_b200.so paper_2605_25282_b200/lib/libvlbm_$1.so
python -m paper_2605_25282_b200.build -f > /dev/null
ls -la paper_2605_25282_b200/lib/libvlbm_$1.so
